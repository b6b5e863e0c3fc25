// pxg_kernels.cu — the per-pass kernels of proxy-BDPT and the C ABI (include/pxg.h).
//
// One progressive pass (proj/src/proxy.cpp:683-827) is a fixed sequence of launches on the
// context's stream:
//   Stage 1 (pool, proxy.cpp:684-736)
//     k_pool_walks    one thread per pool walk: light walk on its own Philox stream, every
//                     dropout-eligible prefix end gets a 64-bit priority key
//     (CUB radix sort of the keys; the pool_budget smallest are kept, ordered by walk,end)
//     k_pool_entries  one thread per kept entry: re-trace its walk, dropout, 4 probes
//     k_pool_bounds   one thread: probes -> bucket max in entry order -> B per entry
//     k_recip_eval/   reciprocal runs in rounds: all pending tree nodes evaluated in parallel
//     k_recip_dfs     (node-keyed streams), then each run's DFS resumes over them
//     k_pool_finish   one thread: means, moments, validity, diagnostics, bucket lists
//   Stage 2 (per pixel, proxy.cpp:738-819)
//     k_trace         one thread per pixel: eye sub-path then light sub-path on the pixel's
//                     persistent stream -> SoA vertex pools in HBM
//     k_connect       one thread per pixel: all standard strategies with reciprocal-aware MIS
//     k_proxy         one thread per pixel: gamma draw, pool pick, proxy_connect
//                     (speculatively, before the gate is known)
//     k_gate          one thread per 10x10 gate cell: the reference's scan-order gate,
//                     proxy normalisation, film accumulation, grid shares
//   then the gamma rows are rebuilt from the pixel-order contribution sum.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <string>
#include <vector>

#include "pxg.h"
#include "pxg_host.h"
#include "pxg_wave.cuh"

using namespace pxg;

namespace {

constexpr int kBuckets = 4000;
constexpr int kS = 100, kT = 32;
thread_local std::string g_global_err;

struct ProxRec {
  double c[3];
  double u_gate;
  double q_sel;
  int t_label, chosen, key, flags;  // flags bit0 tp>=2, bit1 attempted, bit2 z_norm>0
};

struct GammaRec {
  double value;
  int bin;       // t*100+s, -1 none
  int pad;
};

struct PassState {  // device-resident per-pass scalars
  double kappa;
  int n_kept;
  int err;
  long long pool_kept_total;
};

#define CK(x)                                                                           \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) throw CudaErr(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct CudaErr {
  std::string msg;
  explicit CudaErr(std::string m) : msg(std::move(m)) {}
};
struct InvalidErr {
  std::string msg;
};
struct RuntimeErr {
  std::string msg;
};

template <typename T>
T* dalloc(size_t n) {
  T* p = nullptr;
  if (n == 0) n = 1;
  CK(cudaMalloc(&p, n * sizeof(T)));
  return p;
}
template <typename T>
T* dupload(const T* src, size_t n) {
  T* p = dalloc<T>(n);
  if (n) CK(cudaMemcpy(p, src, n * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

__device__ __forceinline__ Rng make_rng(uint64_t seed, uint32_t kind, uint32_t sub, uint64_t stream) {
  Rng r;
  r.r = pxg_rng_make(seed, kind, sub, stream);
  return r;
}

__device__ __forceinline__ uint64_t unit_stream(int pass, int walk) {
  return (static_cast<uint64_t>(pass) << 32) | static_cast<uint32_t>(walk);
}

__device__ __forceinline__ void set_err(int* err, int code) { atomicCAS(err, 0, code); }

// ------------------------------------------------------------------ Stage 1 kernels
// Eligible prefix ends of the traced pool walks get a 64-bit priority key each
// (the priority-reservoir replacement of Algorithm R, proxy.cpp:696-711).
__global__ void k_pool_keys(const PV* wpool, const int* wnv, int n_walks, uint64_t seed, int pass, int walk_begin,
                            unsigned long long* keys, unsigned* vals, int* count, int cap) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_walks) return;
  const int w = walk_begin + i;
  const int n = wnv[i];
  int flag[kMaxLight], emitter[kMaxLight];
  double pdf[kMaxLight];
  for (int k = 0; k < n; ++k) {
    const PV& v = wpool[static_cast<size_t>(k) * n_walks + i];
    flag[k] = v.flag;
    emitter[k] = v.emitter;
    pdf[k] = v.pdf_fwd;
  }
  for (int end = 2; end <= n; ++end) {
    if (flag[end - 1] != kSpecular) continue;
    if (!dropout_eligible(flag, emitter, pdf, end)) continue;
    Rng kr = make_rng(seed, PXG_KIND_RESERVOIR, static_cast<uint32_t>(end), unit_stream(pass, w));
    unsigned long long hi = pxg_next_u32(&kr.r);
    unsigned long long key = (hi << 32) | pxg_next_u32(&kr.r);
    int slot = atomicAdd(count, 1);
    if (slot < cap) {
      keys[slot] = key;
      vals[slot] = (static_cast<unsigned>(w) << 5) | static_cast<unsigned>(end);
    }
  }
}

__global__ void k_pool_entries(SceneView S, Mapper M, uint64_t seed, int pass, int n_ent, const unsigned* sel,
                               const PV* wpool, int n_walks, int walk_begin, IncHdr* inc, PV* prefix,
                               double* probe, int* probe_ok, int repeats) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_ent) return;
  const int w = static_cast<int>(sel[k] >> 5), end = static_cast<int>(sel[k] & 31u);
  PV v[kMaxLight];
  for (int q = 0; q < end; ++q) v[q] = wpool[static_cast<size_t>(q) * n_walks + (w - walk_begin)];
  IncHdr h;
  PV* pre = prefix + static_cast<size_t>(k) * kMaxLight;
  const bool ok = dropout(M, v, end, h, pre);
  h.walk = w;
  h.end = end;
  h.valid = ok ? 1 : 0;
  inc[k] = h;
  for (int i = 0; i < 4; ++i) probe_ok[k * 4 + i] = 0;
  if (!ok || repeats < 1) return;
  Rng pr = make_rng(seed, PXG_KIND_PROBE, static_cast<uint32_t>(end), unit_stream(pass, w));
  for (int i = 0; i < 4; ++i) {
    Cand c;
    support_sample(S, h, pre, pr, c);
    if (!(c.q > 0.0)) continue;
    double f = c.escaped ? 0.0 : target_density(S, h, pre, c.g);
    probe[k * 4 + i] = f / c.q;
    probe_ok[k * 4 + i] = 1;
  }
}

// pretrace_statistics (proj/src/subspace.cpp:190-218), one Philox stream per walk. The
// bucket max and count are order-independent, so atomics reproduce the sequential result.
__global__ void k_pretrace(SceneView S, Mapper M, uint64_t seed, int n_paths, double* max_ratio,
                           long long* ratio_cnt, int* touched, int* err) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= n_paths) return;
  Rng rng = make_rng(seed, PXG_KIND_PRETRACE, 0, static_cast<uint64_t>(w));
  PV v[7];
  const int n = trace_light_subpath(S, 7, rng, v, 1);
  for (int end = 2; end <= n; ++end) {
    if (v[end - 1].flag != kSpecular) continue;
    IncHdr h;
    if (!dropout(M, v, end, h, nullptr)) continue;
    for (int probe = 0; probe < 2; ++probe) {
      Cand c;
      support_sample(S, h, v, rng, c);
      if (!(c.q > 0.0)) continue;
      const double f = c.escaped ? 0.0 : target_density(S, h, v, c.g);
      const double r = f / c.q;
      if (!isfinite(r) || r < 0.0) {
        set_err(err, kErrRatio);
        return;
      }
      atomicMax(reinterpret_cast<unsigned long long*>(max_ratio + h.key),
                static_cast<unsigned long long>(__double_as_longlong(r)));
      atomicAdd(reinterpret_cast<unsigned long long*>(ratio_cnt + h.key), 1ull);
      touched[h.key] = 1;
    }
  }
}

// Sequential in pool order: B of entry k sees the probes of entries <= k (proxy.cpp:389-395).
__global__ void k_pool_bounds(int n_ent, const IncHdr* inc, const double* probe, const int* probe_ok,
                              double* max_ratio, long long* ratio_cnt, int* touched, double* bound, int* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int k = 0; k < n_ent; ++k) {
    const int key = inc[k].key;
    for (int i = 0; i < 4; ++i) {
      if (!probe_ok[k * 4 + i]) continue;
      const double r = probe[k * 4 + i];
      if (!isfinite(r) || r < 0.0) {
        set_err(err, kErrRatio);
        return;
      }
      max_ratio[key] = dmax(max_ratio[key], r);
      ratio_cnt[key] += 1;
      touched[key] = 1;
    }
    bound[k] = touched[key] ? 2.0 * max_ratio[key] : 0.0;
  }
}

// Phase A of the reciprocal runs: evaluate nodes [avail, avail + chunk) of every active
// run in parallel. Node k draws its support sample from (RECIP_NODE, k) and its split
// decision from (RECIP_SPLIT, k) (include/pxg_philox.h), so its value does not depend on
// the tree shape; draw_g (recip.hpp:69-77) and stochastic_split (recip.hpp:49-56).
__global__ void k_recip_eval(SceneView S, uint64_t seed, int pass, int repeats, long long cap, const IncHdr* inc,
                             const PV* prefix, const double* bound, const int* active, const int* n_active,
                             int chunk, const RunState* st, double* g, long long* nsplit, int* nerr) {
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long a = tid / chunk;
  if (a >= *n_active) return;
  const int j = active[a];
  const long long k = st[j].avail + tid % chunk;
  if (k >= cap) return;
  const int e = j / repeats, r = j % repeats;
  const IncHdr& h = inc[e];
  const PV* pre = prefix + static_cast<size_t>(e) * kMaxLight;
  const double B = bound[e];
  const uint64_t stream = pxg_recip_stream(pass, h.walk, h.end, r);
  Rng nr = make_rng(seed, PXG_KIND_RECIP_NODE, static_cast<uint32_t>(k), stream);
  int err = 0;
  const double gv = draw_g(S, h, pre, B, nr, err);
  long long n = 0;
  if (!err) {
    Rng sr = make_rng(seed, PXG_KIND_RECIP_SPLIT, static_cast<uint32_t>(k), stream);
    n = split_count(gv, sr, err);
  }
  const size_t o = static_cast<size_t>(j) * cap + k;
  g[o] = gv;
  nsplit[o] = n;
  nerr[o] = err;
}

// The two-point fixture f = {1, 3}, q = 1/2 (proj/tests/test_recip.cpp:16-23) as Phase A.
__global__ void k_twopoint_eval(uint64_t seed, double bound, long long cap, const int* active, const int* n_active,
                                int chunk, const RunState* st, double* g, long long* nsplit, int* nerr) {
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long a = tid / chunk;
  if (a >= *n_active) return;
  const int j = active[a];
  const long long k = st[j].avail + tid % chunk;
  if (k >= cap) return;
  Rng nr = make_rng(seed, PXG_KIND_RECIP_NODE, static_cast<uint32_t>(k), static_cast<uint64_t>(j));
  const int x = nr.next_double() < 0.5 ? 0 : 1;
  const double fx = x == 0 ? 1.0 : 3.0;
  const double gv = 1.0 - fx / (bound * 0.5);
  int err = 0;
  Rng sr = make_rng(seed, PXG_KIND_RECIP_SPLIT, static_cast<uint32_t>(k), static_cast<uint64_t>(j));
  const long long n = split_count(gv, sr, err);
  const size_t o = static_cast<size_t>(j) * cap + k;
  g[o] = gv;
  nsplit[o] = n;
  nerr[o] = err;
}

__global__ void k_recip_init(int runs, int repeats, const IncHdr* inc, const double* bound, RunState* st,
                             int* active, int* n_active, double* est, long long* cost, int* trunc) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= runs) return;
  RunState s;
  s.depth = s.cost = s.avail = 0;
  s.ret = 0.0;
  s.entering = 1;
  s.truncated = 0;
  s.err = 0;
  const int e = j / repeats;
  const bool live = inc ? (inc[e].valid && bound[e] > 0.0) : true;
  s.done = live ? 0 : 1;
  st[j] = s;
  est[j] = 0.0;
  cost[j] = 0;
  trunc[j] = 0;
  if (live) active[atomicAdd(n_active, 1)] = j;
}

// Phase B: resume the DFS of every active run over its newly evaluated nodes.
__global__ void k_recip_dfs(int repeats, long long cap, const double* bound, double fixed_bound, const int* active,
                            const int* n_active, int chunk, RunState* st, const double* g, const long long* nsplit,
                            const int* nerr, RecipFrame* frames, double* est, long long* cost, int* trunc,
                            int* next, int* n_next, int* err) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= *n_active) return;
  const int j = active[a];
  RunState s = st[j];
  s.avail = min(cap, s.avail + chunk);
  const double B = bound ? bound[j / repeats] : fixed_bound;
  const size_t o = static_cast<size_t>(j) * cap;
  const bool done = dfs_resume(s, g + o, nsplit + o, nerr + o, frames + o, B, cap);
  st[j] = s;
  if (!done) {
    next[atomicAdd(n_next, 1)] = j;
    return;
  }
  if (s.err) {
    set_err(err, s.err);
    return;
  }
  est[j] = s.ret;
  cost[j] = s.cost;
  trunc[j] = s.truncated;
}

__global__ void k_pool_finish(int n_ent, int repeats, IncHdr* inc, const double* bound, const double* est,
                              const int* trunc, double* sum_est, double* sum_sq, long long* est_cnt, int* touched,
                              long long* diag, int* diag_touched, int* kept, int* label_start, int* label_list,
                              PassState* ps) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int n_kept = 0;
  int label_count[kS];
  for (int s = 0; s < kS; ++s) label_count[s] = 0;
  for (int k = 0; k < n_ent; ++k) {
    IncHdr& h = inc[k];
    if (!h.valid) continue;
    const int key = h.key;
    diag_touched[key] = 1;
    bool valid = false;
    if (repeats >= 1 && bound[k] > 0.0) {
      double sum = 0.0, sq = 0.0;
      int tr = 0;
      for (int r = 0; r < repeats; ++r) {
        const double e = est[k * repeats + r];
        sum += e;
        sq += e * e;
        tr += trunc[k * repeats + r];
      }
      const double mean = sum / repeats;
      const double m2 = sq / repeats;
      diag[key * 5 + 3] += tr;
      if (isfinite(mean) && mean > 0.0) {
        valid = true;
        h.inverse_p = mean;
        h.inverse_p_m2 = m2;
        sum_est[key] += mean;
        sum_sq[key] += mean * mean;
        est_cnt[key] += 1;
        touched[key] = 1;
      }
    }
    diag[key * 5 + 2] += repeats;
    if (!valid) {
      diag[key * 5 + 4] += 1;
      continue;
    }
    kept[n_kept++] = k;
    label_count[h.s_label] += 1;
  }
  int acc = 0;
  for (int s = 0; s < kS; ++s) {
    label_start[s] = acc;
    acc += label_count[s];
  }
  label_start[kS] = acc;
  for (int s = 0; s < kS; ++s) label_count[s] = 0;
  for (int i = 0; i < n_kept; ++i) {
    const int s = inc[kept[i]].s_label;
    label_list[label_start[s] + label_count[s]++] = kept[i];
  }
  ps->n_kept = n_kept;
  ps->pool_kept_total += n_kept;
}

// ------------------------------------------------------------------ Stage 2 kernels
struct Stage2 {
  SceneView S;
  Mapper M;
  StatsView st;
  PV* eye;
  PV* light;
  int* n_eye;
  int* n_light;
  unsigned* ctr;
  double* bdpt;  // [n*3]
  int* eye_prims;
  int* light_prims;
  int n, row0, width, height, max_depth;
  uint64_t seed;
  int record_prims;
};

__global__ void k_record_prims(const PV* eye, const int* n_eye, const PV* light, const int* n_light, int n,
                               int max_depth, int* eye_prims, int* light_prims) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int ne = n_eye[i], nl = n_light[i];
  for (int k = 0; k <= max_depth; ++k)
    eye_prims[static_cast<size_t>(i) * (max_depth + 1) + k] = k < ne ? eye[static_cast<size_t>(k) * n + i].prim : -2;
  for (int k = 0; k < max_depth - 1; ++k)
    light_prims[static_cast<size_t>(i) * (max_depth - 1) + k] =
        k < nl ? light[static_cast<size_t>(k) * n + i].prim : -2;
}

__global__ void k_proxy(Stage2 P, int pass, int n_px_total, const IncHdr* inc, const PV* prefix,
                        const int* label_start, const int* label_list, const double* gamma_rows,
                        const PassState* ps, ProxRec* out, PV* scratch) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  ProxRec o;
  o.c[0] = o.c[1] = o.c[2] = 0.0;
  o.u_gate = 0.0;
  o.q_sel = 0.0;
  o.t_label = o.chosen = o.key = -1;
  o.flags = 0;
  if (ps->n_kept <= 0) {
    out[i] = o;
    return;
  }
  const PV* eye = P.eye + i;
  const size_t es = static_cast<size_t>(P.n);
  const int ne = P.n_eye[i];
  int tp = 0;
  for (int k = 1; k < ne; ++k) {
    const int f = eye[k * es].flag;
    if (f == kDiffuse) {
      tp = k + 1;
      break;
    }
    if (f != kSpecular) break;
  }
  if (tp < 2) {
    out[i] = o;
    return;
  }
  o.flags |= 1;
  const int idx = P.row0 * P.width + i;
  Rng prox = make_rng(P.seed, PXG_KIND_REF, 0,
                      (uint64_t(2) << 32) + static_cast<uint64_t>(pass) * static_cast<uint64_t>(n_px_total) + idx);
  o.u_gate = prox.next_double();
  const PV& z = eye[(tp - 1) * es];
  const int t_label = classify_eye(P.M, z.p, -z.wi);
  const double* row = gamma_rows + t_label * kS;
  double z_norm = 0.0;
  for (int sl = 0; sl < kS; ++sl)
    if (label_start[sl + 1] > label_start[sl]) z_norm += row[sl];
  if (!(z_norm > 0.0)) {
    out[i] = o;
    return;
  }
  o.flags |= 4;
  const double uu = prox.next_double() * z_norm;
  int chosen = -1;
  double cdf = 0.0;
  for (int sl = 0; sl < kS; ++sl) {
    if (label_start[sl + 1] == label_start[sl]) continue;
    chosen = sl;
    cdf += row[sl];
    if (uu < cdf) break;
  }
  const double row_p = row[chosen] / z_norm;
  const int bsize = label_start[chosen + 1] - label_start[chosen];
  const int e = label_list[label_start[chosen] + static_cast<int>(prox.next_below(static_cast<uint32_t>(bsize)))];
  const IncHdr& h = inc[e];
  const int s_rep = h.n_prefix + h.u + 1;
  o.t_label = t_label;
  o.chosen = chosen;
  o.key = h.key;
  o.q_sel = row_p / static_cast<double>(bsize);
  if (s_rep + tp <= P.max_depth + 1) {
    o.flags |= 2;
    V3 c = proxy_connect(P.S, P.M, P.st, eye, es, tp, h, prefix + static_cast<size_t>(e) * kMaxLight, prox,
                         scratch + static_cast<size_t>(i) * kMaxLight);
    o.c[0] = c.x;
    o.c[1] = c.y;
    o.c[2] = c.z;
  }
  out[i] = o;
}

// Per 10x10 cell in the reference's scan order (proxy.cpp:761-817).
__global__ void k_gate(int n_cells, int grid_w, int row0, int rows, int width, int pass, double gate_high,
                       double gate_low, double gate_threshold, double light_walks, int proxy_on,
                       const PassState* ps, const double* bdpt, const ProxRec* prox, double* acc, double* val,
                       double* grid_total, double* grid_proxy, GammaRec* grec, int* pflags,
                       unsigned long long* diag_attempt, unsigned long long* diag_accept, int* diag_touched) {
  const int cell = blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= n_cells) return;
  const int cx = cell % grid_w, cy = cell / grid_w;
  const double kappa = ps->kappa;
  const int y_end = min(rows, cy * 10 + 10);
  const int x_end = min(width, cx * 10 + 10);
  double gt = grid_total[cell], gp = grid_proxy[cell];
  for (int y = cy * 10; y < y_end; ++y) {
    for (int x = cx * 10; x < x_end; ++x) {
      const int i = y * width + x;
      V3 v = v3(bdpt[3 * i], bdpt[3 * i + 1], bdpt[3 * i + 2]);
      int fl = 0;
      GammaRec gr;
      gr.bin = -1;
      gr.value = 0.0;
      gr.pad = 0;
      if (proxy_on) {
        const ProxRec& o = prox[i];
        fl = o.flags & 1;
        if (o.flags & 1) {
          double gate = gate_high;
          if (pass > 0) {
            double share = gt > 0.0 ? gp / gt : 0.0;
            gate = share > gate_threshold ? gate_high : gate_low;
          }
          if (gate > 0.0 && o.u_gate < gate && (o.flags & 4)) {
            fl |= 4;
            if (o.flags & 2) {
              fl |= 2;
              atomicAdd(&diag_attempt[o.key], 1ull);
              diag_touched[o.key] = 1;
              V3 c = v3(o.c[0], o.c[1], o.c[2]);
              if (!near_zero(c)) {
                fl |= 8;
                atomicAdd(&diag_accept[o.key], 1ull);
                V3 contrib = c / (light_walks * kappa * gate * o.q_sel);
                v += contrib;
                gr.bin = o.t_label * kS + o.chosen;
                gr.value = luminance(c) / o.q_sel;
                gp += luminance(contrib);
              }
            }
          }
        }
      }
      acc[3 * i] += v.x;
      acc[3 * i + 1] += v.y;
      acc[3 * i + 2] += v.z;
      val[3 * i] = v.x;
      val[3 * i + 1] = v.y;
      val[3 * i + 2] = v.z;
      gt += luminance(v);
      grec[i] = gr;
      pflags[i] = fl;
    }
  }
  grid_total[cell] = gt;
  grid_proxy[cell] = gp;
}

// ------------------------------------------------------------------ test kernels
__global__ void k_intersect(SceneView S, int n, const double* rays, const double* tmax, int* prim, double* t) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* r = rays + 6 * static_cast<size_t>(i);
  Hit h;
  double tm = tmax ? tmax[i] : 1e30;
  if (intersect(S, v3(r[0], r[1], r[2]), v3(r[3], r[4], r[5]), h, tm)) {
    prim[i] = h.prim;
    t[i] = h.t;
  } else {
    prim[i] = -1;
    t[i] = 0.0;
  }
}

__global__ void k_occluded(SceneView S, int n, const double* segs, int* occ) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* s = segs + 6 * static_cast<size_t>(i);
  occ[i] = occluded(S, v3(s[0], s[1], s[2]), v3(s[3], s[4], s[5])) ? 1 : 0;
}

__global__ void k_rng(uint64_t seed, unsigned kind, unsigned sub, uint64_t stream, int n, unsigned* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  PxgRng r = pxg_rng_make(seed, kind, sub, stream);
  for (int i = 0; i < n; ++i) out[i] = pxg_next_u32(&r);
}

inline int blocks(long long n, int t) { return static_cast<int>((n + t - 1) / t); }

}  // namespace

// ------------------------------------------------------------------ context
struct pxg_ctx {
  std::string err;
  int device = 0;
  cudaStream_t stream = nullptr;
  SceneHost host;
  pxg_params P{};
  pxg_shard shard{};
  uint64_t seed = 0;
  int width = 0, height = 0, max_depth = 0, n = 0, n_px_total = 0, row0 = 0, rows = 0;
  int light_walks = 0;
  int grid_w = 0, grid_h = 0, n_cells = 0;
  bool proxy_on = false;
  int passes_done = 0;
  std::vector<void*> allocs;

  SceneView S{};
  Mapper M{};
  // stage 2
  PV* d_eye = nullptr;
  PV* d_light = nullptr;
  int *d_neye = nullptr, *d_nlight = nullptr;
  unsigned* d_ctr = nullptr;
  double *d_bdpt = nullptr, *d_val = nullptr, *d_acc = nullptr;
  ProxRec* d_prox = nullptr;
  PV* d_scratch = nullptr;
  double *d_grid_total = nullptr, *d_grid_proxy = nullptr;
  GammaRec* d_grec = nullptr;
  int* d_pflags = nullptr;
  int *d_eye_prims = nullptr, *d_light_prims = nullptr;
  // stats
  double *d_max_ratio = nullptr, *d_sum_est = nullptr, *d_sum_sq = nullptr;
  long long *d_ratio_cnt = nullptr, *d_est_cnt = nullptr;
  int* d_touched = nullptr;
  // gamma (host-authoritative rows, device copy)
  std::vector<double> gamma_rows, gamma_accum;
  bool gamma_learning = true;
  int gamma_iter = 0;
  double* d_gamma = nullptr;
  // pool
  int cand_cap = 0;
  unsigned long long *d_ckey = nullptr, *d_ckey_alt = nullptr;
  unsigned *d_cval = nullptr, *d_cval_alt = nullptr;
  int* d_ccount = nullptr;
  void* d_sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  unsigned* d_sel = nullptr;
  IncHdr* d_inc = nullptr;
  PV* d_inc_prefix = nullptr;
  double* d_probe = nullptr;
  int* d_probe_ok = nullptr;
  double* d_bound = nullptr;
  double* d_run_est = nullptr;
  long long* d_run_cost = nullptr;
  int* d_run_trunc = nullptr;
  RecipFrame* d_frames = nullptr;
  RunState* d_rstate = nullptr;
  double* d_rg = nullptr;
  long long* d_rn = nullptr;
  int* d_re = nullptr;
  int* d_ract[2] = {nullptr, nullptr};
  int* d_rnact = nullptr;
  int recip_rounds = 0;
  int *d_kept = nullptr, *d_label_start = nullptr, *d_label_list = nullptr;
  PassState* d_ps = nullptr;
  int* d_err = nullptr;
  // diagnostics
  long long* d_diag = nullptr;  // [4000*5]: cols 2..4 written by k_pool_finish
  unsigned long long *d_diag_attempt = nullptr, *d_diag_accept = nullptr;
  int* d_diag_touched = nullptr;
  long long pool_raw_total = 0;
  // last pass pool (host copy for dumps)
  int last_n_ent = 0;
  long long last_raw = 0;
  // wavefront queues and buffers
  RayQueue qA{}, qB{}, qS{};
  ConnBuf conn{};
  double *d_ebeta = nullptr, *d_epdf = nullptr, *d_lbeta = nullptr, *d_lpdf = nullptr;
  void* d_scan_tmp = nullptr;
  size_t scan_tmp_bytes = 0;
  int max_slots = 0;
  PV* d_wpool = nullptr;
  int* d_wnv = nullptr;
  unsigned* d_wctr = nullptr;
  double *d_wbeta = nullptr, *d_wpdf = nullptr;
  int n_walks = 0;
  // timing
  cudaEvent_t ev[8];
  cudaEvent_t ev_call[2];
  double stage_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long launches = 0;

  template <typename T>
  T* alloc(size_t n_) {
    T* p = dalloc<T>(n_);
    allocs.push_back(p);
    return p;
  }
  template <typename T>
  T* upload(const std::vector<T>& v) {
    T* p = alloc<T>(v.size());
    if (!v.empty()) CK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return p;
  }
  template <typename T>
  T* zeros(size_t n_) {
    T* p = alloc<T>(n_);
    CK(cudaMemset(p, 0, std::max<size_t>(n_, 1) * sizeof(T)));
    return p;
  }
  ~pxg_ctx() {
    for (void* p : allocs) cudaFree(p);
    if (d_sort_tmp) cudaFree(d_sort_tmp);
    if (d_scan_tmp) cudaFree(d_scan_tmp);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

void check_err(pxg_ctx* c) {
  int e = 0;
  CK(cudaMemcpyAsync(&e, c->d_err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (e) {
    const char* what = e == kErrIntegrand ? "reciprocal: integrand must be finite and non-negative"
                       : e == kErrSupport ? "reciprocal: support pdf must be finite and positive"
                       : e == kErrSplit   ? "stochastic_split: bad ratio"
                                          : "update_ratio: ratio must be finite and non-negative";
    throw RuntimeErr{what};
  }
}

void gamma_end_iteration(pxg_ctx* c) {
  // GammaMatrix::end_iteration (proj/src/subspace.cpp:164-182)
  if (!c->gamma_learning) return;
  const double eps = 1e-3 / kS;
  for (int t = 0; t < kT; ++t) {
    double* row = c->gamma_rows.data() + t * kS;
    const double* acc = c->gamma_accum.data() + t * kS;
    double total = 0.0;
    for (int s = 0; s < kS; ++s) total += acc[s];
    if (total <= 0.0) {
      for (int s = 0; s < kS; ++s) row[s] = 1.0 / kS;
      continue;
    }
    const double keep = 1.0 - eps * kS;
    for (int s = 0; s < kS; ++s) row[s] = keep * (acc[s] / total) + eps;
  }
  ++c->gamma_iter;
  if (c->gamma_iter >= c->P.freeze_iteration) c->gamma_learning = false;
  CK(cudaMemcpyAsync(c->d_gamma, c->gamma_rows.data(), sizeof(double) * kT * kS, cudaMemcpyHostToDevice,
                     c->stream));
}

// PXG_PROFILE=1: synchronise and print host-side stage timestamps (debugging aid).
struct HostProbe {
  pxg_ctx* c;
  bool on;
  std::chrono::steady_clock::time_point t0;
  explicit HostProbe(pxg_ctx* c_) : c(c_), on(std::getenv("PXG_PROFILE") != nullptr) {
    t0 = std::chrono::steady_clock::now();
  }
  void mark(const char* what);
};

RayQueue make_queue(pxg_ctx* c, size_t cap) {
  RayQueue q;
  q.ray = c->alloc<double4>(2 * cap);
  q.path = c->alloc<int>(cap);
  q.hit_prim = c->alloc<int>(cap);
  q.hit_t = c->alloc<double>(cap);
  q.count = c->zeros<int>(1);
  q.cap = static_cast<int>(cap);
  return q;
}

// Sub-path wavefront: start kernel, then one (closest-hit, shade) pair per bounce.
void trace_paths(pxg_ctx* c, const PathSet& P) {
  RayQueue in = c->qA, out = c->qB;
  CK(cudaMemsetAsync(in.count, 0, sizeof(int), c->stream));
  const int T = 128;
  if (P.eye)
    k_eye_start<<<blocks(P.n, T), T, 0, c->stream>>>(c->S, P, in, c->row0);
  else
    k_light_start<<<blocks(P.n, T), T, 0, c->stream>>>(c->S, P, in);
  ++c->launches;
  for (int b = 0; b + 1 < P.max_vertices; ++b) {
    k_closest<<<blocks(P.n, T), T, 0, c->stream>>>(c->S, in);
    CK(cudaMemsetAsync(out.count, 0, sizeof(int), c->stream));
    k_shade<<<blocks(P.n, T), T, 0, c->stream>>>(c->S, P, in, out);
    c->launches += 2;
    std::swap(in, out);
  }
}

// Standard strategies of every pixel (weighted_bdpt_value, proxy.cpp:621-643).
void connections(pxg_ctx* c, bool use_stats) {
  const int n = c->n, D = c->max_depth, T = 128;
  ConnBuf& C = c->conn;
  k_conn_count<<<blocks(n, T), T, 0, c->stream>>>(c->d_neye, c->d_nlight, n, D, C.count);
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, C.count, C.offset, n + 1, c->stream);
  if (need > c->scan_tmp_bytes) {
    if (c->d_scan_tmp) cudaFree(c->d_scan_tmp);
    CK(cudaMalloc(&c->d_scan_tmp, need));
    c->scan_tmp_bytes = need;
  }
  CK(cub::DeviceScan::ExclusiveSum(c->d_scan_tmp, c->scan_tmp_bytes, C.count, C.offset, n + 1, c->stream));
  k_conn_enum<<<blocks(n, T), T, 0, c->stream>>>(c->d_neye, c->d_nlight, n, D, C);
  CK(cudaMemsetAsync(c->qS.count, 0, sizeof(int), c->stream));
  const long long slots = static_cast<long long>(n) * c->max_slots;
  k_conn_eval<<<blocks(slots, T), T, 0, c->stream>>>(c->S, c->d_eye, c->d_light, n, C, c->qS);
  k_anyhit<<<blocks(slots, T), T, 0, c->stream>>>(c->S, c->qS);
  k_conn_visibility<<<blocks(slots, T), T, 0, c->stream>>>(c->qS, C);
  k_conn_mis<<<blocks(slots, T), T, 0, c->stream>>>(
      c->S, c->M, StatsView{c->d_max_ratio, c->d_sum_est, c->d_sum_sq, c->d_est_cnt}, use_stats ? 1 : 0, c->d_eye,
      c->d_light, n, C);
  k_conn_sum<<<blocks(n, T), T, 0, c->stream>>>(n, C, c->d_bdpt);
  c->launches += 9;
}

void HostProbe::mark(const char* what) {
  if (!on) return;
  cudaStreamSynchronize(c->stream);
  auto t = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[pxg] %-14s %9.3f ms\n", what, std::chrono::duration<double, std::milli>(t - t0).count());
  t0 = t;
}

// The reciprocal runs of one pass: rounds of (parallel node evaluation, DFS resume) with
// the evaluated prefix doubling per round, until every run has finished.
template <typename Eval>
int recip_rounds(cudaStream_t stream, int runs, int* act[2], int* nact, Eval&& eval_and_dfs) {
  int cur = 0, chunk = 16, rounds = 0;
  for (;;) {
    int count = 0;
    CK(cudaMemcpyAsync(&count, nact + cur, sizeof(int), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    if (count == 0) break;
    CK(cudaMemsetAsync(nact + (1 - cur), 0, sizeof(int), stream));
    eval_and_dfs(cur, count, chunk);
    cur = 1 - cur;
    chunk = std::min(chunk * 2, 4096);
    ++rounds;
  }
  (void)runs;
  return rounds;
}

void stage1(pxg_ctx* c, int pass) {
  HostProbe hp(c);
  const int walks = c->shard.walk_end - c->shard.walk_begin;
  CK(cudaMemsetAsync(c->d_ccount, 0, sizeof(int), c->stream));
  if (walks > 0) {
    CK(cudaMemsetAsync(c->d_wctr, 0, sizeof(unsigned) * walks, c->stream));
    PathSet W{c->d_wpool, c->d_wnv, c->d_wctr, c->d_wbeta, c->d_wpdf, c->seed,
              (static_cast<uint64_t>(pass) << 32) + static_cast<uint64_t>(c->shard.walk_begin),
              PXG_KIND_POOL_WALK, walks, c->max_depth - 1, 0};
    trace_paths(c, W);
    hp.mark("walks");
    k_pool_keys<<<blocks(walks, 128), 128, 0, c->stream>>>(c->d_wpool, c->d_wnv, walks, c->seed, pass,
                                                           c->shard.walk_begin, c->d_ckey, c->d_cval, c->d_ccount,
                                                           c->cand_cap);
    ++c->launches;
  }
  int raw = 0;
  CK(cudaMemcpyAsync(&raw, c->d_ccount, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (raw > c->cand_cap) throw RuntimeErr{"pool candidate buffer overflow"};
  const int budget = c->P.pool_budget;
  int n_ent = std::min(raw, std::max(budget, 0));
  std::vector<unsigned> sel(n_ent);
  if (n_ent > 0) {
    const unsigned* src = c->d_cval;
    if (raw > budget) {
      size_t need = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, need, c->d_ckey, c->d_ckey_alt, c->d_cval, c->d_cval_alt, raw, 0, 64,
                                      c->stream);
      if (need > c->sort_tmp_bytes) {
        if (c->d_sort_tmp) cudaFree(c->d_sort_tmp);
        CK(cudaMalloc(&c->d_sort_tmp, need));
        c->sort_tmp_bytes = need;
      }
      CK(cub::DeviceRadixSort::SortPairs(c->d_sort_tmp, c->sort_tmp_bytes, c->d_ckey, c->d_ckey_alt, c->d_cval,
                                         c->d_cval_alt, raw, 0, 64, c->stream));
      ++c->launches;
      src = c->d_cval_alt;
    }
    CK(cudaMemcpyAsync(sel.data(), src, sizeof(unsigned) * n_ent, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    // keys tie only with probability ~2^-64; ties are broken by (walk, end) like the oracle
    std::sort(sel.begin(), sel.end());  // (walk << 5 | end) order == (walk, end) order
    CK(cudaMemcpyAsync(c->d_sel, sel.data(), sizeof(unsigned) * n_ent, cudaMemcpyHostToDevice, c->stream));
  }
  hp.mark("select");
  c->pool_raw_total += raw;
  c->last_raw = raw;
  c->last_n_ent = n_ent;
  PassState ps_host;
  ps_host.kappa = raw > 0 ? std::min(1.0, static_cast<double>(budget) / static_cast<double>(raw)) : 1.0;
  CK(cudaMemcpyAsync(&c->d_ps->kappa, &ps_host.kappa, sizeof(double), cudaMemcpyHostToDevice, c->stream));
  const int R = c->P.recip_repeats;
  bool ran_recip = false;
  if (n_ent > 0) {
    k_pool_entries<<<blocks(n_ent, 64), 64, 0, c->stream>>>(c->S, c->M, c->seed, pass, n_ent, c->d_sel, c->d_wpool,
                                                           walks, c->shard.walk_begin, c->d_inc, c->d_inc_prefix,
                                                           c->d_probe, c->d_probe_ok, R);
    k_pool_bounds<<<1, 1, 0, c->stream>>>(n_ent, c->d_inc, c->d_probe, c->d_probe_ok, c->d_max_ratio,
                                          c->d_ratio_cnt, c->d_touched, c->d_bound, c->d_err);
    c->launches += 2;
    hp.mark("entries+bounds");
    if (R >= 1) {
      CK(cudaEventRecord(c->ev[2], c->stream));
      const int runs = n_ent * R;
      const long long cap = c->P.recursion_cap;
      CK(cudaMemsetAsync(c->d_rnact, 0, 2 * sizeof(int), c->stream));
      k_recip_init<<<blocks(runs, 128), 128, 0, c->stream>>>(runs, R, c->d_inc, c->d_bound, c->d_rstate,
                                                            c->d_ract[0], c->d_rnact, c->d_run_est, c->d_run_cost,
                                                            c->d_run_trunc);
      c->recip_rounds = recip_rounds(c->stream, runs, c->d_ract, c->d_rnact, [&](int cur, int count, int chunk) {
        k_recip_eval<<<blocks(static_cast<long long>(count) * chunk, 64), 64, 0, c->stream>>>(
            c->S, c->seed, pass, R, cap, c->d_inc, c->d_inc_prefix, c->d_bound, c->d_ract[cur], c->d_rnact + cur,
            chunk, c->d_rstate, c->d_rg, c->d_rn, c->d_re);
        k_recip_dfs<<<blocks(count, 64), 64, 0, c->stream>>>(
            R, cap, c->d_bound, 0.0, c->d_ract[cur], c->d_rnact + cur, chunk, c->d_rstate, c->d_rg, c->d_rn, c->d_re,
            c->d_frames, c->d_run_est, c->d_run_cost, c->d_run_trunc, c->d_ract[1 - cur], c->d_rnact + (1 - cur),
            c->d_err);
        c->launches += 2;
      });
      CK(cudaEventRecord(c->ev[3], c->stream));
      ++c->launches;
      ran_recip = true;
      hp.mark("recip");
    }
  }
  if (!ran_recip) {
    CK(cudaEventRecord(c->ev[2], c->stream));
    CK(cudaEventRecord(c->ev[3], c->stream));
  }
  k_pool_finish<<<1, 1, 0, c->stream>>>(n_ent, R, c->d_inc, c->d_bound, c->d_run_est, c->d_run_trunc, c->d_sum_est,
                                        c->d_sum_sq, c->d_est_cnt, c->d_touched, c->d_diag, c->d_diag_touched,
                                        c->d_kept, c->d_label_start, c->d_label_list, c->d_ps);
  ++c->launches;
  hp.mark("finish");
}

void render_pass(pxg_ctx* c, bool record_prims) {
  const int pass = c->passes_done;
  CK(cudaEventRecord(c->ev[0], c->stream));
  if (c->proxy_on) {
    stage1(c, pass);
  } else {
    CK(cudaMemsetAsync(&c->d_ps->n_kept, 0, sizeof(int), c->stream));
    CK(cudaEventRecord(c->ev[2], c->stream));
    CK(cudaEventRecord(c->ev[3], c->stream));
  }
  CK(cudaEventRecord(c->ev[1], c->stream));
  Stage2 P;
  P.S = c->S;
  P.M = c->M;
  P.st = StatsView{c->d_max_ratio, c->d_sum_est, c->d_sum_sq, c->d_est_cnt};
  P.eye = c->d_eye;
  P.light = c->d_light;
  P.n_eye = c->d_neye;
  P.n_light = c->d_nlight;
  P.ctr = c->d_ctr;
  P.bdpt = c->d_bdpt;
  P.eye_prims = c->d_eye_prims;
  P.light_prims = c->d_light_prims;
  P.n = c->n;
  P.row0 = c->row0;
  P.width = c->width;
  P.height = c->height;
  P.max_depth = c->max_depth;
  P.seed = c->seed;
  P.record_prims = record_prims ? 1 : 0;
  const int T = 128;
  HostProbe hp(c);
  {
    PathSet E{c->d_eye, c->d_neye, c->d_ctr, c->d_ebeta, c->d_epdf, c->seed,
              static_cast<uint64_t>(c->row0) * c->width, PXG_KIND_REF, c->n, c->max_depth + 1, 1};
    trace_paths(c, E);
    PathSet L{c->d_light, c->d_nlight, c->d_ctr, c->d_lbeta, c->d_lpdf, c->seed,
              static_cast<uint64_t>(c->row0) * c->width, PXG_KIND_REF, c->n, c->max_depth - 1, 0};
    trace_paths(c, L);
    if (record_prims) {
      k_record_prims<<<blocks(c->n, T), T, 0, c->stream>>>(c->d_eye, c->d_neye, c->d_light, c->d_nlight, c->n,
                                                          c->max_depth, c->d_eye_prims, c->d_light_prims);
      ++c->launches;
    }
  }
  hp.mark("trace");
  CK(cudaEventRecord(c->ev[4], c->stream));
  connections(c, c->proxy_on);
  CK(cudaEventRecord(c->ev[5], c->stream));
  hp.mark("connect");
  if (c->proxy_on) {
    k_proxy<<<blocks(c->n, T), T, 0, c->stream>>>(P, pass, c->n_px_total, c->d_inc, c->d_inc_prefix,
                                                  c->d_label_start, c->d_label_list, c->d_gamma, c->d_ps, c->d_prox,
                                                  c->d_scratch);
    ++c->launches;
  }
  CK(cudaEventRecord(c->ev[6], c->stream));
  k_gate<<<blocks(c->n_cells, 64), 64, 0, c->stream>>>(
      c->n_cells, c->grid_w, c->row0, c->rows, c->width, pass, c->P.gate_high, c->P.gate_low, c->P.gate_threshold,
      static_cast<double>(c->light_walks), c->proxy_on ? 1 : 0, c->d_ps, c->d_bdpt, c->d_prox, c->d_acc, c->d_val,
      c->d_grid_total, c->d_grid_proxy, c->d_grec, c->d_pflags, c->d_diag_attempt, c->d_diag_accept,
      c->d_diag_touched);
  CK(cudaEventRecord(c->ev[7], c->stream));
  ++c->launches;
  hp.mark("proxy+gate");
  if (c->proxy_on) {
    check_err(c);
    if (c->gamma_learning) {
      // GammaMatrix::record_contribution in pixel scan order (proxy.cpp:807-808)
      std::vector<GammaRec> gr(c->n);
      CK(cudaMemcpyAsync(gr.data(), c->d_grec, sizeof(GammaRec) * c->n, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      for (int i = 0; i < c->n; ++i) {
        if (gr[i].bin < 0) continue;
        const double v = gr[i].value;
        if (!std::isfinite(v) || v < 0.0) continue;
        c->gamma_accum[gr[i].bin] += v;
      }
    }
    gamma_end_iteration(c);
  }
  ++c->passes_done;
}

void accumulate_timing(pxg_ctx* c) {
  // ev0 pass start, ev2/ev3 around the reciprocal runs (inside stage 1), ev1 stage-1 end,
  // ev4 trace end, ev5 connect end, ev6 proxy end, ev7 gate end.
  auto el = [&](int a, int b) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]) != cudaSuccess) {
      cudaGetLastError();
      ms = 0.f;
    }
    return static_cast<double>(ms);
  };
  c->stage_ms[0] += el(0, 1);
  c->stage_ms[1] += el(2, 3);
  c->stage_ms[2] += el(1, 4);
  c->stage_ms[3] += el(4, 5);
  c->stage_ms[4] += el(5, 6);
  c->stage_ms[5] += el(6, 7);
}

int fail(pxg_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  g_global_err = msg;
  return code;
}

template <typename F>
int guarded(pxg_ctx* c, F&& f) {
  try {
    if (c) CK(cudaSetDevice(c->device));
    f();
    return PXG_OK;
  } catch (const CudaErr& e) {
    return fail(c, PXG_E_CUDA, e.msg);
  } catch (const InvalidErr& e) {
    return fail(c, PXG_E_INVALID, e.msg);
  } catch (const RuntimeErr& e) {
    return fail(c, PXG_E_RUNTIME, e.msg);
  } catch (const std::exception& e) {
    return fail(c, PXG_E_INVALID, e.what());
  }
}

}  // namespace

// ------------------------------------------------------------------ C ABI
extern "C" {

void pxg_default_params(pxg_params* p) {
  p->enabled = 1;
  p->pool_budget = 400;
  p->recip_repeats = 5;
  p->freeze_iteration = 40;
  p->recursion_cap = 10000;
  p->pretrace_paths = 20000;
  p->light_walks = 0;
  p->gate_high = 1.0;
  p->gate_low = 0.2;
  p->gate_threshold = 0.05;
}

int pxg_abi_version(void) { return PXG_ABI_VERSION; }

int pxg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

const char* pxg_last_error(const pxg_ctx* ctx) { return ctx ? ctx->err.c_str() : g_global_err.c_str(); }

void pxg_destroy(pxg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  delete ctx;
}

int pxg_create(const pxg_scene_desc* sd, const pxg_params* params, uint64_t seed, int device,
               const pxg_shard* shard, pxg_ctx** out) {
  if (!sd || !out) return fail(nullptr, PXG_E_INVALID, "pxg_create: null argument");
  *out = nullptr;
  if (pxg_device_count() <= 0) return fail(nullptr, PXG_E_NODEVICE, "pxg_create: no CUDA device");
  auto* c = new pxg_ctx();
  c->device = device;
  int rc = guarded(c, [&]() {
    if (sd->max_depth < 1) throw InvalidErr{"scene: max_depth must be at least 1"};
    if (sd->max_depth + 1 > kMaxPath - 2 || sd->max_depth - 1 > kMaxLight - 1)
      throw InvalidErr{"pxg: max_depth above 16 is not supported"};
    if (params) c->P = *params; else pxg_default_params(&c->P);
    c->seed = seed;
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    for (auto& e : c->ev) CK(cudaEventCreate(&e));
    for (auto& e : c->ev_call) CK(cudaEventCreate(&e));
    finalize_scene(*sd, c->host);
    SceneHost& h = c->host;
    c->width = sd->width;
    c->height = sd->height;
    c->max_depth = sd->max_depth;
    c->n_px_total = sd->width * sd->height;
    c->light_walks = c->P.light_walks > 0 ? c->P.light_walks : c->n_px_total;
    if (shard) {
      c->shard = *shard;
    } else {
      c->shard = pxg_shard{0, sd->height, 0, c->light_walks};
    }
    if (c->shard.row_begin < 0 || c->shard.row_end > sd->height || c->shard.row_begin >= c->shard.row_end ||
        (c->shard.row_begin % 10) != 0 || c->shard.walk_begin < 0 || c->shard.walk_end > c->light_walks ||
        c->shard.walk_begin > c->shard.walk_end)
      throw InvalidErr{"pxg_create: invalid shard"};
    c->row0 = c->shard.row_begin;
    c->rows = c->shard.row_end - c->shard.row_begin;
    c->n = c->rows * c->width;
    bool any_spec = false;
    std::vector<Material> mats(sd->n_materials);
    for (int m = 0; m < sd->n_materials; ++m) {
      const double* q = sd->materials + 7 * m;
      Material& M = mats[m];
      M.base_color = v3(q[0], q[1], q[2]);
      M.metallic = q[3];
      M.roughness = q[4];
      M.transmission = q[5];
      M.ior = q[6];
      M.specular = ((M.metallic >= 0.5 || M.transmission >= 0.5) && M.roughness < 0.2) ? 1 : 0;
      M.pad = 0;
      any_spec = any_spec || M.specular;
    }
    c->proxy_on = c->P.enabled != 0;
    (void)any_spec;
    // device scene
    SceneView& S = c->S;
    S.nodes = reinterpret_cast<const BvhNode*>(c->upload(h.nodes));
    S.recs = reinterpret_cast<const PrimRec*>(c->upload(h.recs));
    S.prim_mat = c->upload(h.prim_mat);
    S.prim_emitter = c->upload(h.prim_emitter);
    S.prim_geo = c->upload(h.prim_geo);
    S.prim_center = c->upload(h.prim_center);
    S.prim_shape = c->upload(h.prim_shape);
    S.prim_abc = c->upload(h.prim_abc);
    S.materials = c->upload(mats);
    S.emitter_prim = c->upload(std::vector<int>(sd->emitter_prim, sd->emitter_prim + sd->n_emitters));
    S.emitter_rad = c->upload(std::vector<double>(sd->emitter_radiance, sd->emitter_radiance + 3 * sd->n_emitters));
    S.emitter_cum = c->upload(h.emitter_cum);
    S.n_prims = sd->n_prims;
    S.n_emit = sd->n_emitters;
    S.n_nodes = static_cast<int>(h.nodes.size());
    S.n_mat = sd->n_materials;
    S.total_emitter_area = h.total_emitter_area;
    S.bbox_min = v3(h.bbox_min[0], h.bbox_min[1], h.bbox_min[2]);
    S.bbox_max = v3(h.bbox_max[0], h.bbox_max[1], h.bbox_max[2]);
    S.cam_pos = v3(h.cam[0], h.cam[1], h.cam[2]);
    S.cam_fwd = v3(h.cam[3], h.cam[4], h.cam[5]);
    S.cam_right = v3(h.cam[6], h.cam[7], h.cam[8]);
    S.cam_up = v3(h.cam[9], h.cam[10], h.cam[11]);
    S.tan_half = h.tan_half;
    S.aspect = h.aspect;
    S.width = sd->width;
    S.height = sd->height;
    S.max_depth = sd->max_depth;
    c->M.bmin = S.bbox_min;
    c->M.bmax = S.bbox_max;
    // stage-2 buffers
    const size_t n = c->n;
    c->d_eye = c->alloc<PV>(n * (c->max_depth + 1));
    c->d_light = c->alloc<PV>(n * std::max(c->max_depth - 1, 1));
    c->d_neye = c->zeros<int>(n);
    c->d_nlight = c->zeros<int>(n);
    c->d_ctr = c->zeros<unsigned>(n);
    c->d_bdpt = c->zeros<double>(3 * n);
    c->d_val = c->zeros<double>(3 * n);
    c->d_acc = c->zeros<double>(3 * n);
    c->d_prox = c->zeros<ProxRec>(n);
    c->d_scratch = c->alloc<PV>(n * kMaxLight);
    c->d_ebeta = c->zeros<double>(3 * n);
    c->d_epdf = c->zeros<double>(n);
    c->d_lbeta = c->zeros<double>(3 * n);
    c->d_lpdf = c->zeros<double>(n);
    {
      int ms = 0;
      for (int t = 2; t <= c->max_depth + 1; ++t) ms += 1 + std::min(c->max_depth - 1, c->max_depth + 1 - t);
      c->max_slots = ms;
    }
    const size_t slots = n * static_cast<size_t>(c->max_slots);
    c->conn.count = c->zeros<int>(n + 1);
    c->conn.offset = c->zeros<int>(n + 1);
    c->conn.desc = c->alloc<int2>(slots);
    c->conn.value = c->alloc<double>(3 * slots);
    c->conn.state = c->zeros<int>(slots);
    c->conn.total = c->zeros<int>(1);
    c->qS = make_queue(c, slots);
    c->n_walks = c->shard.walk_end - c->shard.walk_begin;
    {
      const size_t qcap = std::max<size_t>(n, static_cast<size_t>(c->n_walks));
      c->qA = make_queue(c, qcap);
      c->qB = make_queue(c, qcap);
    }
    if (c->proxy_on && c->n_walks > 0) {
      const size_t w = c->n_walks;
      c->d_wpool = c->alloc<PV>(w * std::max(c->max_depth - 1, 1));
      c->d_wnv = c->zeros<int>(w);
      c->d_wctr = c->zeros<unsigned>(w);
      c->d_wbeta = c->zeros<double>(3 * w);
      c->d_wpdf = c->zeros<double>(w);
    }
    c->grid_w = (c->width + 9) / 10;
    c->grid_h = (c->rows + 9) / 10;
    c->n_cells = c->grid_w * c->grid_h;
    c->d_grid_total = c->zeros<double>(c->n_cells);
    c->d_grid_proxy = c->zeros<double>(c->n_cells);
    c->d_grec = c->zeros<GammaRec>(n);
    c->d_pflags = c->zeros<int>(n);
    c->d_eye_prims = c->zeros<int>(n * (c->max_depth + 1));
    c->d_light_prims = c->zeros<int>(n * std::max(c->max_depth - 1, 1));
    // stats
    c->d_max_ratio = c->zeros<double>(kBuckets);
    c->d_sum_est = c->zeros<double>(kBuckets);
    c->d_sum_sq = c->zeros<double>(kBuckets);
    c->d_ratio_cnt = c->zeros<long long>(kBuckets);
    c->d_est_cnt = c->zeros<long long>(kBuckets);
    c->d_touched = c->zeros<int>(kBuckets);
    c->gamma_rows.assign(kT * kS, 1.0 / kS);
    c->gamma_accum.assign(kT * kS, 0.0);
    c->gamma_learning = true;
    c->gamma_iter = 0;
    c->d_gamma = c->upload(c->gamma_rows);
    // pool
    const int walks = c->shard.walk_end - c->shard.walk_begin;
    c->cand_cap = std::max(1, walks) * std::max(1, c->max_depth - 2);
    c->d_ckey = c->alloc<unsigned long long>(c->cand_cap);
    c->d_ckey_alt = c->alloc<unsigned long long>(c->cand_cap);
    c->d_cval = c->alloc<unsigned>(c->cand_cap);
    c->d_cval_alt = c->alloc<unsigned>(c->cand_cap);
    c->d_ccount = c->zeros<int>(1);
    {
      // sort scratch sized once for the largest possible candidate count (no per-pass realloc)
      size_t need = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, need, c->d_ckey, c->d_ckey_alt, c->d_cval, c->d_cval_alt,
                                      c->cand_cap, 0, 64, c->stream);
      CK(cudaMalloc(&c->d_sort_tmp, need));
      c->sort_tmp_bytes = need;
    }
    const int B = std::max(c->P.pool_budget, 1);
    const int R = std::max(c->P.recip_repeats, 1);
    c->d_sel = c->alloc<unsigned>(B);
    c->d_inc = c->zeros<IncHdr>(B);
    c->d_inc_prefix = c->alloc<PV>(static_cast<size_t>(B) * kMaxLight);
    c->d_probe = c->zeros<double>(4 * B);
    c->d_probe_ok = c->zeros<int>(4 * B);
    c->d_bound = c->zeros<double>(B);
    c->d_run_est = c->zeros<double>(static_cast<size_t>(B) * R);
    c->d_run_cost = c->zeros<long long>(static_cast<size_t>(B) * R);
    c->d_run_trunc = c->zeros<int>(static_cast<size_t>(B) * R);
    if (c->P.recursion_cap > (1 << 20) || c->P.recip_repeats > 255)
      throw InvalidErr{"pxg: recursion_cap above 2^20 or recip_repeats above 255 is not supported"};
    if (c->proxy_on && c->P.recursion_cap > 0) {
      const size_t rc = static_cast<size_t>(B) * R * static_cast<size_t>(c->P.recursion_cap);
      c->d_frames = c->alloc<RecipFrame>(rc);
      c->d_rg = c->alloc<double>(rc);
      c->d_rn = c->alloc<long long>(rc);
      c->d_re = c->alloc<int>(rc);
    }
    c->d_rstate = c->alloc<RunState>(static_cast<size_t>(B) * R);
    c->d_ract[0] = c->alloc<int>(static_cast<size_t>(B) * R);
    c->d_ract[1] = c->alloc<int>(static_cast<size_t>(B) * R);
    c->d_rnact = c->zeros<int>(2);
    c->d_kept = c->zeros<int>(B);
    c->d_label_start = c->zeros<int>(kS + 1);
    c->d_label_list = c->zeros<int>(B);
    c->d_ps = c->zeros<PassState>(1);
    c->d_err = c->zeros<int>(1);
    c->d_diag = c->zeros<long long>(kBuckets * 5);
    c->d_diag_attempt = c->zeros<unsigned long long>(kBuckets);
    c->d_diag_accept = c->zeros<unsigned long long>(kBuckets);
    c->d_diag_touched = c->zeros<int>(kBuckets);
    if (c->proxy_on) {
      const int np = std::max(c->P.pretrace_paths, 1000);
      k_pretrace<<<blocks(np, 64), 64, 0, c->stream>>>(c->S, c->M, c->seed, np, c->d_max_ratio, c->d_ratio_cnt,
                                                       c->d_touched, c->d_err);
      CK(cudaGetLastError());
      check_err(c);
    }
    CK(cudaDeviceSynchronize());
  });
  if (rc != PXG_OK) {
    g_global_err = c->err;
    delete c;
    return rc;
  }
  *out = c;
  return PXG_OK;
}

int pxg_render_passes(pxg_ctx* c, int npass) {
  if (!c) return fail(nullptr, PXG_E_INVALID, "null context");
  return guarded(c, [&]() {
    for (int k = 0; k < 8; ++k) c->stage_ms[k] = 0.0;
    c->launches = 0;
    CK(cudaEventRecord(c->ev_call[0], c->stream));
    for (int p = 0; p < npass; ++p) {
      render_pass(c, false);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(c->stream));
      accumulate_timing(c);
    }
    CK(cudaEventRecord(c->ev_call[1], c->stream));
    CK(cudaEventSynchronize(c->ev_call[1]));
    float total = 0.f;
    CK(cudaEventElapsedTime(&total, c->ev_call[0], c->ev_call[1]));
    c->stage_ms[6] = total;
    check_err(c);
  });
}

int pxg_render_pass(pxg_ctx* c) { return pxg_render_passes(c, 1); }

int pxg_render_pass_traced(pxg_ctx* c) {
  if (!c) return fail(nullptr, PXG_E_INVALID, "null context");
  return guarded(c, [&]() {
    render_pass(c, true);
    CK(cudaGetLastError());
    check_err(c);
  });
}

int pxg_synchronize(pxg_ctx* c) {
  return guarded(c, [&]() { CK(cudaStreamSynchronize(c->stream)); });
}

int pxg_read_accum(pxg_ctx* c, double* rgb, int* passes) {
  return guarded(c, [&]() {
    CK(cudaMemcpyAsync(rgb, c->d_acc, sizeof(double) * 3 * c->n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (passes) *passes = c->passes_done;
  });
}

int pxg_read_mean(pxg_ctx* c, double* rgb, int* passes) {
  return guarded(c, [&]() {
    CK(cudaMemcpyAsync(rgb, c->d_acc, sizeof(double) * 3 * c->n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const double d = static_cast<double>(c->passes_done > 0 ? c->passes_done : 1);
    for (size_t i = 0; i < 3 * static_cast<size_t>(c->n); ++i) rgb[i] = rgb[i] * (1.0 / d);
    if (passes) *passes = c->passes_done;
  });
}

int pxg_read_diag(pxg_ctx* c, long long* rows, int* touched, long long* pool) {
  return guarded(c, [&]() {
    std::vector<long long> d(kBuckets * 5);
    std::vector<unsigned long long> at(kBuckets), ac(kBuckets);
    std::vector<int> tc(kBuckets);
    PassState ps;
    CK(cudaMemcpy(d.data(), c->d_diag, sizeof(long long) * kBuckets * 5, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(at.data(), c->d_diag_attempt, sizeof(unsigned long long) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ac.data(), c->d_diag_accept, sizeof(unsigned long long) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(tc.data(), c->d_diag_touched, sizeof(int) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&ps, c->d_ps, sizeof(PassState), cudaMemcpyDeviceToHost));
    for (int k = 0; k < kBuckets; ++k) {
      d[k * 5 + 0] = static_cast<long long>(at[k]);
      d[k * 5 + 1] = static_cast<long long>(ac[k]);
    }
    if (rows) std::memcpy(rows, d.data(), sizeof(long long) * kBuckets * 5);
    if (touched) std::memcpy(touched, tc.data(), sizeof(int) * kBuckets);
    if (pool) {
      pool[0] = c->pool_raw_total;
      pool[1] = ps.pool_kept_total;
    }
  });
}

int pxg_read_stats(pxg_ctx* c, double* stats3, long long* counts2, double* gamma_rows) {
  return guarded(c, [&]() {
    std::vector<double> a(kBuckets), b(kBuckets), s(kBuckets);
    std::vector<long long> rc(kBuckets), ec(kBuckets);
    CK(cudaMemcpy(a.data(), c->d_max_ratio, sizeof(double) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), c->d_sum_est, sizeof(double) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(s.data(), c->d_sum_sq, sizeof(double) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(rc.data(), c->d_ratio_cnt, sizeof(long long) * kBuckets, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ec.data(), c->d_est_cnt, sizeof(long long) * kBuckets, cudaMemcpyDeviceToHost));
    for (int k = 0; k < kBuckets; ++k) {
      if (stats3) {
        stats3[3 * k] = a[k];
        stats3[3 * k + 1] = b[k];
        stats3[3 * k + 2] = s[k];
      }
      if (counts2) {
        counts2[2 * k] = rc[k];
        counts2[2 * k + 1] = ec[k];
      }
    }
    if (gamma_rows) std::memcpy(gamma_rows, c->gamma_rows.data(), sizeof(double) * kT * kS);
  });
}

int pxg_dump_pass(pxg_ctx* c, double* val, double* bdpt, double* cc, int* flags) {
  return guarded(c, [&]() {
    const size_t n = c->n;
    if (val) CK(cudaMemcpy(val, c->d_val, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
    if (bdpt) CK(cudaMemcpy(bdpt, c->d_bdpt, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost));
    if (cc) {
      std::vector<ProxRec> pr(n);
      CK(cudaMemcpy(pr.data(), c->d_prox, sizeof(ProxRec) * n, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) cc[3 * i + k] = c->proxy_on ? pr[i].c[k] : 0.0;
    }
    if (flags) CK(cudaMemcpy(flags, c->d_pflags, sizeof(int) * n, cudaMemcpyDeviceToHost));
  });
}

int pxg_dump_prims(pxg_ctx* c, int* eye, int* light) {
  return guarded(c, [&]() {
    const size_t n = c->n;
    if (eye) CK(cudaMemcpy(eye, c->d_eye_prims, sizeof(int) * n * (c->max_depth + 1), cudaMemcpyDeviceToHost));
    if (light)
      CK(cudaMemcpy(light, c->d_light_prims, sizeof(int) * n * std::max(c->max_depth - 1, 1), cudaMemcpyDeviceToHost));
  });
}

int pxg_dump_pool(pxg_ctx* c, int cap, int* n_out, long long* raw, int* walk, int* end, int* key, double* inv_p,
                  double* inv_p_m2, double* bound) {
  return guarded(c, [&]() {
    PassState ps;
    CK(cudaMemcpy(&ps, c->d_ps, sizeof(PassState), cudaMemcpyDeviceToHost));
    const int n_ent = c->last_n_ent;
    std::vector<IncHdr> inc(n_ent);
    std::vector<int> kept(std::max(ps.n_kept, 0));
    std::vector<double> bd(n_ent);
    if (n_ent) {
      CK(cudaMemcpy(inc.data(), c->d_inc, sizeof(IncHdr) * n_ent, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(bd.data(), c->d_bound, sizeof(double) * n_ent, cudaMemcpyDeviceToHost));
    }
    if (ps.n_kept > 0) CK(cudaMemcpy(kept.data(), c->d_kept, sizeof(int) * ps.n_kept, cudaMemcpyDeviceToHost));
    const int m = std::min(cap, ps.n_kept);
    for (int i = 0; i < m; ++i) {
      const IncHdr& h = inc[kept[i]];
      if (walk) walk[i] = h.walk;
      if (end) end[i] = h.end;
      if (key) key[i] = h.key;
      if (inv_p) inv_p[i] = h.inverse_p;
      if (inv_p_m2) inv_p_m2[i] = h.inverse_p_m2;
      if (bound) bound[i] = bd[kept[i]];
    }
    if (n_out) *n_out = ps.n_kept;
    if (raw) *raw = c->last_raw;
  });
}

int pxg_intersect(pxg_ctx* c, int n, const double* rays, const double* tmax, int* prim, double* t) {
  return guarded(c, [&]() {
    if (n <= 0) return;
    double* dr = dupload(rays, static_cast<size_t>(n) * 6);
    double* dt = tmax ? dupload(tmax, n) : nullptr;
    int* dp = dalloc<int>(n);
    double* dtt = dalloc<double>(n);
    k_intersect<<<blocks(n, 128), 128, 0, c->stream>>>(c->S, n, dr, dt, dp, dtt);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(prim, dp, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(t, dtt, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(dr);
    if (dt) cudaFree(dt);
    cudaFree(dp);
    cudaFree(dtt);
  });
}

int pxg_occluded(pxg_ctx* c, int n, const double* segs, int* occ) {
  return guarded(c, [&]() {
    if (n <= 0) return;
    double* ds = dupload(segs, static_cast<size_t>(n) * 6);
    int* dout = dalloc<int>(n);
    k_occluded<<<blocks(n, 128), 128, 0, c->stream>>>(c->S, n, ds, dout);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(occ, dout, sizeof(int) * n, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(ds);
    cudaFree(dout);
  });
}

int pxg_recip_twopoint(int n, double bound, long long cap, uint64_t seed, double* est, long long* cost,
                       int* truncated) {
  return guarded(nullptr, [&]() {
    if (!(bound > 0.0)) throw RuntimeErr{"reciprocal: bound must be positive"};
    if (n <= 0) return;
    if (cap < 0 || cap > (1 << 20)) throw InvalidErr{"pxg_recip_twopoint: cap out of range"};
    const long long capa = std::max<long long>(cap, 1);
    cudaStream_t st = nullptr;
    std::vector<void*> tmp;
    auto A = [&](size_t bytes) {
      void* p = nullptr;
      CK(cudaMalloc(&p, std::max<size_t>(bytes, 1)));
      tmp.push_back(p);
      return p;
    };
    try {
      const size_t nc = static_cast<size_t>(n) * capa;
      auto* de = static_cast<double*>(A(sizeof(double) * n));
      auto* dc = static_cast<long long*>(A(sizeof(long long) * n));
      auto* dt = static_cast<int*>(A(sizeof(int) * n));
      auto* rs = static_cast<RunState*>(A(sizeof(RunState) * n));
      auto* g = static_cast<double*>(A(sizeof(double) * nc));
      auto* ns = static_cast<long long*>(A(sizeof(long long) * nc));
      auto* ne = static_cast<int*>(A(sizeof(int) * nc));
      auto* fr = static_cast<RecipFrame*>(A(sizeof(RecipFrame) * nc));
      int* act[2] = {static_cast<int*>(A(sizeof(int) * n)), static_cast<int*>(A(sizeof(int) * n))};
      auto* nact = static_cast<int*>(A(sizeof(int) * 2));
      auto* derr = static_cast<int*>(A(sizeof(int)));
      CK(cudaMemset(nact, 0, 2 * sizeof(int)));
      CK(cudaMemset(derr, 0, sizeof(int)));
      k_recip_init<<<blocks(n, 128), 128>>>(n, 1, nullptr, nullptr, rs, act[0], nact, de, dc, dt);
      recip_rounds(st, n, act, nact, [&](int cur, int count, int chunk) {
        k_twopoint_eval<<<blocks(static_cast<long long>(count) * chunk, 128), 128>>>(seed, bound, cap, act[cur],
                                                                                     nact + cur, chunk, rs, g, ns, ne);
        k_recip_dfs<<<blocks(count, 128), 128>>>(1, cap, nullptr, bound, act[cur], nact + cur, chunk, rs, g, ns, ne,
                                                 fr, de, dc, dt, act[1 - cur], nact + (1 - cur), derr);
      });
      CK(cudaGetLastError());
      CK(cudaMemcpy(est, de, sizeof(double) * n, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(cost, dc, sizeof(long long) * n, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(truncated, dt, sizeof(int) * n, cudaMemcpyDeviceToHost));
    } catch (...) {
      for (void* p : tmp) cudaFree(p);
      throw;
    }
    for (void* p : tmp) cudaFree(p);
  });
}

int pxg_rng_draws(uint64_t seed, unsigned kind, unsigned sub, uint64_t stream, int n, unsigned* out) {
  return guarded(nullptr, [&]() {
    if (n <= 0) return;
    unsigned* d = dalloc<unsigned>(n);
    k_rng<<<1, 1>>>(seed, kind, sub, stream, n, d);
    CK(cudaGetLastError());
    CK(cudaMemcpy(out, d, sizeof(unsigned) * n, cudaMemcpyDeviceToHost));
    cudaFree(d);
  });
}

int pxg_read_timing(pxg_ctx* c, double* t, long long* counts) {
  if (!c) return fail(nullptr, PXG_E_INVALID, "null context");
  for (int k = 0; k < 8; ++k) t[k] = c->stage_ms[k];
  if (counts) {
    counts[0] = c->launches;
    counts[1] = 0;
  }
  return PXG_OK;
}

}  // extern "C"
