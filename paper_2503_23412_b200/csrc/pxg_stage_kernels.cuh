// pxg_stage_kernels.cuh — the per-pass kernels of proxy-BDPT (included by pxg_main.cu).
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
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "pxg.h"
#include "pxg_host.h"
#include "pxg_prims.cuh"
#include "pxg_proxy_wave.cuh"

using namespace pxg;

namespace {

constexpr int kBuckets = 4000;
constexpr int kS = 100, kT = 32;
thread_local std::string g_global_err;





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

constexpr int kBatchSetMax = 32;  // passes per Stage-1 batch, at most

// ------------------------------------------------------------------ Stage 1 kernels
// Eligible prefix ends of the traced pool walks get a 64-bit priority key each
// (the priority-reservoir replacement of Algorithm R, proxy.cpp:696-711).
// All passes of a Stage-1 batch at once: walk i of the batch belongs to pass pass0 + i / n_walks
// (the pool of the batch is vertex-major over L * n_walks paths); pass b's candidates go to
// keys / vals + b * cap, counted in count[b].
__global__ void k_pool_keys(const PV* wpool, const int* wnv, int n_walks, int L, uint64_t seed, int pass0,
                            int walk_begin, unsigned long long* keys, unsigned* vals, int* count, int cap) {
  const unsigned FULL = 0xffffffffu;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int total = L * n_walks;
  const bool live = i < total;
  const int b = live ? i / n_walks : -1;
  const int pass = pass0 + b;
  const int w = live ? walk_begin + i % n_walks : 0;
  const int n = live ? wnv[i] : 0;
  // dropout eligibility (proxy.cpp:59-94) of every prefix end in one forward pass, in registers: the trailing
  // specular run length u, the running pdf product (the same left-to-right product the
  // reference forms for each end) and sliding windows of the last prefix products and
  // emitter ids, enough for u <= 4 (proxy.cpp:59-94). The eligible ends are only recorded
  // (bit `end` of emask): the per-pass candidate counters are single addresses, and an atomic
  // per candidate inside this loop put its round trip on every iteration's critical path
  // (ncu: 42% of the stall samples waited for it).
  double P = 1.0, Pw[5] = {1.0, 1.0, 1.0, 1.0, 1.0};  // Pw[m] = product of pdf[0 .. k-m-1]
  int Ew[6] = {-1, -1, -1, -1, -1, -1};                 // Ew[m] = emitter[k-m]
  int flag0 = -1, run = 0;
  unsigned emask = 0u;
  for (int k = 0; k < n; ++k) {
    const PV& v = wpool[static_cast<size_t>(k) * total + i];
    const int fk = v.flag;
#pragma unroll
    for (int m = 4; m > 0; --m) Pw[m] = Pw[m - 1];
    Pw[0] = P;
#pragma unroll
    for (int m = 5; m > 0; --m) Ew[m] = Ew[m - 1];
    Ew[0] = v.emitter;
    if (k == 0) flag0 = fk;
    run = fk == kSpecular ? run + 1 : 0;
    P *= v.pdf_fwd;
    const int end = k + 1;
    if (end < 2 || fk != kSpecular || run > 4 || run >= end) continue;
    const int u = run, terminal = k - u;
    const int em = u == 1 ? Ew[2] : u == 2 ? Ew[3] : u == 3 ? Ew[4] : Ew[5];  // emitter[terminal - 1]
    const double pp = u == 1 ? Pw[1] : u == 2 ? Pw[2] : u == 3 ? Pw[3] : Pw[4];  // product of pdf[0 .. terminal-1]
    if ((terminal > 0 ? em >= 0 : flag0 == kLight) && pp > 0.0) emask |= 1u << end;
  }
  // one atomic per (warp, pass): the lanes of a pass take consecutive slots (a warp straddles a
  // pass boundary at most once per pass, hence the grouping by pass)
  const int lane = threadIdx.x & 31;
  const int cnt = __popc(emask);
  const unsigned peers = __match_any_sync(FULL, b);
  int before = 0, group = 0;  // candidates of lower lanes of this lane's group / of the whole group
#pragma unroll
  for (int l = 0; l < 32; ++l) {
    const int c = __shfl_sync(FULL, cnt, l);
    if (peers >> l & 1u) {
      group += c;
      if (l < lane) before += c;
    }
  }
  const int leader = __ffs(peers) - 1;
  int base = 0;
  if (live && lane == leader && group > 0) base = atomicAdd(count + b, group);
  base = __shfl_sync(FULL, base, leader);
  int slot = base + before;
  for (unsigned m = emask; m; m &= m - 1, ++slot) {
    if (slot >= cap) break;
    const int end = __ffs(m) - 1;
    Rng kr = make_rng(seed, PXG_KIND_RESERVOIR, static_cast<uint32_t>(end), unit_stream(pass, w));
    unsigned long long hi = pxg_next_u32(&kr.r);
    unsigned long long key = (hi << 32) | pxg_next_u32(&kr.r);
    keys[static_cast<size_t>(b) * cap + slot] = key;
    vals[static_cast<size_t>(b) * cap + slot] = (static_cast<unsigned>(w) << 5) | static_cast<unsigned>(end);
  }
}

// Sorts n (a power of two) (key, value) pairs ascending, lexicographically; all threads.
__device__ void bitonic_sort_pairs(unsigned long long* k, unsigned* v, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int j = size >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj <= i) continue;
        const bool up = (i & size) == 0;
        const unsigned long long ka = k[i], kb = k[ixj];
        const unsigned va = v[i], vb = v[ixj];
        const bool gt = ka > kb || (ka == kb && va > vb);
        if (gt == up) {
          k[i] = kb;
          k[ixj] = ka;
          v[i] = vb;
          v[ixj] = va;
        }
      }
      __syncthreads();
    }
  }
}

// Priority selection of the pool (deviation 2 for Algorithm R, proxy.cpp:696-711) on the
// device, so Stage 1 never waits for the host: the `budget` smallest keys (ties by
// (walk, end)) in (walk, end) order. One block. A key threshold T is bisected until the
// keys below it number between need = min(raw, budget) and the shared-memory capacity `cap`
// (keys are i.i.d. uniform, so the first guess, 2 x budget / raw of the key range, almost
// always lands); those keys are compacted and bitonic-sorted by (key, value), and the
// values of the first `need` are sorted again. Writes n_ent, raw and kappa of the pass.
// Per-pass pointers of a Stage-1 batch (kernel parameter, by value).
struct FrontSet {
  PassState* ps[kBatchSetMax];
  IncHdr* inc[kBatchSetMax];
  PV* prefix[kBatchSetMax];
  int n;
};

__global__ void __launch_bounds__(1024) k_pool_select(const unsigned long long* keys, const unsigned* vals,
                                                      const int* count, int cand_cap, int budget, int cap,
                                                      unsigned* sel, const __grid_constant__ FrontSet fs, int* err) {
  // block b selects pass b of the batch
  const int bb = blockIdx.x;
  keys += static_cast<size_t>(bb) * cand_cap;
  vals += static_cast<size_t>(bb) * cand_cap;
  count += bb;
  sel += static_cast<size_t>(bb) * max(budget, 1);
  PassState* ps = fs.ps[bb];
  extern __shared__ unsigned long long sk[];  // [cap] keys, then [cap] values
  unsigned* sv = reinterpret_cast<unsigned*>(sk + cap);
  __shared__ int s_cnt;
  const int raw = *count;
  const int need = min(raw, max(budget, 0));
  if (threadIdx.x == 0) {
    ps->raw = raw;
    ps->n_ent = raw > cand_cap ? 0 : need;
    const double r = static_cast<double>(budget) / static_cast<double>(raw);
    ps->kappa = raw > 0 ? (r < 1.0 ? r : 1.0) : 1.0;  // std::min(1.0, budget / raw)
    if (raw > cand_cap) set_err(err, kErrPool);
  }
  if (raw > cand_cap || need == 0) return;
  const bool all = raw <= budget;
  unsigned long long lo = 0, hi = ~0ull, T = ~0ull;
  if (!all) {
    const double f = 2.0 * static_cast<double>(budget) / static_cast<double>(raw);
    T = f >= 1.0 ? ~0ull : static_cast<unsigned long long>(f * 18446744073709551616.0);
  }
  for (int it = 0;; ++it) {
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < raw; i += blockDim.x) {
      const unsigned long long key = keys[i];
      if (all || key < T) {
        const int slot = atomicAdd(&s_cnt, 1);
        if (slot < cap) {
          sk[slot] = key;
          sv[slot] = vals[i];
        }
      }
    }
    __syncthreads();
    const int cnt = s_cnt;
    if (all || (cnt >= need && cnt <= cap)) break;
    if (cnt < need) lo = T; else hi = T;
    const unsigned long long nT = lo + (hi - lo) / 2;
    if (nT == T || it > 130) {  // only possible with > cap equal keys
      if (threadIdx.x == 0) {
        set_err(err, kErrPool);
        ps->n_ent = 0;
      }
      return;
    }
    T = nT;
    __syncthreads();
  }
  const int cnt = min(s_cnt, cap);
  int n2 = 1;
  while (n2 < cnt) n2 <<= 1;
  for (int i = cnt + threadIdx.x; i < n2; i += blockDim.x) {
    sk[i] = ~0ull;
    sv[i] = ~0u;
  }
  __syncthreads();
  if (!all) bitonic_sort_pairs(sk, sv, n2);
  // the first `need` values, sorted: (walk << 5 | end) order == (walk, end) order
  int m2 = 1;
  while (m2 < need) m2 <<= 1;
  for (int i = threadIdx.x; i < m2; i += blockDim.x) {  // each index read and written by one thread
    const unsigned long long x = i < need ? static_cast<unsigned long long>(sv[i]) : ~0ull;
    sk[i] = x;
    sv[i] = 0u;
  }
  __syncthreads();
  bitonic_sort_pairs(sk, sv, m2);
  for (int i = threadIdx.x; i < need; i += blockDim.x) sel[i] = static_cast<unsigned>(sk[i]);
}

// Materialise the kept entries (dropout on the stored walk prefix, proxy.cpp:59-94).
// blockIdx.y = pass b of the batch: its selection at sel + b * sel_stride, its walks at
// wpool + b * n_walks_pass in the batch's vertex-major pool (stride n_walks).
__global__ void k_pool_entries(Mapper M, const __grid_constant__ FrontSet fs, const unsigned* sel, int sel_stride,
                               const PV* wpool, int n_walks, int n_walks_pass, int walk_begin) {
  const int b = blockIdx.y;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= fs.ps[b]->n_ent) return;
  sel += static_cast<size_t>(b) * sel_stride;
  wpool += static_cast<size_t>(b) * n_walks_pass;
  IncHdr* inc = fs.inc[b];
  PV* prefix = fs.prefix[b];
  const int w = static_cast<int>(sel[k] >> 5), end = static_cast<int>(sel[k] & 31u);
  PV v[kMaxLight];
  for (int q = 0; q < end; ++q) v[q] = wpool[static_cast<size_t>(q) * n_walks + (w - walk_begin)];
  IncHdr h;
  const bool ok = dropout(M, v, end, h, prefix + static_cast<size_t>(k) * kMaxLight);
  h.walk = w;
  h.end = end;
  h.valid = ok ? 1 : 0;
  inc[k] = h;
}

// The four f/q probes of every entry (estimate_inverse_p, proxy.cpp:389-394), one thread
// per probe on its own stream (PROBE, end | i << 8).
// blockIdx.y = pass b of the batch (pass0 + b); probes of pass b at probe + b * probe_stride.
__global__ void k_pool_probes(SceneView S, uint64_t seed, int pass0, const __grid_constant__ FrontSet fs,
                              double* probe, int* probe_ok, int probe_stride, int repeats) {
  const int b = blockIdx.y;
  const int pass = pass0 + b;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 4 * fs.ps[b]->n_ent) return;
  const IncHdr* inc = fs.inc[b];
  const PV* prefix = fs.prefix[b];
  probe += static_cast<size_t>(b) * probe_stride;
  probe_ok += static_cast<size_t>(b) * probe_stride;
  const int k = t >> 2, i = t & 3;
  probe_ok[t] = 0;
  const IncHdr& h = inc[k];
  if (!h.valid || repeats < 1) return;
  const PV* pre = prefix + static_cast<size_t>(k) * kMaxLight;
  Rng pr = make_rng(seed, PXG_KIND_PROBE, static_cast<uint32_t>(h.end) | (static_cast<uint32_t>(i) << 8),
                    unit_stream(pass, h.walk));
  Cand c;
  support_sample(S, h, pre, pr, c);
  if (!(c.q > 0.0)) return;
  const double f = c.escaped ? 0.0 : target_density(S, h, pre, c.g);
  probe[t] = f / c.q;
  probe_ok[t] = 1;
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

// B of entry k = 2 * max over the bucket's ratio history and the probes of entries <= k
// of the same bucket (the sequential update_ratio/b_bound order of proxy.cpp:389-395).
// Maxima are order-independent, so every entry computes its own prefix maximum; the last
// entry of each bucket then commits the bucket state. One block.
__global__ void k_pool_bounds(const PassState* ps, const IncHdr* inc, const double* probe, const int* probe_ok,
                              double* max_ratio, long long* ratio_cnt, int* touched, double* bound, int* err) {
  // shared: [n_ent] prefix max, [n_ent] touched flags, [4 n_ent] probes (doubles), then
  // [n_ent] keys (-1 = invalid entry), [4 n_ent] probe flags (ints)
  extern __shared__ double sm[];
  const int n_ent = ps->n_ent;
  double* s_pr = sm + 2 * n_ent;
  int* s_key = reinterpret_cast<int*>(s_pr + 4 * n_ent);
  int* s_ok = s_key + n_ent;
  for (int k = threadIdx.x; k < n_ent; k += blockDim.x) s_key[k] = inc[k].valid ? inc[k].key : -1;
  for (int t = threadIdx.x; t < 4 * n_ent; t += blockDim.x) {
    s_ok[t] = probe_ok[t];
    s_pr[t] = s_ok[t] ? probe[t] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n_ent; k += blockDim.x) {
    const int key = inc[k].key;
    double m = max_ratio[key];
    int tch = touched[key];
    for (int k2 = 0; k2 <= k; ++k2) {
      if (s_key[k2] != key) continue;
      for (int i = 0; i < 4; ++i) {
        if (!s_ok[k2 * 4 + i]) continue;
        const double r = s_pr[k2 * 4 + i];
        if (!isfinite(r) || r < 0.0) {
          set_err(err, kErrRatio);
          continue;
        }
        m = dmax(m, r);
        tch = 1;
      }
    }
    bound[k] = (s_key[k] >= 0 && tch) ? 2.0 * m : 0.0;
    sm[k] = m;
    sm[n_ent + k] = tch;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n_ent; k += blockDim.x) {
    const int key = s_key[k];
    if (key < 0) continue;
    bool last = true;
    long long cnt = 0;
    for (int k2 = 0; k2 < n_ent; ++k2) {
      if (s_key[k2] != key) continue;
      if (k2 > k) last = false;
      for (int i = 0; i < 4; ++i) cnt += s_ok[k2 * 4 + i];
    }
    if (!last) continue;
    max_ratio[key] = sm[k];
    ratio_cnt[key] += cnt;
    if (sm[n_ent + k] != 0.0) touched[key] = 1;
  }
}

// One pass of a Stage-1 batch, as seen by the reciprocal-run kernels. Run j of a batch is
// (pass b = j / stride, entry e = (j % stride) / repeats, run r = j % repeats).
struct BatchPass {
  const IncHdr* inc;
  const PV* prefix;
  const double* bound;
  const PassState* ps;  // n_ent is device-resident (selected on the device)
  int pass;
};

// The passes of one Stage-1 batch, passed BY VALUE as a __grid_constant__ kernel parameter
// (no host-to-device copy, so enqueueing a batch never waits for the host). n == 0: the
// two-point fixture (every run live, fixed bound).
struct BatchSet {
  BatchPass p[kBatchSetMax];
  int n;
};

// A node as the DFS consumes it: its frame value g / B (the division is done here, in
// parallel, instead of on the DFS's serial chain; same fp64 operation, same result), its
// split count, and its error code with the sign of g in bits 8 (> 0) and 9 (< 0).
__device__ __forceinline__ void store_node(double* g, long long* nsplit, int* nerr, double gv, double B, long long n,
                                           int err) {
  *g = gv / B;
  *nsplit = n;
  *nerr = err | ((gv > 0.0) ? 0x100 : 0) | ((gv < 0.0) ? 0x200 : 0);
}

// Phase A of the reciprocal runs: evaluate nodes [avail, avail + chunk) of every active
// run in parallel. Node k draws its support sample from (RECIP_NODE, k) and its split
// decision from (RECIP_SPLIT, k) (include/pxg_philox.h), so its value does not depend on
// the tree shape; draw_g (recip.hpp:69-77) and stochastic_split (recip.hpp:49-56).
__global__ void k_recip_eval(SceneView S, uint64_t seed, int repeats, int stride, long long cap,
                             const __grid_constant__ BatchSet bs, const int* active, const int* n_active,
                             int chunk, const RunState* st, double* g, long long* nsplit, int* nerr) {
  const long long total = static_cast<long long>(*n_active) * chunk;
  for (long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; tid < total;
       tid += static_cast<long long>(gridDim.x) * blockDim.x) {
  const long long a = tid / chunk;
  const int j = active[a];
  const long long k = st[j].avail + tid % chunk;
  if (k >= cap) continue;
  const BatchPass& P = bs.p[j / stride];
  const int w = j % stride;
  const int e = w / repeats, r = w % repeats;
  const IncHdr& h = P.inc[e];
  const PV* pre = P.prefix + static_cast<size_t>(e) * kMaxLight;
  const double B = P.bound[e];
  const uint64_t stream = pxg_recip_stream(P.pass, h.walk, h.end, r);
  Rng nr = make_rng(seed, PXG_KIND_RECIP_NODE, static_cast<uint32_t>(k), stream);
  int err = 0;
  const double gv = draw_g(S, h, pre, B, nr, err);
  long long n = 0;
  if (!err) {
    Rng sr = make_rng(seed, PXG_KIND_RECIP_SPLIT, static_cast<uint32_t>(k), stream);
    n = split_count(gv, sr, err);
  }
  const size_t o = static_cast<size_t>(j) * cap + k;
  store_node(g + o, nsplit + o, nerr + o, gv, B, n, err);
  }
}

// Phase A as a block-local wavefront (same values as k_recip_eval, bit for bit). A node's
// draw_g is a chain of up to 4 closest-hit rays (support_sample) and up to 10 visibility rays
// (support_pdf + target_density); one thread per node running them back to back leaves most
// lanes idle (nodes escape after 1 ray or run all 14). Here a block takes 128 nodes at a time:
// every node's glue code runs on its own thread, but each ray phase traces only the rays that
// exist, compacted onto the first threads of the block: (1) sampling chain, <= 4 rounds of
// compacted closest-hit rays; (2) the visibility segments of every node (the density code run
// with a functor that records them and their endpoints, VisDirect's segment ids, and answers
// "visible") as one compacted any-hit list; (3) the recorded density terms, each zeroed when
// one of its segments is hidden (exactly what the reference's early exits produce). Candidate
// vertices and segment endpoints live in a global scratch slot per (block, node).
// Its rays are traced by rw_trace with the persistent kernels' step functions (quantised
// nodes, 32-byte loads); same hits as intersect() / visible() (closest hit with the id tie
// rule and the any-hit boolean do not depend on the visiting order).
#ifndef PXG_RW_WARP
#define PXG_RW_WARP 0  // 1: the warp traces its lanes' rays together with postponed leaf tests
#endif                 //    (warp_trace; measured C4 -1.6%, C2 -2.3%)
__device__ __forceinline__ void thread_trace_closest(const SceneView& S, TravState& ts) {
  int stack_mem[kStack];
  LocalStack stack{stack_mem};
  while (!closest_step(S, ts, stack)) {
  }
}

__device__ __forceinline__ bool thread_trace_any(const SceneView& S, TravState& ts) {
  int stack_mem[kStack];
  LocalStack stack{stack_mem};
  int r;
  while ((r = any_step(S, ts, stack)) == 0) {
  }
  return r == 1;
}

// The reciprocal wavefront's trace of a lane's ray (all lanes of the warp call it; has = the
// lane holds a ray). Closest hit: ts.best / ts.t_best; any hit: true when occluded.
template <bool kAny>
__device__ __forceinline__ bool rw_trace(const SceneView& S, TravState& ts, bool has) {
#if PXG_RW_WARP
  int stack_mem[kStack];
  LocalStack stack{stack_mem};
  return warp_trace<kAny>(S, ts, stack, has);
#else
  if (!has) return false;
  if (kAny) return thread_trace_any(S, ts);
  thread_trace_closest(S, ts);
  return false;
#endif
}

constexpr int kRW = 128;  // nodes per block batch = threads per block
enum { kRWNone = 0, kRWRay = 1, kRWSampled = 2, kRWEscaped = 3 };

struct VisRecord {  // phase 2a: record every segment the density code asks for, answer "visible"
  unsigned* mask;
  double* ends;  // [10][6]: the segment's endpoints a, b
  __device__ __forceinline__ bool operator()(int seg, const V3& a, const V3& b) const {
    *mask |= 1u << seg;
    double* e = ends + 6 * seg;
    e[0] = a.x, e[1] = a.y, e[2] = a.z, e[3] = b.x, e[4] = b.y, e[5] = b.z;
    return true;
  }
};
#ifndef PXG_RW_MINB
#define PXG_RW_MINB 8  // resident blocks per SM (0: none; 8 measured C2 +0.5%, C4 +2.3%, 6 less); the grid follows the occupancy query
#endif
#if PXG_RW_MINB
__global__ void __launch_bounds__(kRW, PXG_RW_MINB) k_recip_eval_wave(
#else
__global__ void __launch_bounds__(kRW) k_recip_eval_wave(
#endif
SceneView S, uint64_t seed, int repeats, int stride,
                                                          long long cap, const __grid_constant__ BatchSet bs,
                                                          const int* active, const int* n_active, int chunk,
                                                          const RunState* st, double* g, long long* nsplit,
                                                          int* nerr, PV* scratch, double* seg_ends, int first_run) {
  __shared__ int s_j[kRW], s_k[kRW];
  __shared__ unsigned s_ctr[kRW], s_need[kRW], s_vis[kRW];
  __shared__ unsigned char s_state[kRW], s_strand[kRW], s_step[kRW];
  __shared__ int s_src[kRW];  // ray origin: -1 spec_end, -2 control vertex, j >= 0 candidate vertex j
  __shared__ double s_dir[kRW][3];
  __shared__ short s_list[kRW];
  __shared__ unsigned short s_seg[kRW * 10];
  __shared__ int s_n, s_nseg;
  const int t = threadIdx.x;
  PV* gv = scratch + (static_cast<size_t>(blockIdx.x) * kRW + t) * 4;  // this thread's node's candidate
  double* ends_block = seg_ends + static_cast<size_t>(blockIdx.x) * kRW * 60;  // [node][seg][6]
  const long long total = static_cast<long long>(*n_active) * chunk;
  // first_run > 0: the global wavefront (pxg_recip_queue.cuh) took the first runs of the list
  for (long long base = static_cast<long long>(first_run) * chunk + static_cast<long long>(blockIdx.x) * kRW;
       base < total; base += static_cast<long long>(gridDim.x) * kRW) {
    // ---- setup + first ray of support_sample (proxy.cpp:211-269)
    const long long tid = base + t;
    int j = -1, k = -1;
    unsigned char state = kRWNone;
    if (tid < total) {
      j = active[tid / chunk];
      const long long kk = st[j].avail + tid % chunk;
      if (kk < cap) k = static_cast<int>(kk);
    }
    if (k >= 0) {
      const BatchPass& P = bs.p[j / stride];
      const int w = j % stride;
      const int e = w / repeats, r = w % repeats;
      const IncHdr& h = P.inc[e];
      const PV* pre = P.prefix + static_cast<size_t>(e) * kMaxLight;
      Rng nr = make_rng(seed, PXG_KIND_RECIP_NODE, static_cast<uint32_t>(k), pxg_recip_stream(P.pass, h.walk, h.end, r));
      const PV* hc = inc_control(h, pre);
      const int strand = (h.u == 1) ? static_cast<int>(nr.next_below(2)) : 0;
      s_strand[t] = static_cast<unsigned char>(strand);
      s_step[t] = 0;
      if (strand == 1 && hc == nullptr) {
        LightPoint lp = sample_light_point(S, nr);
        PV v;
        v.p = lp.p;
        v.n = lp.n;
        v.wi = v3(0.0);
        v.thr = v3(1.0);
        v.pdf_fwd = 0.0;
        v.mat = S.prim_mat[lp.prim];
        v.prim = lp.prim;
        v.emitter = S.prim_emitter[lp.prim];
        v.flag = kLight;
        v.pad = 0.0;
        gv[0] = v;
        state = kRWSampled;
      } else if (strand == 1) {
        V3 dir;
        state = kRWRay;
        if (h.has_cdir) {
          BsdfSample b = sample_bsdf(S.materials[hc->mat], hc->n, -h.cdir, nr);
          if (!b.valid || b.pdf <= 0.0) state = kRWEscaped;
          dir = b.wo;
        } else {
          dir = sample_cosine_hemisphere(hc->n, nr);
        }
        s_src[t] = -2;
        s_dir[t][0] = dir.x, s_dir[t][1] = dir.y, s_dir[t][2] = dir.z;
      } else {
        V3 axis = nr.next_double() < 0.5 ? h.spec_end.n : -h.spec_end.n;
        V3 dir = sample_cosine_hemisphere(axis, nr);
        s_src[t] = -1;
        s_dir[t][0] = dir.x, s_dir[t][1] = dir.y, s_dir[t][2] = dir.z;
        state = kRWRay;
      }
      s_ctr[t] = nr.r.i;
    }
    s_j[t] = j;
    s_k[t] = k;
    s_state[t] = state;
    // ---- (1) sampling chain: <= 4 rounds of compacted closest-hit rays
    for (int round = 0; round < 4; ++round) {
      if (t == 0) s_n = 0;
      __syncthreads();
      if (s_state[t] == kRWRay) s_list[atomicAdd(&s_n, 1)] = static_cast<short>(t);
      __syncthreads();
      const int nray = s_n;
      if (nray == 0) break;  // block-uniform
      if ((t & ~31) < nray) {  // warps holding rays trace them together (postponed leaves)
        const bool has = t < nray;
        int q = 0;
        PV* gq = nullptr;
        TravState ts;
        if (has) {
          q = s_list[t];
          const int jq = s_j[q];
          const BatchPass& P = bs.p[jq / stride];
          const int e = (jq % stride) / repeats;
          const IncHdr& h = P.inc[e];
          const PV* pre = P.prefix + static_cast<size_t>(e) * kMaxLight;
          gq = scratch + (static_cast<size_t>(blockIdx.x) * kRW + q) * 4;
          const int src = s_src[q];
          ts.o = src == -1 ? h.spec_end.p : (src == -2 ? inc_control(h, pre)->p : gq[src].p);
          ts.d = v3(s_dir[q][0], s_dir[q][1], s_dir[q][2]);
          ts.rf = make_rayf(ts.o, ts.d);
          ts.t_best = 1e30;
          ts.best = -1;
          ts.node = 0;
          ts.sp = 0;
          ts.pend_node = 0;
          ts.pend_mask = 0u;
        }
        rw_trace<false>(S, ts, has);
        if (has) {
          if (ts.best < 0) {
            s_state[q] = kRWEscaped;
          } else {
            Hit hit;
            hit.t = ts.t_best;
            hit.p = ts.o + ts.t_best * ts.d;
            hit.prim = ts.best;
            hit.n = prim_normal(S, ts.best, hit.p);
            hit.material = S.prim_mat[ts.best];
            hit.emitter = S.prim_emitter[ts.best];
            gq[s_strand[q] == 1 ? 0 : s_step[q]] = vertex_from_hit(S, hit, -ts.d);
            s_state[q] = kRWSampled;  // provisional: the glue below decides
          }
        }
      }
      __syncthreads();
      // glue: continue the chain of the nodes that just got a vertex (strand 0, u > step+1)
      if (k >= 0 && state == kRWRay) {
        state = s_state[t];
        if (state == kRWSampled && s_strand[t] == 0) {
          const BatchPass& P = bs.p[j / stride];
          const int e = (j % stride) / repeats;
          const IncHdr& h = P.inc[e];
          const int step = s_step[t] + 1;
          s_step[t] = static_cast<unsigned char>(step);
          if (step < h.u) {
            Rng nr = make_rng(seed, PXG_KIND_RECIP_NODE, static_cast<uint32_t>(k),
                              pxg_recip_stream(P.pass, h.walk, h.end, (j % stride) % repeats));
            nr.r.i = s_ctr[t];
            const PV& prev = gv[step - 1];
            BsdfSample b = sample_bsdf(S.materials[prev.mat], prev.n, prev.wi, nr);
            s_ctr[t] = nr.r.i;
            if (!b.valid || b.pdf <= 0.0) {
              state = kRWEscaped;
            } else {
              s_src[t] = step - 1;
              s_dir[t][0] = b.wo.x, s_dir[t][1] = b.wo.y, s_dir[t][2] = b.wo.z;
              state = kRWRay;
            }
          }
        }
        s_state[t] = state;
      }
    }
    // ---- (2a) record the visibility segments the densities ask for
    if (t == 0) s_nseg = 0;
    __syncthreads();
    unsigned need = 0;
    // the densities assuming every segment visible; a hidden segment only zeroes its term
    // (support q_fs: segments 0-3, q_other: 4, target: 5-9), which (2c) applies without
    // evaluating the fp64 densities again
    double qfs_all = 0.0, qoth_all = 0.0, f_all = 0.0;
    int u_node = 0;
    if (k >= 0 && state == kRWSampled) {
      const BatchPass& P = bs.p[j / stride];
      const int e = (j % stride) / repeats;
      const IncHdr& h = P.inc[e];
      const PV* pre = P.prefix + static_cast<size_t>(e) * kMaxLight;
      const VisRecord rec{&need, ends_block + t * 60};
      support_terms_v(S, h, pre, gv, rec, qfs_all, qoth_all);
      u_node = h.u;
      if (support_combine(u_node, qfs_all, qoth_all) > 0.0) {
        unsigned tneed = 0;
        f_all = target_density_v(S, h, pre, gv, VisRecord{&tneed, ends_block + t * 60});
        need |= tneed;
      }
      for (unsigned m = need; m; m &= m - 1)
        s_seg[atomicAdd(&s_nseg, 1)] = static_cast<unsigned short>(t * 16 + (__ffs(m) - 1));
    }
    s_need[t] = need;
    s_vis[t] = 0u;
    __syncthreads();
    // ---- (2b) trace the recorded segments, compacted over the block
    const int nseg = s_nseg;
    for (int i0 = t & ~31; i0 < nseg; i0 += kRW) {  // warp-uniform: lanes of a warp trace together
      const int i = i0 + (t & 31);
      bool has = i < nseg, vis = true;
      int q = 0, sg = 0;
      TravState ts;
      if (has) {
        q = s_seg[i] >> 4;
        sg = s_seg[i] & 15;
        const double* e = ends_block + q * 60 + 6 * sg;
        // visible(from, to) = !occluded (scene.cpp:170-177): unit direction, tmax = dist (1 - 1e-6)
        const V3 from = v3(e[0], e[1], e[2]);
        const V3 dv = v3(e[3], e[4], e[5]) - from;
        const double dist = length(dv);
        if (dist < kRayEps) {
          has = false;  // never occluded
        } else {
          ts.o = from;
          ts.d = dv / dist;
          ts.rf = make_rayf(ts.o, ts.d);
          ts.t_best = dist * (1.0 - 1e-6);
          ts.best = -1;
          ts.node = 0;
          ts.sp = 0;
          ts.pend_node = 0;
          ts.pend_mask = 0u;
        }
      }
      if (rw_trace<true>(S, ts, has)) vis = false;
      if (i < nseg && vis) atomicOr(&s_vis[q], 1u << sg);
    }
    __syncthreads();
    // ---- (2c) the densities with the traced visibilities; draw_g (recip.hpp:69-77), split
    if (k >= 0) {
      const BatchPass& P = bs.p[j / stride];
      const int w = j % stride;
      const int e = w / repeats, r = w % repeats;
      const IncHdr& h = P.inc[e];
      const PV* pre = P.prefix + static_cast<size_t>(e) * kMaxLight;
      const double B = P.bound[e];
      double qx = 1.0, fx = 0.0;
      if (state == kRWSampled) {
        const unsigned hidden = need & ~s_vis[t];
        const double q_fs = (hidden & 0xfu) ? 0.0 : qfs_all;
        const double q_other = (hidden & 0x10u) ? 0.0 : qoth_all;
        qx = support_combine(u_node, q_fs, q_other);
        if (!(qx > 0.0)) qx = 1.0;  // escaped (support_sample's q <= 0 branch)
        else fx = (hidden & 0x3e0u) ? 0.0 : f_all;
      }
      int err = 0;
      if (!isfinite(fx) || fx < 0.0) err = kErrIntegrand;
      else if (!isfinite(qx) || qx <= 0.0) err = kErrSupport;
      const double gval = 1.0 - fx / (B * qx);
      long long n = 0;
      if (!err) {
        Rng sr = make_rng(seed, PXG_KIND_RECIP_SPLIT, static_cast<uint32_t>(k), pxg_recip_stream(P.pass, h.walk, h.end, r));
        n = split_count(gval, sr, err);
      }
      const size_t o = static_cast<size_t>(j) * cap + k;
      store_node(g + o, nsplit + o, nerr + o, gval, B, n, err);
    }
    __syncthreads();  // s_* reused by the next batch
  }
}

}  // namespace
#include "pxg_recip_queue.cuh"
namespace {

// The two-point fixture f = {1, 3}, q = 1/2 (proj/tests/test_recip.cpp:16-23) as Phase A.
__global__ void k_twopoint_eval(uint64_t seed, double bound, long long cap, const int* active, const int* n_active,
                                int chunk, const RunState* st, double* g, long long* nsplit, int* nerr) {
  const long long total = static_cast<long long>(*n_active) * chunk;
  for (long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; tid < total;
       tid += static_cast<long long>(gridDim.x) * blockDim.x) {
  const long long a = tid / chunk;
  const int j = active[a];
  const long long k = st[j].avail + tid % chunk;
  if (k >= cap) continue;
  Rng nr = make_rng(seed, PXG_KIND_RECIP_NODE, static_cast<uint32_t>(k), static_cast<uint64_t>(j));
  const int x = nr.next_double() < 0.5 ? 0 : 1;
  const double fx = x == 0 ? 1.0 : 3.0;
  const double gv = 1.0 - fx / (bound * 0.5);
  int err = 0;
  Rng sr = make_rng(seed, PXG_KIND_RECIP_SPLIT, static_cast<uint32_t>(k), static_cast<uint64_t>(j));
  const long long n = split_count(gv, sr, err);
  const size_t o = static_cast<size_t>(j) * cap + k;
  store_node(g + o, nsplit + o, nerr + o, gv, bound, n, err);
  }
}

// bp == nullptr: every run is live (the two-point fixture).
__global__ void k_recip_init(int runs, int repeats, int stride, const __grid_constant__ BatchSet bs, RunState* st,
                             int* active,
                             int* n_active, double* est, long long* cost, int* trunc) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= runs) return;
  RunState s;
  s.depth = s.cost = s.avail = 0;
  s.ret = 0.0;
  s.entering = 1;
  s.truncated = 0;
  s.err = 0;
  bool live = true;
  if (bs.n) {
    const BatchPass& P = bs.p[j / stride];
    const int e = (j % stride) / repeats;
    live = e < P.ps->n_ent && P.inc[e].valid && P.bound[e] > 0.0;
  }
  s.done = live ? 0 : 1;
  st[j] = s;
  est[j] = 0.0;
  cost[j] = 0;
  trunc[j] = 0;
  if (live) active[atomicAdd(n_active, 1)] = j;
}

// Phase B, warp-cooperative: one warp per active run. The DFS state machine (main_tree,
// recip.hpp:89-97, on an explicit frame stack) runs redundantly (warp-uniform) in every lane; node values are fetched 32 at a time with
// one coalesced load per lane and broadcast by shuffle, and the frame stack's top W frames
// live in shared memory (frames below are spilled to the run's global frame array and
// reloaded in blocks). A long run then costs a few shared-memory round trips per node
// instead of dependent global loads (the single-thread kernel's long-run tail). Same
// arithmetic in the same order as the reference's recursion, so estimates are bit-identical.
template <int W>
__global__ void __launch_bounds__(128) k_recip_dfs_warp(int repeats, int stride, long long cap,
                                                        const __grid_constant__ BatchSet bs, double fixed_bound, const int* active, const int* n_active,
                                                        int chunk, RunState* st, const double* g,
                                                        const long long* nsplit, const int* nerr, RecipFrame* frames,
                                                        double* est, long long* cost, int* trunc, int* next,
                                                        int* n_next, int* err, unsigned long long* node_stat = nullptr) {
  constexpr unsigned FULL = 0xffffffffu;
  __shared__ double s_ans[4][W];
  __shared__ long long s_rem[4][W];
  __shared__ signed char s_sgn[4][W];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_act = *n_active;
  for (long long a = static_cast<long long>(blockIdx.x) * 4 + warp; a < n_act;
       a += static_cast<long long>(gridDim.x) * 4) {  // warp-uniform
  const int j = active[a];
  RunState s = st[j];
  s.avail = min(cap, s.avail + chunk);
  const double B = bs.n ? bs.p[j / stride].bound[(j % stride) / repeats] : fixed_bound;
  const size_t o = static_cast<size_t>(j) * cap;
  const double* G = g + o;
  const long long* N = nsplit + o;
  const int* E = nerr + o;
  RecipFrame* F = frames + o;
  double* sa = s_ans[warp];
  long long* sr = s_rem[warp];
  signed char* sg = s_sgn[warp];
  long long lo = s.depth;  // frames [lo, depth) are in shared memory, [0, lo) in F
  long long base = -1;     // node window: lane i holds node base + i
  double wg = 0.0;
  long long wn = 0;
  int we = 0;
  bool done;
  for (;;) {
    if (s.entering) {
      if (s.depth >= cap || s.cost >= cap) {
        s.entering = 0;
        s.truncated = 1;
        s.ret = 0.0;
      } else {
        const long long k = s.cost;
        if (k >= s.avail) {
          done = false;
          break;
        }
        if (base < 0 || k >= base + 32) {
          base = k;
          const long long kk = k + lane;
          if (kk < s.avail) {
            wg = G[kk];
            wn = N[kk];
            we = E[kk];
          }
        }
        const int src = static_cast<int>(k - base);
        const int ew = __shfl_sync(FULL, we, src);
        const int ek = ew & 0xff;
        s.entering = 0;
        if (ek) {
          s.err = ek;
          s.done = 1;
          done = true;
          break;
        }
        const double ans = __shfl_sync(FULL, wg, src);  // g / B, divided in phase A
        const long long nk = __shfl_sync(FULL, wn, src);
        ++s.cost;
        if (nk > 0) {
          const long long d = s.depth;
          if (d - lo == W) {  // window full: spill its bottom frame
            const int ls = static_cast<int>(lo % W);
            if (lane == 0) F[lo] = RecipFrame{sa[ls], static_cast<double>(sg[ls]), sr[ls]};
            ++lo;
          }
          const int slot = static_cast<int>(d % W);
          sa[slot] = ans;
          sg[slot] = static_cast<signed char>(((ew >> 8) & 1) - ((ew >> 9) & 1));
          sr[slot] = nk - 1;
          ++s.depth;
          s.entering = 1;
          continue;
        }
        s.ret = ans;
      }
    }
    if (s.depth == 0) {
      s.done = 1;
      s.ret = 1.0 / B + s.ret;
      done = true;
      break;
    }
    --s.depth;
    if (s.depth < lo) {  // reload frames [new_lo, depth] spilled earlier
      const long long nl = s.depth - W + 1 > 0 ? s.depth - W + 1 : 0;
      __syncwarp();
      for (long long i = nl + lane; i <= s.depth; i += 32) {
        const RecipFrame fr = F[i];
        const int sl = static_cast<int>(i % W);
        sa[sl] = fr.ans;
        sg[sl] = static_cast<signed char>(fr.sgn);
        sr[sl] = fr.rem;
      }
      __syncwarp();
      lo = nl;
    }
    const int slot = static_cast<int>(s.depth % W);
    const double pa = sa[slot] + static_cast<double>(sg[slot]) * s.ret;
    long long rem = sr[slot];
    sa[slot] = pa;
    // Once cost reaches the cap, every further main_tree call returns 0 from its guard
    // (recip.hpp:79-85) and adds sgn * 0.0 to its parent, which leaves the parent's sum
    // unchanged (it is never -0.0). The reference still loops over all remaining split
    // children (up to |g| of them); here they are skipped, with the same truncation flag.
    if (rem > 0 && s.cost >= cap) {
      s.truncated = 1;
      rem = 0;
      sr[slot] = 0;
    }
    if (rem > 0) {
      sr[slot] = rem - 1;
      ++s.depth;
      s.entering = 1;
      continue;
    }
    s.ret = pa;
  }
  if (!done) {  // flush the window; the next round resumes from global frames
    __syncwarp();
    for (long long i = lo + lane; i < s.depth; i += 32) {
      const int sl = static_cast<int>(i % W);
      F[i] = RecipFrame{sa[sl], static_cast<double>(sg[sl]), sr[sl]};
    }
  }
  if (lane == 0) {
    st[j] = s;
    if (!done) {
      next[atomicAdd(n_next, 1)] = j;
    } else if (s.err) {
      set_err(err, s.err);
    } else {
      est[j] = s.ret;
      cost[j] = s.cost;
      trunc[j] = s.truncated;
      if (node_stat) {  // evaluated vs consumed tree nodes of the finished run
        atomicAdd(node_stat + 0, static_cast<unsigned long long>(s.avail));
        atomicAdd(node_stat + 1, static_cast<unsigned long long>(s.cost));
        atomicAdd(node_stat + 2, 1ull);
      }
    }
  }
  __syncwarp();
  }
}

// Sorts n (a power of two) 64-bit keys ascending in shared memory; all threads.
__device__ void bitonic_sort_u64(unsigned long long* k, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int j = size >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj <= i) continue;
        const unsigned long long a = k[i], b = k[ixj];
        if ((a > b) == ((i & size) == 0)) {
          k[i] = b;
          k[ixj] = a;
        }
      }
      __syncthreads();
    }
  }
}

// Per entry: mean and second moment of its runs, validity (proxy.cpp:409-427); per bucket
// the estimate sums in pool order; the kept list and the per-label lists in pool order
// (proxy.cpp:729-735); then the stats snapshot Stage 2 of this pass reads. One block of
// 1024 threads; the orders come from shared-memory sorts of (bucket | label, entry) keys, so
// every bucket's sum runs over its entries in entry order exactly like the reference.
__global__ void __launch_bounds__(1024) k_pool_finish(int repeats, IncHdr* inc, const double* bound,
                                                      const double* est, const int* trunc, double* sum_est,
                                                      double* sum_sq, long long* est_cnt, int* touched,
                                                      long long* diag, int* diag_touched, int* kept, int* label_start,
                                                      int* label_list, PassState* ps, double* snap_sum,
                                                      double* snap_sq, long long* snap_cnt) {
  const int n_ent = ps->n_ent;
  int n2 = 1;
  while (n2 < n_ent) n2 <<= 1;
  // shared: [n2] sort keys (u64), [n_ent] inverse_p (double), [n_ent] valid flags, [n_ent]
  // labels, [kS] label counts, [1024] scan
  extern __shared__ unsigned long long smk[];
  unsigned long long* sk = smk;
  double* s_inv = reinterpret_cast<double*>(sk + n2);
  int* ok = reinterpret_cast<int*>(s_inv + n_ent);
  int* s_lab = ok + n_ent;
  int* lcount = s_lab + n_ent;
  int* scan = lcount + kS;
  for (int s = threadIdx.x; s < kS; s += blockDim.x) lcount[s] = 0;
  for (int k = threadIdx.x; k < n_ent; k += blockDim.x) {
    IncHdr& h = inc[k];
    ok[k] = 0;
    s_lab[k] = h.s_label;
    sk[k] = ~0ull;
    if (!h.valid) continue;
    const int key = h.key;
    diag_touched[key] = 1;
    bool valid = false;
    if (repeats >= 1 && bound[k] > 0.0) {
      double sum = 0.0, sq = 0.0;
      long long tr = 0;
      for (int r = 0; r < repeats; ++r) {
        const double e = est[k * repeats + r];
        sum += e;
        sq += e * e;
        tr += trunc[k * repeats + r];
      }
      const double mean = sum / repeats;
      const double m2 = sq / repeats;
      atomicAdd(reinterpret_cast<unsigned long long*>(&diag[key * 5 + 3]), static_cast<unsigned long long>(tr));
      if (isfinite(mean) && mean > 0.0) {
        valid = true;
        h.inverse_p = mean;
        h.inverse_p_m2 = m2;
        s_inv[k] = mean;
      }
    }
    atomicAdd(reinterpret_cast<unsigned long long*>(&diag[key * 5 + 2]), static_cast<unsigned long long>(repeats));
    if (!valid) atomicAdd(reinterpret_cast<unsigned long long*>(&diag[key * 5 + 4]), 1ull);
    ok[k] = valid ? 1 : 0;
    if (valid) sk[k] = (static_cast<unsigned long long>(key) << 32) | static_cast<unsigned>(k);
  }
  for (int k = n_ent + threadIdx.x; k < n2; k += blockDim.x) sk[k] = ~0ull;
  __syncthreads();
  // bucket sums in pool order (SubspaceStats::update_estimate, subspace.cpp:64-70): after the
  // sort by (bucket, entry) each bucket is one segment, summed by one thread in entry order
  bitonic_sort_u64(sk, n2);
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    if (sk[i] == ~0ull) continue;
    const int key = static_cast<int>(sk[i] >> 32);
    if (i > 0 && static_cast<int>(sk[i - 1] >> 32) == key) continue;
    double se = sum_est[key], sq = sum_sq[key];
    long long cnt = est_cnt[key];
    for (int j = i; j < n2 && sk[j] != ~0ull && static_cast<int>(sk[j] >> 32) == key; ++j) {
      const double m = s_inv[static_cast<unsigned>(sk[j])];
      se += m;
      sq += m * m;
      ++cnt;
    }
    sum_est[key] = se;
    sum_sq[key] = sq;
    est_cnt[key] = cnt;
    touched[key] = 1;
  }
  __syncthreads();
  // kept list in entry order: block exclusive scan of the valid flags over chunks
  const int chunk = (n_ent + blockDim.x - 1) / blockDim.x;
  const int k0 = threadIdx.x * chunk;
  int mine = 0;
  for (int k = k0; k < min(n_ent, k0 + chunk); ++k) mine += ok[k];
  scan[threadIdx.x] = mine;
  __syncthreads();
  for (int off = 1; off < static_cast<int>(blockDim.x); off <<= 1) {
    const int v = threadIdx.x >= off ? scan[threadIdx.x - off] : 0;
    __syncthreads();
    scan[threadIdx.x] += v;
    __syncthreads();
  }
  {
    int pos = scan[threadIdx.x] - mine;
    for (int k = k0; k < min(n_ent, k0 + chunk); ++k)
      if (ok[k]) kept[pos++] = k;
  }
  const int n_kept = scan[blockDim.x - 1];
  // label lists: sort by (label, entry); label_start from the per-label counts
  for (int k = threadIdx.x; k < n2; k += blockDim.x) {
    if (k < n_ent && ok[k]) {
      sk[k] = (static_cast<unsigned long long>(s_lab[k]) << 32) | static_cast<unsigned>(k);
      atomicAdd(&lcount[s_lab[k]], 1);
    } else {
      sk[k] = ~0ull;
    }
  }
  __syncthreads();
  bitonic_sort_u64(sk, n2);
  for (int i = threadIdx.x; i < n_kept; i += blockDim.x) label_list[i] = static_cast<int>(static_cast<unsigned>(sk[i]));
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int s = 0; s < kS; ++s) {
      label_start[s] = acc;
      acc += lcount[s];
    }
    label_start[kS] = acc;
    ps->n_kept = n_kept;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kBuckets; b += blockDim.x) {
    snap_sum[b] = sum_est[b];
    snap_sq[b] = sum_sq[b];
    snap_cnt[b] = est_cnt[b];
  }
}

// A pass's Stage-1 diagnostics are folded into the context totals only when the pass is
// rendered, so a look-ahead Stage 1 never shows up in ProxyDiagnostics early.
__global__ void k_fold_diag(const long long* sdiag, const int* stouched, const PassState* ps, long long* diag,
                            int* touched, unsigned long long* kept_total) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0) {
    atomicAdd(kept_total, static_cast<unsigned long long>(ps->n_kept));
    atomicAdd(kept_total + 1, static_cast<unsigned long long>(ps->raw));
  }
  if (b >= kBuckets) return;
  for (int k = 2; k < 5; ++k) diag[b * 5 + k] += sdiag[b * 5 + k];
  if (stouched[b]) touched[b] = 1;
}

// GammaMatrix::record_contribution in pixel scan order (proxy.cpp:807-808) + end_iteration
// (subspace.cpp:164-182). Input: contributions stably sorted by bin (pixel order kept).
__global__ void k_gamma_update(int n, const int* bins_sorted, const double* vals_sorted, double* accum, double* rows,
                               int learning) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;  // one thread per (t, s) bin
  if (b < kT * kS && learning) {
    // segment of bin b+1 (key 0 = no contribution)
    int lo = 0, hi = n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (bins_sorted[mid] < b + 1) lo = mid + 1; else hi = mid;
    }
    double acc = accum[b];
    for (int k = lo; k < n && bins_sorted[k] == b + 1; ++k) {
      const double v = vals_sorted[k];
      if (!isfinite(v) || v < 0.0) continue;
      acc += v;
    }
    accum[b] = acc;
  }
}

__global__ void k_gamma_rows(const double* accum, double* rows) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= kT) return;
  const double eps = 1e-3 / kS;
  double* row = rows + t * kS;
  const double* acc = accum + t * kS;
  double total = 0.0;
  for (int s = 0; s < kS; ++s) total += acc[s];
  if (total <= 0.0) {
    for (int s = 0; s < kS; ++s) row[s] = 1.0 / kS;
    return;
  }
  const double keep = 1.0 - eps * kS;
  for (int s = 0; s < kS; ++s) row[s] = keep * (acc[s] / total) + eps;
}

// ------------------------------------------------------------------ Stage 2 kernels
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

// Per 10x10 cell in the reference's scan order (proxy.cpp:761-817).
__global__ void k_gate(int n_cells, int grid_w, int row0, int rows, int width, int pass, double gate_high,
                       double gate_low, double gate_threshold, double light_walks, int proxy_on,
                       const PassState* ps, const double* bdpt, const ProxRec* prox, double* acc, double* val,
                       double* grid_total, double* grid_proxy, int* gbin, double* gval, int* pflags,
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
      int gb = 0;  // 0: no gamma contribution, else t*100 + s + 1
      double gv = 0.0;
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
                gb = o.t_label * kS + o.chosen + 1;
                gv = luminance(c) / o.q_sel;
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
      gbin[i] = gb;
      gval[i] = gv;
      pflags[i] = fl;
    }
  }
  grid_total[cell] = gt;
  grid_proxy[cell] = gp;
}

// ------------------------------------------------------------------ test kernels
// ---- parity probes of the proxy densities on caller-supplied vertices (pxg_proxy_probe)
// dropout (proxy.cpp:59-94) of a hand-built light walk: info = {valid, u, n_prefix, has_cdir,
// c_label, s_label, key, dflag_last}.
__global__ void k_probe_dropout(Mapper M, const PV* walk, int n_walk, IncHdr* hdr, PV* prefix, int* info,
                                double* prefix_pdf) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  IncHdr h;
  h.valid = 0;
  const bool ok = n_walk <= kMaxLight && dropout(M, walk, n_walk, h, prefix);
  h.valid = ok ? 1 : 0;
  h.walk = 0;
  h.end = n_walk;
  *hdr = h;
  info[0] = h.valid;
  if (!ok) return;
  info[1] = h.u, info[2] = h.n_prefix, info[3] = h.has_cdir, info[4] = h.c_label, info[5] = h.s_label;
  info[6] = h.key, info[7] = h.dflag_last;
  *prefix_pdf = h.prefix_pdf;
}

// support_pdf (proxy.cpp:153-209) and target_density (proxy.cpp:106-151) of candidate blocks
// cand[i * u .. i * u + u) for the probed incomplete sub-path.
__global__ void k_probe_densities(SceneView S, const IncHdr* hdr, const PV* prefix, int n, const PV* cand, double* q,
                                  double* f) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !hdr->valid) return;
  PV g[4];
  for (int k = 0; k < hdr->u; ++k) g[k] = cand[static_cast<size_t>(i) * hdr->u + k];
  q[i] = support_pdf(S, *hdr, prefix, g);
  f[i] = target_density(S, *hdr, prefix, g);
}

// support_sample (proxy.cpp:211-269), draw i on stream (seed, PROBE, 0, i): the candidate
// block, its mixture density (1 for an escaped draw) and the escape flag.
__global__ void k_probe_samples(SceneView S, uint64_t seed, const IncHdr* hdr, const PV* prefix, int n, PV* cand,
                                double* q, int* escaped) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !hdr->valid) return;
  Rng rng = make_rng(seed, PXG_KIND_PROBE, 0, static_cast<uint64_t>(i));
  Cand c;
  support_sample(S, *hdr, prefix, rng, c);
  q[i] = c.q;
  escaped[i] = c.escaped ? 1 : 0;
  if (!c.escaped)
    for (int k = 0; k < hdr->u; ++k) cand[static_cast<size_t>(i) * hdr->u + k] = c.g[k];
}

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

