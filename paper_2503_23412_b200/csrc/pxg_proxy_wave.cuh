// pxg_proxy_wave.cuh — the per-pixel proxy connection as a wavefront.
//
// Same computation as k_proxy / proxy_connect (proj/src/proxy.cpp:548-603, 747-813), split
// so every ray goes through the shared traversal kernels:
//   k_pxw_select   gamma draw, pool pick, eligibility; first retrace BSDF sample -> queue
//   (k_trav_persistent closest + k_pxw_retrace) x u   the retrace_proxy chain (:271-319)
//   k_pxw_value    repair, emission, geometric factors, BSDF kernels; every segment's
//                  visibility becomes a shadow ray (proxy.cpp:569-592)
//   (k_trav_persistent any-hit + k_pxw_occlusion)
//   k_pxw_mis      reciprocal-aware MIS weight and the final value (proxy.cpp:594-602)
// Each pixel still consumes its proxy stream (2<<32)+pass*n_px+idx in the reference order.
#pragma once

#include "pxg_wave.cuh"

namespace pxg {

#if defined(__CUDACC__)

struct ProxRec {
  double c[3];
  double u_gate;
  double q_sel;
  int t_label, chosen, key, flags;  // flags bit0 tp>=2, bit1 attempted, bit2 z_norm>0
};

struct PassState {  // device-resident per-pass scalars of a pool slot
  double kappa;
  int n_kept;
  int err;
  long long pool_kept_total;
  int n_ent;      // entries selected by the priority reservoir (min(raw, budget))
  int pad_;
  long long raw;  // eligible candidates of the pass (ProxyDiagnostics::pool_raw)
};

enum { kPxNone = 0, kPxRetrace = 1, kPxRetraced = 2, kPxShadow = 3 };

struct ProxWave {
  int* entry;       // pool entry index
  int* tp;          // eye cut
  unsigned* ctr;    // proxy stream draw counter
  int* step;        // retrace step
  int* state;
  double* density;  // retrace density
  double* pdf;      // pdf of the pending retrace direction
  double* value;    // [3n] unoccluded value
  int* occl;        // any segment occluded
  PV* lv;           // [n * kMaxLight] repaired light sub-path (prefix, block, endpoint)
};

struct ProxCtx {
  SceneView S;
  Mapper M;
  StatsView st;
  const PV* eye;
  const int* n_eye;
  int n, row0, width, max_depth;
  uint64_t seed;
  const IncHdr* inc;
  const PV* prefix;
  const int* label_start;
  const int* label_list;
  const double* gamma_rows;
  const PassState* ps;
};

__device__ __forceinline__ Rng prox_rng(const ProxCtx& C, const ProxWave& W, int i, int pass, int n_px_total) {
  const int idx = C.row0 * C.width + i;
  Rng r;
  r.r = pxg_rng_make(C.seed, PXG_KIND_REF, 0,
                     (uint64_t(2) << 32) + static_cast<uint64_t>(pass) * static_cast<uint64_t>(n_px_total) + idx);
  r.r.i = W.ctr[i];
  return r;
}

// Selection (proxy.cpp:747-798) and the first retrace sample (proxy.cpp:280-288).
// resident 128-thread blocks per SM of the proxy-wavefront kernels (0: no launch bounds; 6 and 8 measured +1%, 8 kept)
#ifndef PXG_PXW_MINB
#define PXG_PXW_MINB 8
#endif
#if PXG_PXW_MINB
#define PXW_BOUNDS __launch_bounds__(128, PXG_PXW_MINB)
#else
#define PXW_BOUNDS
#endif

__global__ void PXW_BOUNDS k_pxw_select(ProxCtx C, ProxWave W, int pass, int n_px_total, ProxRec* out, RayQueue Q) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= C.n) return;
  ProxRec o;
  o.c[0] = o.c[1] = o.c[2] = 0.0;
  o.u_gate = 0.0;
  o.q_sel = 0.0;
  o.t_label = o.chosen = o.key = -1;
  o.flags = 0;
  W.state[i] = kPxNone;
  W.ctr[i] = 0;
  if (C.ps->n_kept <= 0) {
    out[i] = o;
    return;
  }
  const PV* eye = C.eye + i;
  const size_t es = static_cast<size_t>(C.n);
  // cut the eye sub-path at its first non-specular surface vertex (proxy.cpp:749-757)
  const int ne = C.n_eye[i];
  int tp = 0;
  for (int k = 1; k < ne; ++k) {
    const int f = eye[k * es].flag;
    if (f == kDiffuse) {
      tp = k + 1;
      break;
    }
    if (f != kSpecular) break;
  }
  W.tp[i] = tp;
  if (tp < 2) {
    out[i] = o;
    return;
  }
  o.flags |= 1;
  Rng prox = prox_rng(C, W, i, pass, n_px_total);
  o.u_gate = prox.next_double();
  const PV& z = eye[(tp - 1) * es];
  const int t_label = classify_eye(C.M, z.p, -z.wi);
  const double* row = C.gamma_rows + t_label * 100;
  double z_norm = 0.0;
  for (int sl = 0; sl < 100; ++sl)
    if (C.label_start[sl + 1] > C.label_start[sl]) z_norm += row[sl];
  if (!(z_norm > 0.0)) {
    W.ctr[i] = prox.r.i;
    out[i] = o;
    return;
  }
  o.flags |= 4;
  const double uu = prox.next_double() * z_norm;
  int chosen = -1;
  double cdf = 0.0;
  for (int sl = 0; sl < 100; ++sl) {
    if (C.label_start[sl + 1] == C.label_start[sl]) continue;
    chosen = sl;
    cdf += row[sl];
    if (uu < cdf) break;
  }
  const double row_p = row[chosen] / z_norm;
  const int bsize = C.label_start[chosen + 1] - C.label_start[chosen];
  const int e = C.label_list[C.label_start[chosen] + static_cast<int>(prox.next_below(static_cast<uint32_t>(bsize)))];
  const IncHdr& h = C.inc[e];
  const int s_rep = h.n_prefix + h.u + 1;
  o.t_label = t_label;
  o.chosen = chosen;
  o.key = h.key;
  o.q_sel = row_p / static_cast<double>(bsize);
  W.entry[i] = e;
  if (s_rep + tp <= C.max_depth + 1) {
    o.flags |= 2;
    // proxy_connect preconditions (proxy.cpp:551-558)
    if (h.inverse_p > 0.0 && h.prefix_pdf > 0.0) {
      // retrace_proxy start: the specular endpoint lit from the eye vertex
      const V3 d0 = z.p - h.spec_end.p;
      const double l0 = length(d0);
      if (l0 > 0.0) {
        const V3 wi = d0 / l0;
        BsdfSample bs = sample_bsdf(C.S.materials[h.spec_end.mat], h.spec_end.n, wi, prox);
        if (bs.valid && bs.pdf > 0.0) {
          W.state[i] = kPxRetrace;
          W.step[i] = 0;
          W.density[i] = 1.0;
          W.pdf[i] = bs.pdf;
          push_ray(Q, i, h.spec_end.p, bs.wo, 1e30);
        }
      }
    }
  }
  W.ctr[i] = prox.r.i;
  out[i] = o;
}

// One retrace step (proxy.cpp:285-306) for every ray of the queue.
__global__ void PXW_BOUNDS k_pxw_retrace(ProxCtx C, ProxWave W, int pass, int n_px_total, RayQueue in, RayQueue out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= *in.count) return;
  const int i = in.path[j];
  const int prim = in.hit_prim[j];
  if (prim < 0) {
    W.state[i] = kPxNone;
    return;
  }
  const IncHdr& h = C.inc[W.entry[i]];
  const double4 r0 = in.ray[2 * j], r1 = in.ray[2 * j + 1];
  const V3 o = v3(r0.x, r0.y, r0.z), d = v3(r0.w, r1.x, r1.y);
  const double t = in.hit_t[j];
  Hit hit;
  hit.t = t;
  hit.p = o + t * d;
  hit.prim = prim;
  hit.n = prim_normal(C.S, prim, hit.p);
  hit.material = C.S.prim_mat[prim];
  hit.emitter = C.S.prim_emitter[prim];
  PV v = vertex_from_hit(C.S, hit, -d);
  const double pdf = W.pdf[i];
  double density = W.density[i] * to_area_density(pdf, o, v.p, v.n);
  const int step = W.step[i];
  const int u = h.u;
  const bool terminal = step == u - 1;
  if (!terminal) {
    if (!specmat(C.S, v)) {
      W.state[i] = kPxNone;
      return;
    }
  } else {
    if (specmat(C.S, v)) {
      W.state[i] = kPxNone;
      return;
    }
    if (h.dflag_last == kLight) {
      if (v.emitter < 0) {
        W.state[i] = kPxNone;
        return;
      }
      v.flag = kLight;
    }
  }
  v.pdf_fwd = to_area_density(pdf, o, v.p, v.n);
  // block vertex g[step] goes to repaired slot n_prefix + (u - 1 - step)
  W.lv[static_cast<size_t>(i) * kMaxLight + h.n_prefix + (u - 1 - step)] = v;
  W.density[i] = density;
  if (terminal) {
    W.state[i] = (density > 0.0) ? kPxRetraced : kPxNone;
    return;
  }
  Rng prox = prox_rng(C, W, i, pass, n_px_total);
  BsdfSample bs = sample_bsdf(C.S.materials[v.mat], v.n, v.wi, prox);
  W.ctr[i] = prox.r.i;
  if (!bs.valid || bs.pdf <= 0.0) {
    W.state[i] = kPxNone;
    return;
  }
  W.step[i] = step + 1;
  W.pdf[i] = bs.pdf;
  push_ray(out, i, v.p, bs.wo, 1e30);
}

// Repair, value without visibility, and one shadow ray per segment (proxy.cpp:562-592).
__global__ void PXW_BOUNDS k_pxw_value(ProxCtx C, ProxWave W, RayQueue shadow, ProxRec* rec) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= C.n) return;
  W.occl[i] = 0;
  if (W.state[i] != kPxRetraced) return;
  W.state[i] = kPxNone;
  rec[i].flags |= 16;  // retrace accepted (replay dump)
  const IncHdr& h = C.inc[W.entry[i]];
  const PV* pre = C.prefix + static_cast<size_t>(W.entry[i]) * kMaxLight;
  PV* lv = W.lv + static_cast<size_t>(i) * kMaxLight;
  const int u = h.u;
  const int s = h.n_prefix + u + 1;
  for (int k = 0; k < h.n_prefix; ++k) lv[k] = pre[k];
  lv[s - 1] = h.spec_end;
  // re-orient the block's incident directions to light order (proxy.cpp:310-312)
  for (int jj = 0; jj + 1 < u; ++jj) {
    PV& gj = lv[h.n_prefix + (u - 1 - jj)];
    const PV& gn = lv[h.n_prefix + (u - 1 - (jj + 1))];
    gj.wi = normalize(gn.p - gj.p);
  }
  {
    PV& gl = lv[h.n_prefix];
    gl.wi = h.n_prefix > 0 ? normalize(pre[h.n_prefix - 1].p - gl.p) : v3(0.0);
  }
  const size_t es = static_cast<size_t>(C.n);
  const int tp = W.tp[i];
  const PV& z = C.eye[(tp - 1) * es + i];
  V3 d01 = lv[1].p - lv[0].p;
  double l01 = length(d01);
  if (l01 <= 0.0 || lv[0].emitter < 0) return;
  V3 value = emitted(C.S, lv[0].emitter, lv[0].n, d01 / l01);
  if (near_zero(value)) return;
  // geometric factors; visibility deferred to shadow rays (geometry_term, transport.cpp:168-176)
  for (int k = 0; k < s; ++k) {
    const PV& a = lv[k];
    const PV& b = k + 1 < s ? lv[k + 1] : z;
    V3 dd = b.p - a.p;
    double dist2 = dot(dd, dd);
    if (dist2 <= 0.0) return;
    V3 dir = dd / sqrt(dist2);
    double g = fabs(dot(a.n, dir)) * fabs(dot(b.n, dir)) / dist2;
    if (g <= 0.0) return;
    value = value * g;
  }
  for (int k = 1; k < s; ++k) {
    V3 wi = normalize(lv[k - 1].p - lv[k].p);
    V3 to = k + 1 < s ? lv[k + 1].p : z.p;
    V3 wo = normalize(to - lv[k].p);
    V3 fk = eval_bsdf(C.S.materials[lv[k].mat], lv[k].n, wi, wo);
    if (near_zero(fk)) return;
    value = value * fk;
  }
  V3 fz = eval_bsdf(C.S.materials[z.mat], z.n, z.wi, normalize(lv[s - 1].p - z.p));
  if (near_zero(fz)) return;
  value = value * fz * z.thr;
  W.value[3 * i] = value.x;
  W.value[3 * i + 1] = value.y;
  W.value[3 * i + 2] = value.z;
  W.state[i] = kPxShadow;
  // Scene::occluded of every segment (scene.cpp:170-177)
  for (int k = 0; k < s; ++k) {
    const V3 from = lv[k].p;
    const V3 to = k + 1 < s ? lv[k + 1].p : z.p;
    V3 sd = to - from;
    double dist = length(sd);
    if (dist < kRayEps) continue;
    push_ray(shadow, i, from, sd / dist, dist * (1.0 - 1e-6));
  }
}

__global__ void k_pxw_occlusion(ProxWave W, RayQueue shadow) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= *shadow.count) return;
  if (shadow.hit_prim[q]) W.occl[shadow.path[q]] = 1;
}

// reciprocal_mis_weight of the proxy strategy and the final contribution (proxy.cpp:594-602).
__global__ void PXW_BOUNDS k_pxw_mis(ProxCtx C, ProxWave W, ProxRec* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= C.n) return;
  if (W.state[i] != kPxShadow || W.occl[i]) return;
  const IncHdr& h = C.inc[W.entry[i]];
  const int s = h.n_prefix + h.u + 1;
  const int tp = W.tp[i];
  const PV* lv = W.lv + static_cast<size_t>(i) * kMaxLight;
  FullPath fp = make_fp(lv, 1, C.eye + i, static_cast<size_t>(C.n), s, tp);
  const double w = reciprocal_mis_weight(C.S, C.M, C.st, fp, -1, true);
  if (!(w > 0.0)) return;
  const double scale = h.inverse_p * w / (h.prefix_pdf * W.density[i]);
  out[i].c[0] = W.value[3 * i] * scale;
  out[i].c[1] = W.value[3 * i + 1] * scale;
  out[i].c[2] = W.value[3 * i + 2] * scale;
}

#endif  // __CUDACC__

}  // namespace pxg
