// pxg_recip_queue.cuh — reciprocal tree nodes evaluated as a GLOBAL wavefront (included by
// pxg_stage_kernels.cuh after the block-local k_recip_eval_wave, whose values it reproduces
// bit for bit).
//
// A node's draw_g (recip.hpp:69-77) is a chain of up to 4 closest-hit rays (support_sample,
// proxy.cpp:211-269) and up to 10 visibility segments (support_pdf + target_density). The
// block-local wavefront traced them with per-lane loops inside one kernel: ncu (C4) showed 80%
// of its instructions in traversal at 9 of 32 lanes and 15% of its stall samples at the block
// barriers between phases. Here every phase of ALL pending nodes of a round is one launch:
//
//   k_rq_setup    one thread per node: strand choice, first ray -> closest-hit queue
//   (<= 4 times)  k_trav_persistent<0> over the queue (lane refill, postponed leaves: the
//                 production traversal), then k_rq_glue: hit -> candidate vertex, next ray
//   k_rq_record   both densities with a functor that pushes every visibility segment they ask
//                 for into the any-hit queue and answers "visible"
//                 k_trav_persistent<1> over the segments, k_rq_vis folds the results
//   k_rq_finish   a density term with a hidden segment becomes 0 (what the reference's early
//                 exits yield), g = 1 - f / (B q), stochastic_split -> the DFS's node arrays
//
// so the rays of a round (millions on C4) share the persistent traversal kernels' queue, and
// the glue code runs at full occupancy with no ray in flight. Per-node state lives in HBM
// (RqItem + 4 candidate vertices); a round's nodes beyond the scratch capacity are left to the
// block-local kernel (same values), so no configuration can overflow it.
#pragma once

#ifndef PXG_RQ_MINB
#define PXG_RQ_MINB 8  // resident 128-thread blocks per SM of the glue kernels (64 registers; C2 +1%, C4 neutral vs unbounded)
#endif

namespace {

struct RqItem {  // 48 B per pending node
  int j, k;      // run, tree node (k < 0: nothing to evaluate)
  unsigned ctr;  // Philox counter of the node stream after the draws so far
  unsigned need, vis;
  unsigned char state, strand, step, u;
  double qfs, qoth, f;  // density terms assuming every segment visible
};

struct RqView {
  RqItem* item;
  PV* gv;  // [item][4] candidate block
  int cap; // items
};

// Nodes of this round handled by the global wavefront: the first min(n_active, served) runs.
__device__ __forceinline__ long long rq_total(const int* n_active, int served, int chunk) {
  const int runs = min(*n_active, served);
  return static_cast<long long>(runs) * chunk;
}

__device__ __forceinline__ void rq_push(const RayQueue& Q, int tag, const V3& o, const V3& d, double tmax) {
  const int slot = atomicAdd(Q.count, 1);
  Q.ray[2 * slot] = make_double4(o.x, o.y, o.z, d.x);
  Q.ray[2 * slot + 1] = make_double4(d.y, d.z, tmax, 0.0);
  Q.path[slot] = tag;
}

__global__ void __launch_bounds__(128, PXG_RQ_MINB) k_rq_setup(SceneView S, uint64_t seed, int repeats, int stride, long long cap,
                                                  const __grid_constant__ BatchSet bs, const int* active,
                                                  const int* n_active, int served, int chunk, const RunState* st,
                                                  RqView R, RayQueue Q) {
  const long long total = rq_total(n_active, served, chunk);
  for (long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; tid < total;
       tid += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int j = active[tid / chunk];
    const long long kk = st[j].avail + tid % chunk;
    RqItem it;
    it.j = j;
    it.k = kk < cap ? static_cast<int>(kk) : -1;
    it.ctr = 0u;
    it.need = it.vis = 0u;
    it.state = kRWNone;
    it.strand = it.step = it.u = 0;
    it.qfs = it.qoth = it.f = 0.0;
    if (it.k >= 0) {
      const BatchPass& P = bs.p[j / stride];
      const int w = j % stride;
      const int e = w / repeats, r = w % repeats;
      const IncHdr& h = P.inc[e];
      const PV* pre = P.prefix + static_cast<size_t>(e) * kMaxLight;
      Rng nr = make_rng(seed, PXG_KIND_RECIP_NODE, static_cast<uint32_t>(it.k), pxg_recip_stream(P.pass, h.walk, h.end, r));
      const PV* hc = inc_control(h, pre);
      const int strand = (h.u == 1) ? static_cast<int>(nr.next_below(2)) : 0;
      it.strand = static_cast<unsigned char>(strand);
      it.u = static_cast<unsigned char>(h.u);
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
        R.gv[static_cast<size_t>(tid) * 4] = v;
        it.state = kRWSampled;
      } else if (strand == 1) {
        V3 dir;
        it.state = kRWRay;
        if (h.has_cdir) {
          BsdfSample b = sample_bsdf(S.materials[hc->mat], hc->n, -h.cdir, nr);
          if (!b.valid || b.pdf <= 0.0) it.state = kRWEscaped;
          dir = b.wo;
        } else {
          dir = sample_cosine_hemisphere(hc->n, nr);
        }
        if (it.state == kRWRay) rq_push(Q, static_cast<int>(tid), hc->p, dir, 1e30);
      } else {
        V3 axis = nr.next_double() < 0.5 ? h.spec_end.n : -h.spec_end.n;
        V3 dir = sample_cosine_hemisphere(axis, nr);
        it.state = kRWRay;
        rq_push(Q, static_cast<int>(tid), h.spec_end.p, dir, 1e30);
      }
      it.ctr = nr.r.i;
    }
    R.item[tid] = it;
  }
}

// After a closest-hit round: the hit becomes the next candidate vertex; a from-specular chain
// (strand 0) with vertices left samples its next direction and pushes the next ray. A block
// takes 256 consecutive rays and regroups them in shared memory (counting sort, as k_shade
// does) by what they need: a BSDF sample (by the lobe set of the hit material), only the
// vertex, or nothing (escaped), so the warps that sample run one kind of BSDF and the escaped
// rays cost whole idle warps, not idle lanes (ncu before: 9.4 of 32 lanes).
constexpr int kGlueT = 256;
__global__ void __launch_bounds__(kGlueT, PXG_RQ_MINB / 2) k_rq_glue(SceneView S, uint64_t seed, int repeats, int stride,
                                                                     const __grid_constant__ BatchSet bs, RqView R,
                                                                     RayQueue in, RayQueue out) {
  __shared__ int s_cnt[8];
  __shared__ short s_perm[kGlueT];
  const int n = *in.count;
  for (int s0 = blockIdx.x * kGlueT; s0 < n; s0 += gridDim.x * kGlueT) {  // block-uniform trips
    if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    int cls = 7;  // past the end of the queue
    {
      const int s = s0 + threadIdx.x;
      if (s < n) {
        const int prim = in.hit_prim[s];
        if (prim < 0) {
          cls = 6;  // escaped: only the state changes
        } else {
          const RqItem& it = R.item[in.path[s]];
          cls = 5;  // vertex only
          if (it.strand == 0 && it.step + 1 < it.u) {
            const Material& m = S.materials[S.prim_mat[prim]];
            double wd, wm, wt;
            lobes(m, wd, wm, wt);
            const int bits = ((wd > 0.0) ? 1 : 0) | ((wm > 0.0) ? 2 : 0) | ((wt > 0.0) ? 4 : 0);
            cls = bits == 1 ? 0 : bits == 2 ? 1 : bits == 4 ? 2 : bits == 3 ? 3 : 4;
          }
        }
      }
    }
    const int pos = atomicAdd(&s_cnt[cls], 1);
    __syncthreads();
    int base = 0;
#pragma unroll
    for (int k = 0; k < 7; ++k)
      if (k < cls) base += s_cnt[k];
    if (cls < 7) s_perm[base + pos] = static_cast<short>(threadIdx.x);
    const int live = kGlueT - s_cnt[7];
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < live) {
      const int s = s0 + s_perm[threadIdx.x];
      const int t = in.path[s];
      RqItem& it = R.item[t];
      const int prim = in.hit_prim[s];
      if (prim < 0) {
        it.state = kRWEscaped;
      } else {
        const double4 r0 = in.ray[2 * s], r1 = in.ray[2 * s + 1];
        const V3 o = v3(r0.x, r0.y, r0.z), d = v3(r0.w, r1.x, r1.y);
        Hit hit;
        hit.t = in.hit_t[s];
        hit.p = o + hit.t * d;
        hit.prim = prim;
        hit.n = prim_normal(S, prim, hit.p);
        hit.material = S.prim_mat[prim];
        hit.emitter = S.prim_emitter[prim];
        PV* gv = R.gv + static_cast<size_t>(t) * 4;
        const int strand = it.strand;
        int step = it.step;
        const PV v = vertex_from_hit(S, hit, -d);
        gv[strand == 1 ? 0 : step] = v;
        unsigned char state = kRWSampled;
        if (strand == 0) {
          ++step;
          it.step = static_cast<unsigned char>(step);
          if (step < it.u) {
            const int j = it.j;
            const BatchPass& P = bs.p[j / stride];
            const int w = j % stride;
            const IncHdr& h = P.inc[w / repeats];
            Rng nr = make_rng(seed, PXG_KIND_RECIP_NODE, static_cast<uint32_t>(it.k),
                              pxg_recip_stream(P.pass, h.walk, h.end, w % repeats));
            nr.r.i = it.ctr;
            BsdfSample b = sample_bsdf(S.materials[v.mat], v.n, v.wi, nr);
            it.ctr = nr.r.i;
            if (!b.valid || b.pdf <= 0.0) {
              state = kRWEscaped;
            } else {
              state = kRWRay;
              rq_push(out, t, v.p, b.wo, 1e30);
            }
          }
        }
        it.state = state;
      }
    }
    __syncthreads();  // s_cnt / s_perm are reused by the next tile
  }
}

// The density code's visibility functor: push the segment as an any-hit ray tagged
// (node << 4 | segment id) and answer "visible"; visible(a, b) = !occluded (scene.cpp:170-177):
// unit direction, tmax = dist (1 - 1e-6); a segment shorter than kRayEps is never occluded.
struct VisPush {
  unsigned* need;
  unsigned* vis;
  RayQueue Q;
  int node;
  __device__ __forceinline__ bool operator()(int seg, const V3& a, const V3& b) const {
    *need |= 1u << seg;
    const V3 dv = b - a;
    const double dist = length(dv);
    if (dist < kRayEps) {
      *vis |= 1u << seg;
    } else {
      rq_push(Q, node * 16 + seg, a, dv / dist, dist * (1.0 - 1e-6));
    }
    return true;
  }
};

// The nodes of a block's tile are regrouped like k_rq_glue's rays: by the dropped block's
// length u and by whether a control vertex exists (the two things that decide which density
// terms and how many segments a node has); nodes without a sampled candidate drop out.
__global__ void __launch_bounds__(kGlueT, PXG_RQ_MINB / 2) k_rq_record(SceneView S, int repeats, int stride,
                                                                       const __grid_constant__ BatchSet bs,
                                                                       const int* n_active, int served, int chunk,
                                                                       RqView R, RayQueue Q) {
  __shared__ int s_cnt[9];
  __shared__ short s_perm[kGlueT];
  const long long total = rq_total(n_active, served, chunk);
  for (long long t0 = static_cast<long long>(blockIdx.x) * kGlueT; t0 < total;
       t0 += static_cast<long long>(gridDim.x) * kGlueT) {  // block-uniform trips
    if (threadIdx.x < 9) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    int cls = 8;  // nothing to record
    {
      const long long tid = t0 + threadIdx.x;
      if (tid < total) {
        const RqItem& it = R.item[tid];
        if (it.k >= 0 && it.state == kRWSampled) {
          const BatchPass& P = bs.p[it.j / stride];
          const IncHdr& h = P.inc[(it.j % stride) / repeats];
          cls = 2 * (min(max(h.u, 1), 4) - 1) + (h.n_prefix > 0 ? 1 : 0);
        }
      }
    }
    const int pos = atomicAdd(&s_cnt[cls], 1);
    __syncthreads();
    int base = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (k < cls) base += s_cnt[k];
    if (cls < 8) s_perm[base + pos] = static_cast<short>(threadIdx.x);
    const int live = kGlueT - s_cnt[8];
    __syncthreads();
    if (static_cast<int>(threadIdx.x) < live) {
      const long long tid = t0 + s_perm[threadIdx.x];
      RqItem& it = R.item[tid];
      const int j = it.j;
      const BatchPass& P = bs.p[j / stride];
      const int e = (j % stride) / repeats;
      const IncHdr& h = P.inc[e];
      const PV* pre = P.prefix + static_cast<size_t>(e) * kMaxLight;
      const PV* gv = R.gv + static_cast<size_t>(tid) * 4;
      unsigned need = 0u, vis = 0u;
      double qfs = 0.0, qoth = 0.0, f = 0.0;
      const VisPush rec{&need, &vis, Q, static_cast<int>(tid)};
      support_terms_v(S, h, pre, gv, rec, qfs, qoth);
      if (support_combine(h.u, qfs, qoth) > 0.0) f = target_density_v(S, h, pre, gv, rec);
      it.need = need;
      it.vis = vis;
      it.qfs = qfs;
      it.qoth = qoth;
      it.f = f;
    }
    __syncthreads();  // s_cnt / s_perm are reused by the next tile
  }
}

__global__ void __launch_bounds__(256) k_rq_vis(RayQueue Q, RqView R) {
  const int n = *Q.count;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    if (Q.hit_prim[s] != 0) continue;  // occluded
    const int tag = Q.path[s];
    atomicOr(&R.item[tag >> 4].vis, 1u << (tag & 15));
  }
}

__global__ void __launch_bounds__(128, PXG_RQ_MINB) k_rq_finish(uint64_t seed, int repeats, int stride, long long cap,
                                                   const __grid_constant__ BatchSet bs, const int* n_active,
                                                   int served, int chunk, RqView R, double* g, long long* nsplit,
                                                   int* nerr) {
  const long long total = rq_total(n_active, served, chunk);
  for (long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; tid < total;
       tid += static_cast<long long>(gridDim.x) * blockDim.x) {
    const RqItem it = R.item[tid];
    if (it.k < 0) continue;
    const int j = it.j;
    const BatchPass& P = bs.p[j / stride];
    const int w = j % stride;
    const int e = w / repeats, r = w % repeats;
    const IncHdr& h = P.inc[e];
    const double B = P.bound[e];
    double qx = 1.0, fx = 0.0;
    if (it.state == kRWSampled) {
      const unsigned hidden = it.need & ~it.vis;
      const double q_fs = (hidden & 0xfu) ? 0.0 : it.qfs;
      const double q_other = (hidden & 0x10u) ? 0.0 : it.qoth;
      qx = support_combine(it.u, q_fs, q_other);
      if (!(qx > 0.0)) qx = 1.0;  // escaped (support_sample's q <= 0 branch)
      else fx = (hidden & 0x3e0u) ? 0.0 : it.f;
    }
    int err = 0;
    if (!isfinite(fx) || fx < 0.0) err = kErrIntegrand;
    else if (!isfinite(qx) || qx <= 0.0) err = kErrSupport;
    const double gval = 1.0 - fx / (B * qx);
    long long n = 0;
    if (!err) {
      Rng sr = make_rng(seed, PXG_KIND_RECIP_SPLIT, static_cast<uint32_t>(it.k), pxg_recip_stream(P.pass, h.walk, h.end, r));
      n = split_count(gval, sr, err);
    }
    const size_t o = static_cast<size_t>(j) * cap + it.k;
    store_node(g + o, nsplit + o, nerr + o, gval, B, n, err);
  }
}

}  // namespace
