// pxg_wave.cuh — wavefront kernels: sub-path tracing bounce by bounce over compacted ray
// queues, lean closest-hit / any-hit traversal kernels, and the standard connections
// expanded to one thread per (pixel, t, s) strategy slot.
//
// Why: the per-pixel megakernel version ran at 4.6/32 (trace) and 3.6/32 (connect) active
// threads per warp instruction with 12 warps/SM resident (142 registers) — divergence- and
// latency-bound, DRAM at 1% (profiles/r1_megakernel.md). Splitting the traversal out lets
// every warp of the traversal kernels run the same loop with a small register footprint,
// and the queues keep only live rays.
//
// Bit-exactness is kept: each path still consumes its own Philox stream in the reference
// order (the queue order never matters), and the per-pixel sum of strategy contributions
// is done in the reference's (t, s) order by k_conn_sum.
#pragma once

#include "pxg_proxy.cuh"

namespace pxg {

#if defined(__CUDACC__)

// A set of sub-paths traced in lock-step bounces (eye paths, light paths or pool walks).
struct PathSet {
  PV* pool;          // vertex-major: vertex k of path i at pool[k * n + i]
  int* nv;           // vertices so far
  unsigned* ctr;     // Philox draw counter of the path's stream
  double* beta;      // [n*3]
  double* pdf_dir;   // [n]
  uint64_t seed;
  uint64_t stream_base;  // stream of path i = stream_base + (i / per_pass) << 32 + i % per_pass
  uint32_t kind;
  int n;
  int max_vertices;
  int eye;           // 1: eye sub-path rules (camera vertex, unit-density primary hit)
  int per_pass;      // > 0: paths of several passes back to back (pool walks of a Stage-1 batch)
};

// Ray queue: slot j holds a ray for path[j]; traversal writes hit_prim/hit_t per slot.
struct RayQueue {
  double4* ray;  // [cap*2]: (ox, oy, oz, dx), (dy, dz, tmax, 0)
  int* path;
  int* hit_prim;
  double* hit_t;
  int* count;
  int cap;
};

__device__ __forceinline__ Rng path_rng(const PathSet& P, int i) {
  Rng r;
  const uint64_t q = P.per_pass > 0 ? static_cast<uint64_t>(i / P.per_pass) : 0;
  const uint64_t w = P.per_pass > 0 ? static_cast<uint64_t>(i % P.per_pass) : static_cast<uint64_t>(i);
  r.r = pxg_rng_make(P.seed, P.kind, 0, P.stream_base + (q << 32) + w);
  r.r.i = P.ctr[i];
  return r;
}

__device__ __forceinline__ void push_ray(const RayQueue& Q, int path, const V3& o, const V3& d, double tmax) {
  const int slot = atomicAdd(Q.count, 1);
  Q.ray[2 * slot] = make_double4(o.x, o.y, o.z, d.x);
  Q.ray[2 * slot + 1] = make_double4(d.y, d.z, tmax, 0.0);
  Q.path[slot] = path;
}

// trace_eye_subpath start (transport.cpp:137-152) of path i: camera vertex + jittered pixel
// ray. Returns true with the first ray in (o, d) unless the sub-path ends here.
__device__ __forceinline__ bool eye_start_one(const SceneView& S, const PathSet& P, int i, int row0, V3& o, V3& d) {
  PV z0;
  z0.p = S.cam_pos;
  z0.n = v3(0.0);
  z0.wi = v3(0.0);
  z0.flag = kCamera;
  z0.pdf_fwd = 1.0;
  z0.thr = v3(1.0);
  z0.mat = -1;
  z0.prim = -1;
  z0.emitter = -1;
  z0.pad = 0.0;
  P.pool[i] = z0;
  P.nv[i] = 1;
  if (P.max_vertices == 1) return false;
  Rng rng = path_rng(P, i);
  const int idx = row0 * S.width + i;
  const int x = idx % S.width, y = idx / S.width;
  // generate_ray's two rng arguments are evaluated right to left by the reference build
  const double jv = rng.next_double();
  const double ju = rng.next_double();
  const V3 dir = camera_dir(S, x, y, ju, jv);
  P.ctr[i] = rng.r.i;
  P.beta[3 * i] = 1.0;
  P.beta[3 * i + 1] = 1.0;
  P.beta[3 * i + 2] = 1.0;
  P.pdf_dir[i] = 1.0;
  o = S.cam_pos;
  d = dir;
  return true;
}

__global__ void k_eye_start(SceneView S, PathSet P, RayQueue Q, int row0) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  V3 o, d;
  if (eye_start_one(S, P, i, row0, o, d)) push_ray(Q, i, o, d, 1e30);
}

// trace_light_subpath start (transport.cpp:111-135) of path i: area-sampled emitter point
// and a cosine direction. Returns true with the first ray in (o, d).
__device__ __forceinline__ bool light_start_one(const SceneView& S, const PathSet& P, int i, V3& o, V3& d) {
  P.nv[i] = 0;
  if (P.max_vertices < 1) return false;
  Rng rng = path_rng(P, i);
  LightPoint lp = sample_light_point(S, rng);
  PV y0;
  y0.p = lp.p;
  y0.n = lp.n;
  y0.wi = v3(0.0);
  y0.mat = S.prim_mat[lp.prim];
  y0.prim = lp.prim;
  y0.emitter = S.prim_emitter[lp.prim];
  y0.flag = kLight;
  y0.pdf_fwd = lp.pdf_area;
  y0.thr = v3(1.0 / lp.pdf_area);
  y0.pad = 0.0;
  P.pool[i] = y0;
  P.nv[i] = 1;
  if (P.max_vertices == 1) {
    P.ctr[i] = rng.r.i;
    return false;
  }
  V3 dir = sample_cosine_hemisphere(lp.n, rng);
  P.ctr[i] = rng.r.i;
  double pdf_dir = light_direction_pdf(lp.n, dir);
  if (pdf_dir <= 0.0) return false;
  V3 beta = y0.thr * lp.radiance * (dot(dir, lp.n) / pdf_dir);
  P.beta[3 * i] = beta.x;
  P.beta[3 * i + 1] = beta.y;
  P.beta[3 * i + 2] = beta.z;
  P.pdf_dir[i] = pdf_dir;
  o = lp.p;
  d = dir;
  return true;
}

__global__ void k_light_start(SceneView S, PathSet P, RayQueue Q) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n) return;
  V3 o, d;
  if (light_start_one(S, P, i, o, d)) push_ray(Q, i, o, d, 1e30);
}

// One bounce of extend_walk (transport.cpp:37-56) for path i whose ray (o, d) hit `prim` at
// t (prim >= 0): writes the vertex, samples the BSDF; true with the next ray in (no, nd).
__device__ __forceinline__ bool shade_one(const SceneView& S, const PathSet& P, int i, const V3& o, const V3& d,
                                          int prim, double t, V3& no, V3& nd) {
  Hit hit;
  hit.t = t;
  hit.p = o + t * d;
  hit.prim = prim;
  hit.n = prim_normal(S, prim, hit.p);
  hit.material = S.prim_mat[prim];
  hit.emitter = S.prim_emitter[prim];
  PV v = surface_vertex(S, hit, -d);
  const int n = P.nv[i];
  const bool primary = P.eye && n == 1;
  V3 beta = v3(P.beta[3 * i], P.beta[3 * i + 1], P.beta[3 * i + 2]);
  if (primary) {
    v.pdf_fwd = 1.0;
    v.thr = v3(1.0);
  } else {
    v.pdf_fwd = to_area_density(P.pdf_dir[i], o, v.p, v.n);
    v.thr = beta;
  }
  P.pool[static_cast<size_t>(n) * P.n + i] = v;
  P.nv[i] = n + 1;
  if (n + 1 >= P.max_vertices) return false;
  Rng rng = path_rng(P, i);
  BsdfSample bs = sample_bsdf(S.materials[v.mat], v.n, v.wi, rng);
  P.ctr[i] = rng.r.i;
  if (!bs.valid || bs.pdf <= 0.0) return false;
  beta = beta * bs.value * (fabs(dot(bs.wo, v.n)) / bs.pdf);
  // extend_walk checks the throughput after each of its own samples; the eye walk's first
  // sample (at the primary hit, transport.cpp:160-163) is not checked
  if (!primary && near_zero(beta)) return false;
  P.beta[3 * i] = beta.x;
  P.beta[3 * i + 1] = beta.y;
  P.beta[3 * i + 2] = beta.z;
  P.pdf_dir[i] = bs.pdf;
  no = v.p;
  nd = bs.wo;
  return true;
}

// One bounce of extend_walk (transport.cpp:37-56) for the rays of queue `in`.
// The block's rays are first regrouped by the lobe set of the material they hit (diffuse /
// metal / dielectric and their mixtures; escaped rays last) with a shared-memory counting
// sort, so a warp samples and evaluates one kind of BSDF instead of serialising all of them
// (ncu, C4: pxg_bsdf.cuh ran at 7.3 of 32 lanes with the queue order). Every path keeps its
// own Philox stream and vertex slots, so the grouping cannot change a result.
#ifndef PXG_SHADE_T
#define PXG_SHADE_T 512  // threads per block = rays regrouped together (256: C4 -1.2%, 1024: = on C4, -1% on C2)
#endif
#ifndef PXG_SHADE_MINB
#define PXG_SHADE_MINB 2  // 64 registers: 1024 resident threads per SM (1280 / 1536: -1.8% / -3.1% from spills)
#endif
#ifndef PXG_SHADE_SORT
#define PXG_SHADE_SORT 1
#endif
__global__ void __launch_bounds__(PXG_SHADE_T, PXG_SHADE_MINB) k_shade(SceneView S, PathSet P, RayQueue in,
                                                                       RayQueue out) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int count = *in.count;
#if PXG_SHADE_SORT
  __shared__ int s_cnt[8];
  __shared__ short s_perm[PXG_SHADE_T];
  const int j0 = blockIdx.x * blockDim.x;
  if (j0 >= count) return;  // block-uniform
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  int cls = 7;  // escaped or past the end of the queue
  if (j < count) {
    const int prim = in.hit_prim[j];
    if (prim >= 0) {
      const Material& m = S.materials[S.prim_mat[prim]];
      double wd, wm, wt;
      lobes(m, wd, wm, wt);
      cls = ((wd > 0.0) ? 1 : 0) | ((wm > 0.0) ? 2 : 0) | ((wt > 0.0) ? 4 : 0);
      cls = cls == 0 ? 6 : cls - 1;  // 0..6: the seven lobe sets
    }
  }
  const int pos = atomicAdd(&s_cnt[cls], 1);
  __syncthreads();
  int base = 0;
#pragma unroll
  for (int k = 0; k < 7; ++k)
    if (k < cls) base += s_cnt[k];
  s_perm[base + pos] = static_cast<short>(threadIdx.x);
  const int live = blockDim.x - s_cnt[7];
  __syncthreads();
  if (static_cast<int>(threadIdx.x) >= live) return;
  j = j0 + s_perm[threadIdx.x];
#else
  if (j >= count) return;
#endif
  const int i = in.path[j];
  const int prim = in.hit_prim[j];
  if (prim < 0) return;  // escaped
  const double4 r0 = in.ray[2 * j], r1 = in.ray[2 * j + 1];
  V3 no, nd;
  if (shade_one(S, P, i, v3(r0.x, r0.y, r0.z), v3(r0.w, r1.x, r1.y), prim, in.hit_t[j], no, nd))
    push_ray(out, i, no, nd, 1e30);
}

// ---- two-kernel form of the regrouping (PXG_SHADE_PERM): k_shade_order computes the same
// class order per tile of kOrderT rays and writes it to HBM (perm[tile base + rank] = queue slot,
// -1 past the live rays), k_shade_perm shades in that order with small blocks, so a block's
// registers are released when ITS warps are done instead of when the slowest warp of a
// 512-thread tile is (ncu: k_shade at 26% achieved occupancy of a theoretical 50%).
constexpr int kOrderT = 1024;
__global__ void __launch_bounds__(kOrderT) k_shade_order(SceneView S, RayQueue in, int* perm) {
  __shared__ int s_cnt[8];
  const int count = *in.count;
  const int j0 = blockIdx.x * kOrderT;
  if (j0 >= count) return;  // block-uniform
  const int j = j0 + threadIdx.x;
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  int cls = 7;  // escaped or past the end of the queue
  if (j < count) {
    const int prim = in.hit_prim[j];
    if (prim >= 0) {
      const Material& m = S.materials[S.prim_mat[prim]];
      double wd, wm, wt;
      lobes(m, wd, wm, wt);
      cls = ((wd > 0.0) ? 1 : 0) | ((wm > 0.0) ? 2 : 0) | ((wt > 0.0) ? 4 : 0);
      cls = cls == 0 ? 6 : cls - 1;
    }
  }
  const int pos = atomicAdd(&s_cnt[cls], 1);
  __syncthreads();
  int base = 0;
#pragma unroll
  for (int k = 0; k < 7; ++k)
    if (k < cls) base += s_cnt[k];
  perm[j0 + base + pos] = cls < 7 ? j : -1;
}

#ifndef PXG_SHADE_PERM_MINB
#define PXG_SHADE_PERM_MINB 8
#endif
__global__ void __launch_bounds__(128, PXG_SHADE_PERM_MINB) k_shade_perm(SceneView S, PathSet P, RayQueue in,
                                                                         RayQueue out, const int* perm) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int count = *in.count;
  if ((t & ~(kOrderT - 1)) >= count) return;  // the tile was not ordered (past the queue)
  const int j = perm[t];
  if (j < 0) return;
  const int i = in.path[j];
  const double4 r0 = in.ray[2 * j], r1 = in.ray[2 * j + 1];
  V3 no, nd;
  if (shade_one(S, P, i, v3(r0.x, r0.y, r0.z), v3(r0.w, r1.x, r1.y), in.hit_prim[j], in.hit_t[j], no, nd))
    push_ray(out, i, no, nd, 1e30);
}

// Closest hit over a queue (Scene::intersect semantics, scene.cpp:127-168).
__global__ void __launch_bounds__(128) k_closest(SceneView S, RayQueue Q) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= *Q.count) return;
  const double4 r0 = Q.ray[2 * j], r1 = Q.ray[2 * j + 1];
  double t_best = r1.z;
  const int prim = trace_closest(S, v3(r0.x, r0.y, r0.z), v3(r0.w, r1.x, r1.y), t_best);
  Q.hit_prim[j] = prim;
  Q.hit_t[j] = t_best;
}

// Any hit over a queue (the boolean of Scene::occluded, scene.cpp:170-177): hit_prim = 1
// when occluded.
__global__ void __launch_bounds__(128) k_anyhit(SceneView S, RayQueue Q) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= *Q.count) return;
  const double4 r0 = Q.ray[2 * j], r1 = Q.ray[2 * j + 1];
  Q.hit_prim[j] = trace_any(S, v3(r0.x, r0.y, r0.z), v3(r0.w, r1.x, r1.y), r1.z) ? 1 : 0;
}

// ---------------------------------------------------------------- persistent traversal
// One BVH node step per loop iteration; a lane whose ray finishes takes the next ray of the
// queue (warp-aggregated atomic fetch) instead of idling until the warp's longest ray is
// done (ncu on the one-ray-per-thread kernel: 4.8-7.8 of 32 lanes active). The node step is
// exactly the loop body of trace_closest_t / trace_any_t, so results are identical.
struct TravState {
  V3 o, d;
  RayF rf;
  double t_best;
  int best, node, sp;
  int pend_node;        // postponed leaf tests (PXG_POSTPONE): the node whose hit leaf children ...
  unsigned pend_mask;   // ... bit k: child k still to be tested
};  // the traversal stack is a separate local array so these stay in registers

__device__ __forceinline__ void trav_init(TravState& ts, const RayQueue& Q, int j) {
  const double4 r0 = Q.ray[2 * j], r1 = Q.ray[2 * j + 1];
  ts.o = v3(r0.x, r0.y, r0.z);
  ts.d = v3(r0.w, r1.x, r1.y);
  ts.rf = make_rayf(ts.o, ts.d);
  ts.t_best = r1.z;
  ts.best = -1;
  ts.node = 0;
  ts.sp = 0;
  ts.pend_node = 0;
  ts.pend_mask = 0u;
}

// Returns true when the traversal is complete (closest hit in ts.best / ts.t_best).
// ts.node holds a child code: >= 0 a 4-wide node, < 0 a leaf.
template <bool kCount = false, int kL = -1, class Stack>
__device__ __forceinline__ bool closest_step(const SceneView& S, TravState& ts, Stack& stack, TravCount* cnt = nullptr) {
  // every step visits one 4-wide node; its hit leaf children are tested right away, its hit
  // inner children are ordered nearest-first (the next node, then the stack)
  const Node4Hits h = node4_test<true, kL>(S, ts.node, ts.rf, tbound_f(ts.t_best));
  if (kCount) cnt->nodes += 1;
  for (unsigned leaves = node4_leaves(h); leaves; leaves &= leaves - 1) {
    const int code = ~node4_code(h, __ffs(leaves) - 1);
    const int first = code >> 4, count = code & 15;
    if (kCount) cnt->prims += count;
    for (int i = 0; i < count; ++i) {
      int id;
      const double t = rec_hit(S, first + i, ts.o, ts.d, ts.t_best, id);
      if (t > 0.0 && (t < ts.t_best || id > ts.best)) {
        ts.t_best = t;
        ts.best = id;
      }
    }
  }
  int next = node4_order(node4_inner(h), tbound_f(ts.t_best), stack, ts.sp);
  if (next == kNoChild) {
    if (ts.sp == 0) return true;
    next = stack.pop(ts.sp);
  }
  ts.node = next;
  return false;
}

// Returns 0 while running, 1 on a hit in [kRayEps, tmax] (occluded), 2 when no hit.
template <bool kCount = false, int kL = -1, class Stack>
__device__ __forceinline__ int any_step(const SceneView& S, TravState& ts, Stack& stack, TravCount* cnt = nullptr) {
  const float tb = tbound_f(ts.t_best);
  const Node4Hits h = node4_test<true, kL>(S, ts.node, ts.rf, tb);
  if (kCount) cnt->nodes += 1;
  for (unsigned leaves = node4_leaves(h); leaves; leaves &= leaves - 1) {
    const int code = ~node4_code(h, __ffs(leaves) - 1);
    const int first = code >> 4, count = code & 15;
    for (int i = 0; i < count; ++i) {
      int id;
      if (kCount) cnt->prims += 1;
      if (rec_hit(S, first + i, ts.o, ts.d, ts.t_best, id) > 0.0) return 1;
    }
  }
  int next = node4_order<true>(node4_inner(h), tb, stack, ts.sp);
  if (next == kNoChild) {
    if (ts.sp == 0) return 2;
    next = stack.pop(ts.sp);
  }
  ts.node = next;
  return 0;
}

#ifndef PXG_LEAF_ONE
#define PXG_LEAF_ONE 1  // a leaf phase tests ONE pending leaf per lane (0: all of a lane's; C4 -1.8%)
#endif
// ---- postponed leaf tests (Aila & Laine's "while-while" for the 4-wide node step): a node
// visit only records its hit leaf children; the fp64 primitive tests of the warp run
// together once most active lanes have some (or no lane can visit a node), instead of
// diverging against the node visits of the other lanes on every step. A leaf phase tests ONE
// pending leaf per lane, so its lanes stay together through the fp64 test; a lane with more
// waits for the next phase (testing all of a lane's leaves in one phase ran the 2nd-4th tests
// at 1-5 lanes). Same hits: the
// closest hit with the id tie rule and the any-hit boolean do not depend on the order in
// which primitives are tested; only culling uses a bound that is a few steps older.
constexpr int kDone = static_cast<int>(0x80000001u);  // ts.node once nothing is left to visit

template <int kL = -1>
__device__ __forceinline__ int4 node4_codes(const SceneView& S, int node) {
  if (PXG_NODEQ && (kL == 1 || (kL < 0 && S.nodeq))) return __ldg(reinterpret_cast<const int4*>(S.nodes4q + node) + 1);
  return __ldg(reinterpret_cast<const int4*>(S.nodes4 + node) + 6);
}

// Node visit: hit leaves postponed, the next node chosen (kDone when none is left).
template <int kL = -1, class Stack>
__device__ __forceinline__ void node_step_postponed(const SceneView& S, TravState& ts, Stack& stack, float tb) {
  const Node4Hits h = node4_test<true, kL>(S, ts.node, ts.rf, tb);
  ts.pend_node = ts.node;
  ts.pend_mask = node4_leaves(h);
  int next = node4_order<true>(node4_inner(h), tb, stack, ts.sp);
  if (next == kNoChild) next = ts.sp == 0 ? kDone : stack.pop(ts.sp);
  ts.node = next;
}

// The postponed leaves, closest hit.
template <int kL = -1>
__device__ __forceinline__ void leaf_step_closest(const SceneView& S, TravState& ts) {
  const int4 cc = node4_codes<kL>(S, ts.pend_node);
#if PXG_LEAF_ONE
  {  // one pending leaf per leaf phase: the lanes of a phase stay together through the fp64 test
    const int k = __ffs(ts.pend_mask) - 1;
    ts.pend_mask &= ts.pend_mask - 1;
    const int code = ~(k == 0 ? cc.x : k == 1 ? cc.y : k == 2 ? cc.z : cc.w);
    const int first = code >> 4, count = code & 15;
    for (int i = 0; i < count; ++i) {
      int id;
      const double t = rec_hit(S, first + i, ts.o, ts.d, ts.t_best, id);
      if (t > 0.0 && (t < ts.t_best || id > ts.best)) {
        ts.t_best = t;
        ts.best = id;
      }
    }
    return;
  }
#endif
  for (unsigned leaves = ts.pend_mask; leaves; leaves &= leaves - 1) {
    const int k = __ffs(leaves) - 1;
    const int code = ~(k == 0 ? cc.x : k == 1 ? cc.y : k == 2 ? cc.z : cc.w);
    const int first = code >> 4, count = code & 15;
    for (int i = 0; i < count; ++i) {
      int id;
      const double t = rec_hit(S, first + i, ts.o, ts.d, ts.t_best, id);
      if (t > 0.0 && (t < ts.t_best || id > ts.best)) {
        ts.t_best = t;
        ts.best = id;
      }
    }
  }
  ts.pend_mask = 0u;
}

// The postponed leaves, any hit: true when one of them is hit within tmax.
template <int kL = -1>
__device__ __forceinline__ bool leaf_step_any(const SceneView& S, TravState& ts) {
  const int4 cc = node4_codes<kL>(S, ts.pend_node);
#if PXG_LEAF_ONE
  const unsigned pm = ts.pend_mask & (0u - ts.pend_mask);  // the lowest pending leaf only
  ts.pend_mask &= ts.pend_mask - 1;
#else
  const unsigned pm = ts.pend_mask;
  ts.pend_mask = 0u;
#endif
  for (unsigned leaves = pm; leaves; leaves &= leaves - 1) {
    const int k = __ffs(leaves) - 1;
    const int code = ~(k == 0 ? cc.x : k == 1 ? cc.y : k == 2 ? cc.z : cc.w);
    const int first = code >> 4, count = code & 15;
    for (int i = 0; i < count; ++i) {
      int id;
      if (rec_hit(S, first + i, ts.o, ts.d, ts.t_best, id) > 0.0) return true;
    }
  }
  return false;
}

// ---- pending-leaf LIST (PXG_LEAFQ): a lane keeps up to kLeafQ postponed leaf codes in shared
// memory ([slot][thread]: conflict-free) and goes on visiting nodes while it has room for
// another node's four children, so a lane with one or two untested leaves no longer sits out
// the node phases, and a leaf phase finds more lanes with work. ts.pend_mask is the count.
#ifndef PXG_LEAFQ_N
#define PXG_LEAFQ_N 6  // list slots: a lane visits nodes with up to 2 leaves pending (5: -0.7%, 8: -0.5%, 12: -1.5%)
#endif
constexpr int kLeafQ = PXG_LEAFQ_N;
constexpr int kLeafQBlock = kLeafQ - 4;  // a lane with more pending leaves than this visits no node (a node adds <= 4)

template <int kL = -1, class Stack>
__device__ __forceinline__ void node_step_listed(const SceneView& S, TravState& ts, Stack& stack, float tb,
                                                 int* pend /* this thread's column, stride 128 */) {
  const Node4Hits h = node4_test<true, kL>(S, ts.node, ts.rf, tb);
  const unsigned leaves = node4_leaves(h);
  int np = static_cast<int>(ts.pend_mask);
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (leaves >> k & 1u) pend[(np++) * 128] = h.code[k];
  ts.pend_mask = static_cast<unsigned>(np);
  int next = node4_order<true>(node4_inner(h), tb, stack, ts.sp);
  if (next == kNoChild) next = ts.sp == 0 ? kDone : stack.pop(ts.sp);
  ts.node = next;
}

// Tests the most recently recorded pending leaf (the deepest, usually the nearest).
// Closest hit: updates ts.best / ts.t_best; any hit: returns true when hit within tmax.
template <bool kAny>
__device__ __forceinline__ bool leaf_step_listed(const SceneView& S, TravState& ts, const int* pend) {
  const int np = static_cast<int>(ts.pend_mask) - 1;
  ts.pend_mask = static_cast<unsigned>(np);
  const int code = ~pend[np * 128];
  const int first = code >> 4, count = code & 15;
  for (int i = 0; i < count; ++i) {
    int id;
    const double t = rec_hit(S, first + i, ts.o, ts.d, ts.t_best, id);
    if (kAny) {
      if (t > 0.0) return true;
    } else if (t > 0.0 && (t < ts.t_best || id > ts.best)) {
      ts.t_best = t;
      ts.best = id;
    }
  }
  return false;
}

// The whole warp traces its lanes' rays (lane inactive when !active) to completion with
// postponed leaf tests, no refill: the block-local reciprocal wavefront's compacted rays.
// Closest hit: ts.best / ts.t_best; any hit: returns true when occluded.
template <bool kAny, class Stack>
__device__ __forceinline__ bool warp_trace(const SceneView& S, TravState& ts, Stack& stack, bool active) {
  const unsigned FULL = 0xffffffffu;
  bool live = active, occ = false;
  for (;;) {
    const bool pend = live && ts.pend_mask != 0u;
    const unsigned ma = __ballot_sync(FULL, live), mp = __ballot_sync(FULL, pend);
    if (ma == 0u) break;
    if (mp != 0u && (mp == ma || 2 * __popc(mp) >= __popc(ma))) {
      if (pend) {
        if (kAny) {
          if (leaf_step_any(S, ts)) {
            occ = true;
            live = false;
          } else if (ts.pend_mask == 0u && ts.node == kDone) {
            live = false;
          }
        } else {
          leaf_step_closest(S, ts);
          if (ts.pend_mask == 0u && ts.node == kDone) live = false;
        }
      }
    } else if (live && !pend) {
      node_step_postponed(S, ts, stack, tbound_f(ts.t_best));
      if (ts.pend_mask == 0u && ts.node == kDone) live = false;
    }
  }
  return occ;
}

#ifndef PXG_LEAF_FRAC
#define PXG_LEAF_FRAC 12  // leaf phase once this many 32ths of the active lanes have leaves pending
#endif

#ifndef PXG_REFILL
#define PXG_REFILL 6  // idle lanes before a refill (4: -0.7%, 8: -0.1%, 12: -1.5% with the pending-leaf list)
#endif
#ifndef PXG_LEAFQ
#define PXG_LEAFQ 1  // per-lane list of pending leaves in shared memory (0: one node's leaves; C4 -3.1%)
#endif
#ifndef PXG_LEAFQ_FRAC
#define PXG_LEAFQ_FRAC 14  // leaf phase once this many 32ths of the active lanes hold leaves (12 / 16: -0.3%)
#endif
#ifndef PXG_TOS
#define PXG_TOS 0  // top of the traversal stack in a register (TosStack)
#endif
#ifndef PXG_SSTACK
#define PXG_SSTACK 0  // shared-memory entries of the persistent kernels' traversal stack (0: all local)
#endif
constexpr int kRefill = PXG_REFILL;  // refill a warp's idle lanes once at least this many are idle

// kMinB resident blocks per SM: 8 for scenes traversed with quantised nodes (C4/C5: more
// warps hide the longer node chains, +2.6%), 6 for L2-resident scenes (C2: +0.8%; 7 was the
// single compromise before).
// kPost: postponed leaf tests (+4% on C4's 1M-triangle scene, -0.3% on the L2-resident C2,
// so chosen per scene with the node layout).
template <bool kAny, int kMinB, bool kPost, int kL = -1>
__global__ void __launch_bounds__(128, kMinB) k_trav_persistent(SceneView S, RayQueue Q, int* next_ray) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int total = *Q.count;
  int j = -1;
  bool exhausted = false;
  TravState ts;
  float tb = 0.0f;  // tbound_f(ts.t_best) of the postponed-leaf path: changes only when a leaf test improves the hit
#if PXG_SSTACK > 0
  __shared__ int s_stack[PXG_SSTACK * 128];
  int stack_loc[kStack - PXG_SSTACK];
  SplitStack<PXG_SSTACK> stack{s_stack + threadIdx.x, stack_loc};
#elif PXG_TOS
  int stack_mem[kStack];
  TosStack stack{stack_mem, 0};
#else
  int stack_mem[kStack];
  LocalStack stack{stack_mem};
#endif
#if PXG_LEAFQ
  __shared__ int s_pend[kLeafQ * 128];
  int* const pend = s_pend + threadIdx.x;
#endif
  for (;;) {
    const bool idle = j < 0;
    unsigned m = __ballot_sync(FULL, idle);  // idle lanes; the active mask is its complement
    if (!exhausted && m && (__popc(m) >= kRefill || m == FULL)) {
      const int leader = __ffs(m) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(next_ray, __popc(m));
      base = __shfl_sync(FULL, base, leader);
      if (base + __popc(m) > total) exhausted = true;
      if (idle) {
        const int jj = base + __popc(m & ((1u << lane) - 1));
        if (jj < total) {
          j = jj;
          trav_init(ts, Q, j);
          tb = tbound_f(ts.t_best);
        }
      }
      m = __ballot_sync(FULL, j < 0);  // only a refill changes the mask before the step
    }
    if (m == FULL) {
      if (exhausted || total == 0) break;
      continue;
    }
#if PXG_LEAFQ
    if (kPost) {
      // leaf phase once enough active lanes hold untested leaves, or when no lane can visit a node
      const bool act = j >= 0;
      const int np = act ? static_cast<int>(ts.pend_mask) : 0;
      const bool can_node = act && ts.node != kDone && np <= kLeafQBlock;
      const unsigned ma = ~m, mp = __ballot_sync(FULL, np > 0), mn = __ballot_sync(FULL, can_node);
      const bool leaf_phase = mp != 0u && (mn == 0u || 32 * __popc(mp) >= PXG_LEAFQ_FRAC * __popc(ma));
      if (leaf_phase) {
        if (np > 0) {
          const bool hit = leaf_step_listed<kAny>(S, ts, pend);
          if (kAny) {
            if (hit) {
              Q.hit_prim[j] = 1;
              j = -1;
            }
          } else {
            tb = tbound_f(ts.t_best);
          }
        }
      } else if (can_node) {
        node_step_listed<kL>(S, ts, stack, tb, pend);
      }
      if (j >= 0 && ts.pend_mask == 0u && ts.node == kDone) {  // nothing left to test or visit
        if (kAny) {
          Q.hit_prim[j] = 0;
        } else {
          Q.hit_prim[j] = ts.best;
          Q.hit_t[j] = ts.t_best;
        }
        j = -1;
      }
    } else if (j >= 0) {
      if (kAny) {
        const int r = any_step<false, kL>(S, ts, stack);
        if (r) {
          Q.hit_prim[j] = r == 1 ? 1 : 0;
          j = -1;
        }
      } else if (closest_step<false, kL>(S, ts, stack)) {
        Q.hit_prim[j] = ts.best;
        Q.hit_t[j] = ts.t_best;
        j = -1;
      }
    }
#else
    if (kPost) {
    const bool act = j >= 0;
    const bool pend = act && ts.pend_mask != 0u;
    const unsigned ma = ~m, mp = __ballot_sync(FULL, pend);
    const bool leaf_phase = mp != 0u && (mp == ma || 32 * __popc(mp) >= PXG_LEAF_FRAC * __popc(ma));
    if (leaf_phase) {
      if (pend) {
        if (kAny) {
          if (leaf_step_any<kL>(S, ts)) {
            Q.hit_prim[j] = 1;
            j = -1;
          } else if (ts.pend_mask == 0u && ts.node == kDone) {
            Q.hit_prim[j] = 0;
            j = -1;
          }
        } else {
          leaf_step_closest<kL>(S, ts);
          tb = tbound_f(ts.t_best);
          if (ts.pend_mask == 0u && ts.node == kDone) {
            Q.hit_prim[j] = ts.best;
            Q.hit_t[j] = ts.t_best;
            j = -1;
          }
        }
      }
    } else if (act && !pend) {
      node_step_postponed<kL>(S, ts, stack, tb);
      if (ts.pend_mask == 0u && ts.node == kDone) {  // nothing left to test or visit
        if (kAny) {
          Q.hit_prim[j] = 0;
        } else {
          Q.hit_prim[j] = ts.best;
          Q.hit_t[j] = ts.t_best;
        }
        j = -1;
      }
    }
    } else if (j >= 0) {
      if (kAny) {
        const int r = any_step<false, kL>(S, ts, stack);
        if (r) {
          Q.hit_prim[j] = r == 1 ? 1 : 0;
          j = -1;
        }
      } else if (closest_step<false, kL>(S, ts, stack)) {
        Q.hit_prim[j] = ts.best;
        Q.hit_t[j] = ts.t_best;
        j = -1;
      }
    }
#endif
  }
}

// Instrumented copies of the traversal kernels for the roofline measurement: the same step
// functions on the same queue, counting node visits (pxg_node_bytes(ctx) each: 64 B quantised
// or 128 B 4-wide nodes) and primitive tests (80 B each). Launched after the timed launch; results
// are identical and discarded.
__global__ void __launch_bounds__(128) k_closest_count(SceneView S, RayQueue Q, unsigned long long* acc) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= *Q.count) return;
  TravState ts;
  int stack_mem[kStack];
  LocalStack stack{stack_mem};
  trav_init(ts, Q, j);
  TravCount c{0, 0};
  while (!closest_step<true>(S, ts, stack, &c)) {
  }
  atomicAdd(acc + 0, 1ull);
  atomicAdd(acc + 1, c.nodes);
  atomicAdd(acc + 2, c.prims);
}

__global__ void __launch_bounds__(128) k_anyhit_count(SceneView S, RayQueue Q, unsigned long long* acc) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= *Q.count) return;
  TravState ts;
  int stack_mem[kStack];
  LocalStack stack{stack_mem};
  trav_init(ts, Q, j);
  TravCount c{0, 0};
  while (any_step<true>(S, ts, stack, &c) == 0) {
  }
  atomicAdd(acc + 0, 1ull);
  atomicAdd(acc + 1, c.nodes);
  atomicAdd(acc + 2, c.prims);
}

// ---------------------------------------------------------------- standard connections
// Slot layout per pixel, in the reference's accumulation order (proxy.cpp:627-641):
// for t = 2..n_eye: s = 0 (eye-hit emission), then s = 1..min(n_light, max_depth+1-t).
__device__ __forceinline__ int conn_slots(int ne, int nl, int max_depth) {
  int c = 0;
  for (int t = 2; t <= ne; ++t) c += 1 + min(nl, max_depth + 1 - t);
  return c;
}

struct ConnBuf {
  int* count;      // [n_px] slots per pixel
  int* offset;     // [n_px + 1] exclusive prefix
  int2* desc;      // [slot] pixel, t << 8 | s
  double* value;   // [slot*3]
  int* state;      // [slot] 0 nothing, 1 contributes, 2 waiting for visibility
  int* total;      // device scalar: number of slots
  int* live;       // [slot] compacted list of slots whose value needs the MIS weight
  int* n_live;     // device scalar
};

__global__ void k_conn_count(const int* n_eye, const int* n_light, int n, int max_depth, int* count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  count[i] = conn_slots(n_eye[i], n_light[i], max_depth);
}

__global__ void k_conn_enum(const int* n_eye, const int* n_light, int n, int max_depth, ConnBuf C) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int o = C.offset[i];
  const int ne = n_eye[i], nl = n_light[i];
  for (int t = 2; t <= ne; ++t) {
    const int smax = min(nl, max_depth + 1 - t);
    for (int s = 0; s <= smax; ++s) C.desc[o++] = make_int2(i, (t << 8) | s);
  }
  if (i == n - 1) *C.total = o;
}

// Unoccluded value of every slot; connections that need a shadow ray are queued.
__device__ __forceinline__ void conn_eval_one(const SceneView& S, const PV* eye, const PV* light, int n,
                                              const ConnBuf& C, const RayQueue& shadow, int g) {
  const int2 dsc = C.desc[g];
  const int i = dsc.x, t = dsc.y >> 8, s = dsc.y & 255;
  const size_t st = static_cast<size_t>(n);
  V3 val = v3(0.0);
  int state = 0;
  if (s == 0) {
    const PV& z = eye[(t - 1) * st + i];
    if (z.emitter >= 0) {
      val = z.thr * emitted(S, z.emitter, z.n, z.wi);
      if (!near_zero(val)) state = 1;
    }
  } else {
    // connection_contribution (transport.cpp:187-196) with the visibility deferred
    const PV& y = light[(s - 1) * st + i];
    const PV& z = eye[(t - 1) * st + i];
    if (z.flag == kDiffuse) {
      V3 d = z.p - y.p;
      double len = length(d);
      if (len > 0.0) {
        V3 dir = d / len;
        V3 f_light = v3(0.0);
        bool ok = true;
        if (s == 1) {
          f_light = emitted(S, y.emitter, y.n, dir);
        } else if (y.flag != kDiffuse) {
          ok = false;
        } else {
          f_light = eval_bsdf(S.materials[y.mat], y.n, y.wi, dir);
        }
        if (ok) {
          V3 f_eye = eval_bsdf(S.materials[z.mat], z.n, z.wi, -dir);
          if (!near_zero(f_light) && !near_zero(f_eye)) {
            // geometry_term (transport.cpp:168-176) without the visibility factor
            V3 dd = z.p - y.p;
            double dist2 = dot(dd, dd);
            double gg = 0.0;
            if (dist2 > 0.0) {
              V3 gdir = dd / sqrt(dist2);
              gg = fabs(dot(y.n, gdir)) * fabs(dot(z.n, gdir)) / dist2;
            }
            if (gg > 0.0) {
              val = y.thr * f_light * gg * f_eye * z.thr;
              // Scene::occluded(y.p, z.p)
              V3 sd = z.p - y.p;
              double dist = length(sd);
              if (dist < kRayEps) {
                state = 1;
              } else {
                state = 2;
                const int q = atomicAdd(shadow.count, 1);
                const V3 sdir = sd / dist;
                shadow.ray[2 * q] = make_double4(y.p.x, y.p.y, y.p.z, sdir.x);
                shadow.ray[2 * q + 1] = make_double4(sdir.y, sdir.z, dist * (1.0 - 1e-6), 0.0);
                shadow.path[q] = g;
              }
            }
          }
        }
      }
    }
  }
  C.value[3 * g] = val.x;
  C.value[3 * g + 1] = val.y;
  C.value[3 * g + 2] = val.z;
  C.state[g] = state;
  if (state == 1) C.live[atomicAdd(C.n_live, 1)] = g;
}

// Grid-stride over the enumerated slots (a fixed grid instead of one thread per possible slot:
// most of the n x max_slots threads would only read the count and exit).
#ifndef PXG_EVAL_MINB
#define PXG_EVAL_MINB 8
#endif
__global__ void __launch_bounds__(128, PXG_EVAL_MINB) k_conn_eval(SceneView S, const PV* eye, const PV* light, int n, ConnBuf C, RayQueue shadow) {
  const int total = *C.total;
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < total; g += gridDim.x * blockDim.x)
    conn_eval_one(S, eye, light, n, C, shadow, g);
}

__global__ void k_conn_visibility(RayQueue shadow, ConnBuf C) {
  const int count = *shadow.count;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < count; q += gridDim.x * blockDim.x) {
    const int g = shadow.path[q];
    const int vis = shadow.hit_prim[q] ? 0 : 1;  // occluded -> no contribution
    C.state[g] = vis;
    if (vis) C.live[atomicAdd(C.n_live, 1)] = g;
  }
}

// Per-pixel sub-path step densities (PathCache), evaluated once per pixel and pass.
// One thread per (pixel, sub-path): 2 n threads, each walking a window of three consecutive
// vertices and writing both directions (LF + LR on the light sub-path, ER + EF on the eye
// sub-path); the light thread also writes the light-direction density. (Round 1: one thread per
// (pixel, family), 4 n threads, which read every vertex from HBM twice.)
#ifndef PXG_PF_MINB
#define PXG_PF_MINB 8
#endif
#ifndef PXG_PF_MERGE
#define PXG_PF_MERGE 1  // one thread per (pixel, sub-path) computing both directions (0: per family; C4 -0.7%)
#endif
__global__ void __launch_bounds__(128, PXG_PF_MINB) k_path_factors(SceneView S, const PV* eye, const int* n_eye, const PV* light, const int* n_light,
                               int n, PathCache C) {
  const long long tid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
#if PXG_PF_MERGE
  // one thread per (pixel, sub-path): the forward and the reverse step density of a window of
  // three consecutive vertices (lo, mid, hi) are bsdf_step_v(mid, lo, hi) and
  // bsdf_step_v(mid, hi, lo): LF[w + 2] / LR[w] on the light sub-path, ER[w + 2] / EF[w] on the
  // eye sub-path, so both directions share the window's loads (the per-family threads read
  // every vertex from HBM twice: ncu, 7.6 GB per launch)
  if (tid >= 2ll * n) return;
  {
    const int i = static_cast<int>(tid % n), sub = static_cast<int>(tid / n);
    const size_t st = static_cast<size_t>(n);
    const PV* v = (sub ? eye : light) + i;
    const int cnt = sub ? n_eye[i] : n_light[i];
    double* fwd = sub ? C.ER : C.LF;
    double* rev = sub ? C.EF : C.LR;
    for (int w = 0; w <= cnt - 3; ++w) {
      const PV& lo = v[w * st];
      const PV& mid = v[(w + 1) * st];
      const PV& hi = v[(w + 2) * st];
      const double a = bsdf_step_v(S, mid, lo, hi);
      const double b = bsdf_step_v(S, mid, hi, lo);
      fwd[(w + 2) * st + i] = a;
      rev[w * st + i] = b;
    }
    if (sub) return;
    int ok = 0;
    double area = 0.0;
    if (cnt >= 2) {
      const PV& y0 = v[0];
      const PV& y1 = v[st];
      V3 d = y1.p - y0.p;
      double len = length(d);
      if (len > 0.0) {
        double pdf_w = light_direction_pdf(y0.n, d / len);
        if (pdf_w > 0.0) {
          ok = 1;
          area = to_area_density(pdf_w, y0.p, y1.p, y1.n);
        }
      }
    }
    C.ld_ok[i] = ok;
    C.ld[i] = area;
    return;
  }
#endif
  if (tid >= 4ll * n) return;
  const int i = static_cast<int>(tid % n), fam = static_cast<int>(tid / n);
  const size_t st = static_cast<size_t>(n);
  const PV* y = light + i;
  const PV* e = eye + i;
  if (fam == 1) {
    const int nl = n_light[i];
    for (int j = 0; j <= nl - 3; ++j) C.LR[j * st + i] = bsdf_step_v(S, y[(j + 1) * st], y[(j + 2) * st], y[j * st]);
    return;
  }
  if (fam == 2) {
    const int ne = n_eye[i];
    for (int m = 0; m <= ne - 3; ++m) C.EF[m * st + i] = bsdf_step_v(S, e[(m + 1) * st], e[(m + 2) * st], e[m * st]);
    return;
  }
  if (fam == 3) {
    const int ne = n_eye[i];
    for (int m = 2; m <= ne - 1; ++m) C.ER[m * st + i] = bsdf_step_v(S, e[(m - 1) * st], e[(m - 2) * st], e[m * st]);
    return;
  }
  const int nl = n_light[i];
  for (int k = 2; k <= nl - 1; ++k) C.LF[k * st + i] = bsdf_step_v(S, y[(k - 1) * st], y[(k - 2) * st], y[k * st]);
  int ok = 0;
  double area = 0.0;
  if (nl >= 2) {
    const PV& y0 = y[0];
    const PV& y1 = y[st];
    V3 d = y1.p - y0.p;
    double len = length(d);
    if (len > 0.0) {
      double pdf_w = light_direction_pdf(y0.n, d / len);
      if (pdf_w > 0.0) {
        ok = 1;
        area = to_area_density(pdf_w, y0.p, y1.p, y1.n);
      }
    }
  }
  C.ld_ok[i] = ok;
  C.ld[i] = area;
}

// Per pixel, one warp: stage the pixel's eye and light vertices in shared memory, compute
// the per-sub-path step caches with the lanes, weight every contributing slot
// (reciprocal_mis_weight, proxy.cpp:533-546) with the lanes, then lane 0 accumulates the
// slots in the reference's (t, s) order (proxy.cpp:627-641) into bdpt[i].
constexpr int kConnWarps = 4;
constexpr int kMaxEye = 17;    // max_depth + 1
constexpr int kMaxSlots = 136; // sum over t of (1 + min(n_light, max_depth + 1 - t)) at max_depth 16

// Vertices are stored at a 144-byte stride (not 128): with 128 B every lane reading the
// same field of a different vertex hits the same shared-memory bank.
constexpr int kSmemVtx = 144;
struct ConnSmem {
  alignas(16) char eye[kMaxEye * kSmemVtx];
  alignas(16) char light[kMaxLight * kSmemVtx];
  double LF[kMaxPath], LR[kMaxPath], EF[kMaxPath], ER[kMaxPath];
  double val[kMaxSlots * 3];
  double ld;
  int ld_ok;
};

__global__ void __launch_bounds__(32 * kConnWarps) k_conn_pixel(SceneView S, Mapper M, StatsView st, int use_stats,
                                                                const PV* eye, const int* n_eye, const PV* light,
                                                                const int* n_light, int n, ConnBuf C,
                                                                double* bdpt) {
  __shared__ ConnSmem sm_all[kConnWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int i = blockIdx.x * kConnWarps + wid;
  if (i >= n) return;
  ConnSmem& sm = sm_all[wid];
  const size_t stv = static_cast<size_t>(n);
  const int ne = n_eye[i], nl = n_light[i];
  // stage vertices (16 B per lane per step, coalesced within a vertex)
  for (int k = 0; k < ne; ++k) {
    const double2* src = reinterpret_cast<const double2*>(eye + k * stv + i);
    double2* dst = reinterpret_cast<double2*>(sm.eye + k * kSmemVtx);
    if (lane < 8) dst[lane] = src[lane];
  }
  for (int k = 0; k < nl; ++k) {
    const double2* src = reinterpret_cast<const double2*>(light + k * stv + i);
    double2* dst = reinterpret_cast<double2*>(sm.light + k * kSmemVtx);
    if (lane < 8) dst[lane] = src[lane];
  }
  __syncwarp();
  // per-sub-path step densities (same values as PathCache / k_path_factors)
  const int nLF = nl > 2 ? nl - 2 : 0, nLR = nl > 2 ? nl - 2 : 0;
  const int nEF = ne > 2 ? ne - 2 : 0, nER = ne > 2 ? ne - 2 : 0;
  auto EV = [&](int k) -> const PV& { return *reinterpret_cast<const PV*>(sm.eye + k * kSmemVtx); };
  auto LV = [&](int k) -> const PV& { return *reinterpret_cast<const PV*>(sm.light + k * kSmemVtx); };
  for (int q = lane; q < nLF + nLR + nEF + nER; q += 32) {
    if (q < nLF) {
      const int k = q + 2;
      sm.LF[k] = bsdf_step_v(S, LV(k - 1), LV(k - 2), LV(k));
    } else if (q < nLF + nLR) {
      const int j = q - nLF;
      sm.LR[j] = bsdf_step_v(S, LV(j + 1), LV(j + 2), LV(j));
    } else if (q < nLF + nLR + nEF) {
      const int m = q - nLF - nLR;
      sm.EF[m] = bsdf_step_v(S, EV(m + 1), EV(m + 2), EV(m));
    } else {
      const int m = q - nLF - nLR - nEF + 2;
      sm.ER[m] = bsdf_step_v(S, EV(m - 1), EV(m - 2), EV(m));
    }
  }
  if (lane == 0) {
    int ok = 0;
    double area = 0.0;
    if (nl >= 2) {
      const PV& y0 = LV(0);
      const PV& y1 = LV(1);
      V3 d = y1.p - y0.p;
      double len = length(d);
      if (len > 0.0) {
        double pdf_w = light_direction_pdf(y0.n, d / len);
        if (pdf_w > 0.0) {
          ok = 1;
          area = to_area_density(pdf_w, y0.p, y1.p, y1.n);
        }
      }
    }
    sm.ld = area;
    sm.ld_ok = ok;
  }
  __syncwarp();
  const int a = C.offset[i], b = C.offset[i + 1];
  for (int g = a + lane; g < b; g += 32) {
    const int state = C.state[g];
    double* out = &sm.val[3 * (g - a)];
    if (state != 1) {
      out[0] = out[1] = out[2] = 0.0;
      continue;
    }
    const int ts = C.desc[g].y;
    const int t = ts >> 8, s = ts & 255;
    FullPath fp{sm.light, kSmemVtx, sm.eye, kSmemVtx, s, t};
    PathTable T;
    table_init_local(T, sm.LF, sm.LR, sm.EF, sm.ER, sm.ld, sm.ld_ok, s, t);
    const double w = reciprocal_mis_weight_t(S, M, st, fp, T, s, use_stats != 0);
    out[0] = C.value[3 * g] * w;
    out[1] = C.value[3 * g + 1] * w;
    out[2] = C.value[3 * g + 2] * w;
  }
  __syncwarp();
  if (lane == 0) {
    V3 r = v3(0.0);
    for (int g = a; g < b; ++g) {
      if (C.state[g] != 1) continue;
      const double* v = &sm.val[3 * (g - a)];
      r += v3(v[0], v[1], v[2]);
    }
    bdpt[3 * i] = r.x;
    bdpt[3 * i + 1] = r.y;
    bdpt[3 * i + 2] = r.z;
  }
}

// reciprocal_mis_weight of every live slot; value <- value * w.
#ifndef PXG_MIS_MINB
#define PXG_MIS_MINB 8
#endif
#if PXG_MIS_MINB
__global__ void __launch_bounds__(128, PXG_MIS_MINB) k_conn_mis(
#else
__global__ void k_conn_mis(
#endif
  SceneView S, Mapper M, StatsView st, int use_stats, const PV* eye, const PV* light,
                           int n, ConnBuf C, PathCache PC) {
  const int n_live = *C.n_live;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n_live; q += gridDim.x * blockDim.x) {
  const int g = C.live[q];
  const int2 dsc = C.desc[g];
  const int i = dsc.x, t = dsc.y >> 8, s = dsc.y & 255;
  const size_t st_ = static_cast<size_t>(n);
  FullPath fp = make_fp(light + i, st_, eye + i, st_, s, t);
  PathTable T;
  table_init_cached(T, PC, i, s, t);
  table_fill_junctions(S, fp, T);
  const double w = mis_weight_full(S, M, st, fp, T, s, use_stats != 0);
  C.value[3 * g] = C.value[3 * g] * w;
  C.value[3 * g + 1] = C.value[3 * g + 1] * w;
  C.value[3 * g + 2] = C.value[3 * g + 2] * w;
  }
}

// weighted_bdpt_value's accumulation (proxy.cpp:627-641) in slot order.
__global__ void k_conn_sum(int n, ConnBuf C, double* bdpt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  V3 r = v3(0.0);
  const int a = C.offset[i], b = C.offset[i + 1];
  for (int g = a; g < b; ++g) {
    if (C.state[g] != 1) continue;
    r += v3(C.value[3 * g], C.value[3 * g + 1], C.value[3 * g + 2]);
  }
  bdpt[3 * i] = r.x;
  bdpt[3 * i + 1] = r.y;
  bdpt[3 * i + 2] = r.z;
}

#endif  // __CUDACC__

}  // namespace pxg
