// pxg_scene.cuh — device scene, BVH traversal and light sampling.
//
// HBM layout (built once by pxg_create, see pxg_host.cpp):
//   nodes   BvhNode[n_nodes]   64 B: both child boxes in fp32 (outward-rounded and padded
//                              so the test is conservative w.r.t. the fp64 reference),
//                              child links; read as 4 x 16 B non-coherent vector loads.
//   tris    PrimRec[n_prims]   80 B, in BVH leaf order: fp64 a, e1, e2 (triangle:
//                              e1 = b-a, e2 = c-a; rectangle: e1 = b, e2 = c; sphere:
//                              a = centre, e1.x = radius) + shape + original primitive id.
//   prim_*  per original primitive id: material, emitter index, fp64 normal (tri/rect).
//
// Hit primitive ids equal the reference's Scene::intersect (proj/src/scene.cpp:127-168)
// because (1) the leaf test is the reference's fp64 Moller-Trumbore / sphere test op for
// op (--fmad=false), (2) the fp32 node test never culls a box that contains an accepted
// fp64 hit, and (3) equal-t ties go to the larger primitive id, which is the reference's
// own rule on its linear-scan path (later visited wins, scene.cpp:134-139).
#pragma once

#include "pxg_bsdf.cuh"

namespace pxg {

constexpr double kRayEps = 1e-7;  // scene.cpp:19
constexpr int kStack = 96;  // 4-wide BVH: up to 3 pushes per level

enum Shape { kSphere = 0, kTriangle = 1, kRectangle = 2 };

struct alignas(16) BvhNode {
  float lo0[3], hi0[3];
  float lo1[3], hi1[3];
  int c0, c1;  // >= 0 internal node, < 0 leaf: ~c = first*16 + count
  int pad0, pad1;
};

// 4-wide node (128 B): child boxes as SoA float4 (lo x, lo y, lo z, hi x, hi y, hi z) so a
// step is 7 independent 16-byte loads; child codes as in BvhNode.
struct alignas(32) BvhNode4 {
  float lo[3][4];
  float hi[3][4];
  int child[4];
  int pad[4];
};

// Quantised 4-wide node (64 B, two 32-byte loads): child planes on a per-node grid,
// plane = origin + q * 2^(e-127) per axis (q = byte k of qlo/qhi), rounded outward on the host
// so the decoded boxes contain the fp32 boxes of BvhNode4 (pxg_host.cpp quantize_node).
struct alignas(32) BvhNode4Q {
  float origin[3];
  unsigned exps;
  int child[4];
  unsigned qlo[3];
  unsigned qhi[3];
  unsigned pad[2];
};

struct alignas(16) PrimRec {
  double a[3];
  double e1[3];
  double e2[3];
  int shape;
  int id;
};

struct SceneView {
  const BvhNode* nodes;
  const BvhNode4* nodes4;
  const BvhNode4Q* nodes4q;
  int nodeq;  // persistent kernels use nodes4q (1) or nodes4 (0), chosen per scene in pxg_create
  const PrimRec* recs;
  const int* prim_mat;       // [n_prims]
  const int* prim_emitter;   // [n_prims] emitter index or -1
  const double* prim_geo;    // [n_prims][3] unit normal (tri/rect); sphere: unused
  const double* prim_center; // [n_prims][4] sphere centre + radius (shape 0 only)
  const int* prim_shape;     // [n_prims]
  const double* prim_abc;    // [n_prims][9] a, e1, e2 as in PrimRec, original order
  const Material* materials;
  const int* emitter_prim;   // [n_emit]
  const double* emitter_rad; // [n_emit][3]
  const double* emitter_cum; // [n_emit] running area sum (scene.cpp:183-189 order)
  int n_prims, n_emit, n_nodes, n_mat;
  double total_emitter_area;
  V3 bbox_min, bbox_max;
  // camera (scene.cpp:116-125, basis precomputed on the host with the same ops)
  V3 cam_pos, cam_fwd, cam_right, cam_up;
  double tan_half, aspect;
  int width, height, max_depth;
};

struct Hit {
  double t;
  V3 p, n;
  int prim, material, emitter;
};

// ---- exact fp64 primitive tests (scene.cpp:22-62) ----
PXD double sphere_hit(const double* c, double radius, const V3& o, const V3& d, double t_max) {
  V3 oc = o - v3(c[0], c[1], c[2]);
  double b = dot(oc, d);
  double cc = length_sq(oc) - radius * radius;
  double disc = b * b - cc;
  if (disc < 0.0) return -1.0;
  double sq = sqrt(disc);
  double t = -b - sq;
  if (t < kRayEps) t = -b + sq;
  if (t < kRayEps || t > t_max) return -1.0;
  return t;
}

PXD double triangle_hit(const V3& a, const V3& e1, const V3& e2, const V3& o, const V3& d,
                        double t_max, bool parallelogram) {
  V3 pv = cross(d, e2);
  double det = dot(e1, pv);
  if (fabs(det) < 1e-14) return -1.0;
  double inv = 1.0 / det;
  V3 tv = o - a;
  double u = dot(tv, pv) * inv;
  if (u < 0.0 || u > 1.0) return -1.0;
  V3 qv = cross(tv, e1);
  double v = dot(d, qv) * inv;
  double hi = parallelogram ? 1.0 : 1.0 - u;
  if (v < 0.0 || v > hi) return -1.0;
  double t = dot(e2, qv) * inv;
  if (t < kRayEps || t > t_max) return -1.0;
  return t;
}

#if defined(__CUDACC__)
// Primitive test of leaf-ordered record k: 5 x 16-byte loads (a split 64 B + 16 B layout with
// two 32-byte loads measured slower on C4, 26.9 vs 27.4 Msamples/s). The fp64 test is the
// reference's, op for op.
__device__ __forceinline__ double rec_hit(const SceneView& S, int k, const V3& o, const V3& d, double t_max,
                                          int& id) {
  const double2* q = reinterpret_cast<const double2*>(S.recs + k);
  const double2 w0 = __ldg(q + 0), w1 = __ldg(q + 1), w2 = __ldg(q + 2), w3 = __ldg(q + 3);
  const double2 w4 = __ldg(q + 4);
  const int2 si = *reinterpret_cast<const int2*>(&w4.y);
  const int shape = si.x;
  id = si.y;
  if (shape == kSphere) {
    const double c[3] = {w0.x, w0.y, w1.x};
    return sphere_hit(c, w1.y, o, d, t_max);
  }
  V3 a = v3(w0.x, w0.y, w1.x);
  V3 e1 = v3(w1.y, w2.x, w2.y);
  V3 e2 = v3(w3.x, w3.y, w4.x);
  return triangle_hit(a, e1, e2, o, d, t_max, shape == kRectangle);
}

struct RayF {
  float ox, oy, oz, ix, iy, iz;
  float nx, ny, nz;  // -o * inv(d) per axis: slab distance = fma(plane, inv, n)
};

__device__ __forceinline__ RayF make_rayf(const V3& o, const V3& d) {
  RayF r;
  r.ox = __double2float_rn(o.x);
  r.oy = __double2float_rn(o.y);
  r.oz = __double2float_rn(o.z);
  float dx = __double2float_rn(d.x), dy = __double2float_rn(d.y), dz = __double2float_rn(d.z);
  // a zero component becomes +-1e-30: no 0 * inf = NaN when the origin lies exactly on a
  // slab plane, and the slab is still effectively unbounded along that axis
  if (fabsf(dx) < 1e-30f) dx = copysignf(1e-30f, dx);
  if (fabsf(dy) < 1e-30f) dy = copysignf(1e-30f, dy);
  if (fabsf(dz) < 1e-30f) dz = copysignf(1e-30f, dz);
  r.ix = 1.0f / dx;
  r.iy = 1.0f / dy;
  r.iz = 1.0f / dz;
  r.nx = -r.ox * r.ix;
  r.ny = -r.oy * r.iy;
  r.nz = -r.oz * r.iz;
  return r;
}

// Slab test in fp32 (boxes padded outward on the host, directions never exactly zero).
__device__ __forceinline__ bool box_f(const float* lo, const float* hi, const RayF& r, float tmax,
                                      float& tnear) {
  // one FFMA per slab plane (explicit: the file is built with --fmad=false for the fp64
  // path math). The cancellation error of lo*inv - o*inv is ~|o| * 2^-24 along the ray,
  // far inside the boxes' 1e-5 x scene-scale padding, so the test stays conservative.
  float tx0 = __fmaf_rn(lo[0], r.ix, r.nx), tx1 = __fmaf_rn(hi[0], r.ix, r.nx);
  float ty0 = __fmaf_rn(lo[1], r.iy, r.ny), ty1 = __fmaf_rn(hi[1], r.iy, r.ny);
  float tz0 = __fmaf_rn(lo[2], r.iz, r.nz), tz1 = __fmaf_rn(hi[2], r.iz, r.nz);
  float t0 = fmaxf(fmaxf(fminf(tx0, tx1), fminf(ty0, ty1)), fmaxf(fminf(tz0, tz1), 0.0f));
  float t1 = fminf(fminf(fmaxf(tx0, tx1), fmaxf(ty0, ty1)), fminf(fmaxf(tz0, tz1), tmax));
  tnear = t0;
  return t0 <= t1;
}

// fp64 t bound -> fp32, rounded up with slack so the node test stays conservative.
__device__ __forceinline__ float tbound_f(double t) {
  if (t > 3.0e38) return 3.0e38f;
  return __double2float_ru(t) * 1.0000005f + 1e-30f;
}

// Traversal work counters (instrumented variant only): node visits and primitive tests.
struct TravCount {
  unsigned long long nodes, prims;
};

// One 4-wide node: box tests of the four children (fp32, conservative).
struct Node4Hits {
  float tn[4];
  int code[4];
  unsigned hit;    // bit k: child k's box is hit
  unsigned leafm;  // bit k: child k is a leaf (code < 0)
};

#ifndef PXG_NODE256
#define PXG_NODE256 1
#endif

// 32-byte non-coherent global load (sm_100: LDG.E.ENL2.256). Scattered node fetches are bound
// by the L1 data pipe's wavefronts, one per distinct line per load instruction, so fetching a
// node in 3 x 32 B + 1 x 16 B loads instead of 7 x 16 B cuts the pipe's work per visit.
__device__ __forceinline__ void ldg256(const void* p, float4& a, float4& b) {
  unsigned r0, r1, r2, r3, r4, r5, r6, r7;
  asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3), "=r"(r4), "=r"(r5), "=r"(r6), "=r"(r7)
               : "l"(p));
  a = make_float4(__uint_as_float(r0), __uint_as_float(r1), __uint_as_float(r2), __uint_as_float(r3));
  b = make_float4(__uint_as_float(r4), __uint_as_float(r5), __uint_as_float(r6), __uint_as_float(r7));
}

// kWide: 256-bit loads. Only the persistent traversal kernels use them: ptxas 12.9 crashes
// (segfault) when the v8 load sits in the __noinline__ trace_closest_t / trace_any_t shared
// by several kernels, so those keep the 128-bit loads.
#ifndef PXG_NODEQ
#define PXG_NODEQ 1
#endif

#ifndef PXG_QSIGN
#define PXG_QSIGN 1
#endif
#ifndef PXG_QCVT
#define PXG_QCVT 0
#endif
// Byte k of w as a float, exactly. PXG_QCVT 1: one byte permute builds the fp32 bit pattern
// 0x4B0000bb = 2^23 + b and one exact FADD removes 2^23 (two full-rate instructions instead
// of the quarter-rate I2F.U8).
__device__ __forceinline__ float qbyte(unsigned w, int k) {
#if PXG_QCVT == 2
  // byte k in mantissa bits 8-15 of 1.0f: 1 + q * 2^-15 exactly, one byte permute and no
  // conversion; node4q_test folds the offset into its slopes (A * 2^15, B - A * 2^15)
  return __uint_as_float(__byte_perm(w, 0x3F800000u, 0x7604u | (static_cast<unsigned>(k) << 4)));
#elif PXG_QCVT
  return __uint_as_float(__byte_perm(w, 0x4B000000u, static_cast<unsigned>(k) | 0x7540u)) - 8388608.0f;
#else
  return static_cast<float>((w >> (8 * k)) & 0xffu);
#endif
}

// Box tests of a quantised node: per axis t = q * (step * inv) + (origin - o) * inv, i.e. the
// slab distance of the decoded plane (one FFMA per plane after 2 per axis), conservative
// like box_f (the fp32 rounding is far inside the boxes' padding, see box_f).
// kWide: two 32-byte loads (persistent kernels); otherwise four 16-byte loads (the
// __noinline__ single-ray traversal, where ptxas 12.9 rejects the 32-byte form, see below).
template <bool kWide>
__device__ __forceinline__ Node4Hits node4q_test(const SceneView& S, int node, const RayF& rf, float tb) {
  float4 a, b, c, d;
  if (kWide) {
    ldg256(S.nodes4q + node, a, b);
    ldg256(reinterpret_cast<const char*>(S.nodes4q + node) + 32, c, d);
  } else {
    const float4* q = reinterpret_cast<const float4*>(S.nodes4q + node);
    a = __ldg(q + 0);
    b = __ldg(q + 1);
    c = __ldg(q + 2);
    d = __ldg(q + 3);
  }
  const unsigned ex = __float_as_uint(a.w);
  const float sx = __uint_as_float((ex & 0xffu) << 23), sy = __uint_as_float(((ex >> 8) & 0xffu) << 23),
              sz = __uint_as_float(((ex >> 16) & 0xffu) << 23);
#if PXG_QCVT == 2
  // q * A + B = (1 + q 2^-15) * (A 2^15) + (B - A 2^15); the second term's rounding moves a
  // plane by at most 1/512 of a grid step, inside the boxes' padding (pxg_host.cpp)
  const float Ax = sx * rf.ix * 32768.0f, Ay = sy * rf.iy * 32768.0f, Az = sz * rf.iz * 32768.0f;
  const float Bx = __fmaf_rn(a.x, rf.ix, rf.nx) - Ax, By = __fmaf_rn(a.y, rf.iy, rf.ny) - Ay,
              Bz = __fmaf_rn(a.z, rf.iz, rf.nz) - Az;
#else
  const float Ax = sx * rf.ix, Ay = sy * rf.iy, Az = sz * rf.iz;
  const float Bx = __fmaf_rn(a.x, rf.ix, rf.nx), By = __fmaf_rn(a.y, rf.iy, rf.ny), Bz = __fmaf_rn(a.z, rf.iz, rf.nz);
#endif
  const unsigned lxw = __float_as_uint(c.x), lyw = __float_as_uint(c.y), lzw = __float_as_uint(c.z);
  const unsigned hxw = __float_as_uint(c.w), hyw = __float_as_uint(d.x), hzw = __float_as_uint(d.y);
  Node4Hits r;
  r.hit = 0u;
  r.leafm = (ex >> 24) & 0xfu;  // written by the host quantiser (pxg_host.cpp quantize_node)
  r.code[0] = __float_as_int(b.x);
  r.code[1] = __float_as_int(b.y);
  r.code[2] = __float_as_int(b.z);
  r.code[3] = __float_as_int(b.w);
#if PXG_QSIGN
  // near / far planes picked once per node by the sign of the slope (fma(q, A, B) is monotone
  // in q, so this is exactly the min / max of the two slab distances): 3 + 3 distances and
  // two 3-input min / max per child instead of 6 two-input ones
  const unsigned nxw = Ax < 0.0f ? hxw : lxw, fxw = Ax < 0.0f ? lxw : hxw;
  const unsigned nyw = Ay < 0.0f ? hyw : lyw, fyw = Ay < 0.0f ? lyw : hyw;
  const unsigned nzw = Az < 0.0f ? hzw : lzw, fzw = Az < 0.0f ? lzw : hzw;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float nx = __fmaf_rn(qbyte(nxw, k), Ax, Bx), fx = __fmaf_rn(qbyte(fxw, k), Ax, Bx);
    const float ny = __fmaf_rn(qbyte(nyw, k), Ay, By), fy = __fmaf_rn(qbyte(fyw, k), Ay, By);
    const float nz = __fmaf_rn(qbyte(nzw, k), Az, Bz), fz = __fmaf_rn(qbyte(fzw, k), Az, Bz);
    const float t0 = fmaxf(fmaxf(nx, ny), fmaxf(nz, 0.0f));
    const float t1 = fminf(fminf(fx, fy), fminf(fz, tb));
    if (t0 <= t1) r.hit |= 1u << k;
    r.tn[k] = t0;
  }
#else
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float tx0 = __fmaf_rn(qbyte(lxw, k), Ax, Bx), tx1 = __fmaf_rn(qbyte(hxw, k), Ax, Bx);
    const float ty0 = __fmaf_rn(qbyte(lyw, k), Ay, By), ty1 = __fmaf_rn(qbyte(hyw, k), Ay, By);
    const float tz0 = __fmaf_rn(qbyte(lzw, k), Az, Bz), tz1 = __fmaf_rn(qbyte(hzw, k), Az, Bz);
    const float t0 = fmaxf(fmaxf(fminf(tx0, tx1), fminf(ty0, ty1)), fmaxf(fminf(tz0, tz1), 0.0f));
    const float t1 = fminf(fminf(fmaxf(tx0, tx1), fmaxf(ty0, ty1)), fminf(fmaxf(tz0, tz1), tb));
    if (t0 <= t1) r.hit |= 1u << k;
    r.tn[k] = t0;
  }
#endif
  return r;
}

// kLayout: -1 the context's layout read from S.nodeq on every visit; 0 / 1: 128 B / quantised
// nodes known at compile time (the persistent kernels are instantiated per layout).
template <bool kWide = false, int kLayout = -1>
__device__ __forceinline__ Node4Hits node4_test(const SceneView& S, int node, const RayF& rf, float tb) {
  // the single-ray path keeps the 128 B nodes: 4 x 16 B loads of the quantised node plus its
  // decode measured 1% slower there (C4, same box)
  if (kWide && PXG_NODEQ && (kLayout == 1 || (kLayout < 0 && S.nodeq))) return node4q_test<true>(S, node, rf, tb);
  const float4* __restrict__ q = reinterpret_cast<const float4*>(S.nodes4 + node);
  float4 lx, ly, lz, hx, hy, hz;
  if (kWide && PXG_NODE256) {
    ldg256(q + 0, lx, ly);
    ldg256(q + 2, lz, hx);
    ldg256(q + 4, hy, hz);
  } else {
    lx = __ldg(q + 0), ly = __ldg(q + 1), lz = __ldg(q + 2);
    hx = __ldg(q + 3), hy = __ldg(q + 4), hz = __ldg(q + 5);
  }
  const int4 ch = __ldg(reinterpret_cast<const int4*>(q + 6));
  Node4Hits r;
  r.hit = 0u;
  const float lxs[4] = {lx.x, lx.y, lx.z, lx.w}, lys[4] = {ly.x, ly.y, ly.z, ly.w}, lzs[4] = {lz.x, lz.y, lz.z, lz.w};
  const float hxs[4] = {hx.x, hx.y, hx.z, hx.w}, hys[4] = {hy.x, hy.y, hy.z, hy.w}, hzs[4] = {hz.x, hz.y, hz.z, hz.w};
  r.code[0] = ch.x;
  r.code[1] = ch.y;
  r.code[2] = ch.z;
  r.code[3] = ch.w;
  r.leafm = (ch.x < 0 ? 1u : 0u) | (ch.y < 0 ? 2u : 0u) | (ch.z < 0 ? 4u : 0u) | (ch.w < 0 ? 8u : 0u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float lo[3] = {lxs[k], lys[k], lzs[k]}, hi[3] = {hxs[k], hys[k], hzs[k]};
    float tn;
    if (box_f(lo, hi, rf, tb, tn)) r.hit |= 1u << k;
    r.tn[k] = tn;
  }
  return r;
}

// Pushes the internal children of `h` that are hit within tb, nearest popped first;
// returns the nearest one to visit next (or -1).
__device__ __forceinline__ void cswap4(float& ta, int& ca, float& tb, int& cb) {
  const bool sw = tb < ta;
  const float t = sw ? tb : ta;
  const int c = sw ? cb : ca;
  tb = sw ? ta : tb;
  cb = sw ? ca : cb;
  ta = t;
  ca = c;
}

constexpr int kNoChild = static_cast<int>(0x80000000u);  // never a node or leaf code

// Traversal stacks of child codes. LocalStack: one per-thread local array (kStack entries).
// SplitStack<kS>: the first kS entries in shared memory (entry i of thread t at
// sm[i * 128 + t]: the lanes of a warp hit 32 distinct banks whatever their depths, one
// wavefront per access instead of one L1 line per lane), deeper entries in a local array.
struct LocalStack {
  int* a;
  __device__ __forceinline__ void push(int& sp, int v) {
    if (sp < kStack) a[sp++] = v;
  }
  __device__ __forceinline__ int pop(int& sp) { return a[--sp]; }
};

// LocalStack with the top entry in a register: a pop returns the register and issues the load
// of the entry below, which is consumed only by the NEXT pop, so the local-memory latency is
// off the node chain (ncu: 8% of the traversal's stall samples waited for the popped child).
// Entry i < sp - 1 lives at a[i], entry sp - 1 in tos.
struct TosStack {
  int* a;
  int tos;
  __device__ __forceinline__ void push(int& sp, int v) {
    if (sp >= kStack) return;
    if (sp > 0) a[sp - 1] = tos;
    tos = v;
    ++sp;
  }
  __device__ __forceinline__ int pop(int& sp) {
    const int r = tos;
    --sp;
    if (sp > 0) tos = a[sp - 1];
    return r;
  }
};

template <int kS>
struct SplitStack {
  int* sm;   // this thread's column of the block's shared stack (stride 128)
  int* loc;  // [kStack - kS]
  __device__ __forceinline__ void push(int& sp, int v) {
    if (sp < kS) {
      sm[sp * 128] = v;
    } else {
      if (sp >= kStack) return;
      loc[sp - kS] = v;
    }
    ++sp;
  }
  __device__ __forceinline__ int pop(int& sp) {
    --sp;
    return sp < kS ? sm[sp * 128] : loc[sp - kS];
  }
};

// Orders the children of `h` (internal nodes and leaves) hit within tbn by tnear: the
// nearest is returned (kNoChild if none), the rest are pushed so that nearer ones pop
// first. Non-candidates get +inf keys; a 5-comparator network sorts in registers.
// kSameBound: tbn is the bound the node test itself used (the postponed-leaf path: no leaf
// test ran in between), so a hit child already satisfies tn <= tbn.
template <bool kSameBound = false, class Stack>
__device__ __forceinline__ int node4_order(const Node4Hits& h, float tbn, Stack& stack, int& sp) {
  float t[4];
  int c[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool ok = (h.hit >> k & 1u) && (kSameBound || h.tn[k] <= tbn);
    t[k] = ok ? h.tn[k] : __int_as_float(0x7f800000);
    c[k] = ok ? h.code[k] : kNoChild;
  }
  cswap4(t[0], c[0], t[1], c[1]);
  cswap4(t[2], c[2], t[3], c[3]);
  cswap4(t[0], c[0], t[2], c[2]);
  cswap4(t[1], c[1], t[3], c[3]);
  cswap4(t[1], c[1], t[2], c[2]);
#pragma unroll
  for (int k = 3; k >= 1; --k)
    if (c[k] != kNoChild) stack.push(sp, c[k]);
  return c[0];
}

// Hit leaf children of a visited node (bit k of the result: child k is a hit leaf).
__device__ __forceinline__ unsigned node4_leaves(const Node4Hits& h) { return h.hit & h.leafm; }

__device__ __forceinline__ int node4_code(const Node4Hits& h, int k) {
  return k == 0 ? h.code[0] : k == 1 ? h.code[1] : k == 2 ? h.code[2] : h.code[3];
}

// h with only its inner (node) children left in the hit mask.
__device__ __forceinline__ Node4Hits node4_inner(const Node4Hits& h) {
  Node4Hits hn = h;
  hn.hit &= ~h.leafm;
  return hn;
}

// Closest hit: returns the original primitive id or -1; t_best in/out (fp64). Every step
// visits one 4-wide node: its hit leaf children are tested right away, its hit inner
// children are visited nearest-first (exactly the persistent kernel's closest_step).
template <bool kCount = false>
__device__ __noinline__ int trace_closest_t(const SceneView& S, const V3& o, const V3& d, double& t_best,
                                            TravCount* cnt = nullptr) {
  const RayF rf = make_rayf(o, d);
  int best = -1;
  int stack_mem[kStack];
  LocalStack stack{stack_mem};
  int sp = 0;
  int node = 0;
  for (;;) {
    const Node4Hits h = node4_test(S, node, rf, tbound_f(t_best));
    if (kCount) cnt->nodes += 1;
    for (unsigned leaves = node4_leaves(h); leaves; leaves &= leaves - 1) {
      const int code = ~node4_code(h, __ffs(leaves) - 1);
      const int first = code >> 4, count = code & 15;
      if (kCount) cnt->prims += count;
      for (int i = 0; i < count; ++i) {
        int id;
        const double t = rec_hit(S, first + i, o, d, t_best, id);
        if (t > 0.0 && (t < t_best || id > best)) {
          t_best = t;
          best = id;
        }
      }
    }
    int next = node4_order(node4_inner(h), tbound_f(t_best), stack, sp);
    if (next == kNoChild) {
      if (sp == 0) break;
      next = stack.pop(sp);
    }
    node = next;
  }
  return best;
}

__device__ __forceinline__ int trace_closest(const SceneView& S, const V3& o, const V3& d, double& t_best) {
  return trace_closest_t<false>(S, o, d, t_best);
}

// Any hit with t in [kRayEps, t_max] (the boolean of Scene::occluded, scene.cpp:170-177);
// same visiting order as trace_closest_t (the persistent kernel's any_step).
template <bool kCount = false>
__device__ __noinline__ bool trace_any_t(const SceneView& S, const V3& o, const V3& d, double t_max,
                                         TravCount* cnt = nullptr) {
  const RayF rf = make_rayf(o, d);
  int stack_mem[kStack];
  LocalStack stack{stack_mem};
  int sp = 0;
  int node = 0;
  const float tb = tbound_f(t_max);
  for (;;) {
    const Node4Hits h = node4_test(S, node, rf, tb);
    if (kCount) cnt->nodes += 1;
    for (unsigned leaves = node4_leaves(h); leaves; leaves &= leaves - 1) {
      const int code = ~node4_code(h, __ffs(leaves) - 1);
      const int first = code >> 4, count = code & 15;
      for (int i = 0; i < count; ++i) {
        int id;
        if (kCount) cnt->prims += 1;
        if (rec_hit(S, first + i, o, d, t_max, id) > 0.0) return true;
      }
    }
    int next = node4_order(node4_inner(h), tb, stack, sp);
    if (next == kNoChild) {
      if (sp == 0) break;
      next = stack.pop(sp);
    }
    node = next;
  }
  return false;
}

__device__ __forceinline__ bool trace_any(const SceneView& S, const V3& o, const V3& d, double t_max) {
  return trace_any_t<false>(S, o, d, t_max);
}

// primitive_normal (scene.cpp:65-72)
__device__ __forceinline__ V3 prim_normal(const SceneView& S, int prim, const V3& at) {
  if (S.prim_shape[prim] == kSphere) {
    const double* c = S.prim_center + 4 * prim;
    return (at - v3(c[0], c[1], c[2])) / c[3];
  }
  const double* g = S.prim_geo + 3 * prim;
  return v3(g[0], g[1], g[2]);
}

// Scene::intersect (scene.cpp:127-150)
__device__ __forceinline__ bool intersect(const SceneView& S, const V3& o, const V3& d, Hit& hit,
                                          double t_max = 1e30) {
  double t_best = t_max;
  int best = trace_closest(S, o, d, t_best);
  if (best < 0) return false;
  hit.t = t_best;
  hit.p = o + t_best * d;
  hit.prim = best;
  hit.n = prim_normal(S, best, hit.p);
  hit.material = S.prim_mat[best];
  hit.emitter = S.prim_emitter[best];
  return true;
}

// Scene::occluded (scene.cpp:170-177)
__device__ __forceinline__ bool occluded(const SceneView& S, const V3& from, const V3& to) {
  V3 d = to - from;
  double dist = length(d);
  if (dist < kRayEps) return false;
  return trace_any(S, from, d / dist, dist * (1.0 - 1e-6));
}

__device__ __forceinline__ bool visible(const SceneView& S, const V3& from, const V3& to) {
  return !occluded(S, from, to);
}

struct LightPoint {
  V3 p, n, radiance;
  int prim;
  double pdf_area;
};

// Scene::sample_light_point (scene.cpp:179-223). The linear cumulative scan is a binary
// search over the same running sums; operand order of the rectangle draw follows the
// reference build (GCC evaluates `a + u()*b + u()*c` right to left: c's draw first).
__device__ __forceinline__ LightPoint sample_light_point(const SceneView& S, Rng& rng) {
  double target = rng.next_double() * S.total_emitter_area;
  int lo = 0, hi = S.n_emit - 1;
  while (lo < hi) {  // first i with target < cum[i]
    int mid = (lo + hi) >> 1;
    if (target < S.emitter_cum[mid]) hi = mid; else lo = mid + 1;
  }
  const int chosen = lo;
  const int prim = S.emitter_prim[chosen];
  LightPoint lp;
  lp.radiance = v3(S.emitter_rad[3 * chosen], S.emitter_rad[3 * chosen + 1], S.emitter_rad[3 * chosen + 2]);
  lp.prim = prim;
  lp.pdf_area = 1.0 / S.total_emitter_area;
  const double* g = S.prim_abc + 9 * prim;
  const int shape = S.prim_shape[prim];
  if (shape == kSphere) {
    double z = 1.0 - 2.0 * rng.next_double();
    double r = sqrt(dmax(0.0, 1.0 - z * z));
    double sp, cp;
    sincos_2pi(rng.next_double(), sp, cp);  // phi = 2*pi*u
    V3 n = v3(r * cp, r * sp, z);
    const double* c = S.prim_center + 4 * prim;
    lp.p = v3(c[0], c[1], c[2]) + c[3] * n;
    lp.n = n;
  } else if (shape == kTriangle) {
    double u = rng.next_double(), v = rng.next_double();
    if (u + v > 1.0) {
      u = 1.0 - u;
      v = 1.0 - v;
    }
    lp.p = v3(g[0], g[1], g[2]) + u * v3(g[3], g[4], g[5]) + v * v3(g[6], g[7], g[8]);
    lp.n = prim_normal(S, prim, lp.p);
  } else {
    double vc = rng.next_double();
    double ub = rng.next_double();
    lp.p = v3(g[0], g[1], g[2]) + ub * v3(g[3], g[4], g[5]) + vc * v3(g[6], g[7], g[8]);
    lp.n = prim_normal(S, prim, lp.p);
  }
  return lp;
}

// Scene::emitted (scene.cpp:225-232)
__device__ __forceinline__ V3 emitted(const SceneView& S, int emitter, const V3& n, const V3& dir_out) {
  if (emitter < 0 || dot(dir_out, n) <= 0.0) return v3(0.0);
  const double* r = S.emitter_rad + 3 * emitter;
  return v3(r[0], r[1], r[2]);
}
#endif  // __CUDACC__

}  // namespace pxg
