// pxg_path.cuh — sub-paths, connections and the reciprocal-aware MIS weight on the device.
//
// Restates proj/src/transport.cpp:37-268 and proj/src/proxy.cpp:430-546 for one thread
// per path. Vertices live in HBM (vertex-major: vertex k of pixel i at base[k*stride+i]).
//
// MIS cost. The reference evaluates strategy_pdf from scratch for every split of every
// connection, O(n^2) BSDF pdfs per connection (proxy.cpp:542-543). Every factor of
// strategy_pdf (transport.cpp:206-253) and of proxy_weight_density (proxy.cpp:469-514)
// is one of three per-path quantities — the light-direction density LD of y0->y1, the
// forward step F(i) = bsdf_step(i-1, i-2, i) and the reverse step R(j) = bsdf_step(j+1,
// j+2, j) — so PathTable memoises them: each distinct step is evaluated once (<= 2n pdfs
// per connection) and every strategy density is then the same product, multiplied in the
// same order, as in the reference. Results are bit-identical; the cost drops from O(n^3)
// to O(n^2) multiplies and O(n) pdf evaluations.
#pragma once

#include "pxg_scene.cuh"

namespace pxg {

enum VertexFlag { kLight = 0, kDiffuse = 1, kSpecular = 2, kCamera = 3 };
constexpr int kMaxPath = 20;  // >= max_depth + 1 eye + max_depth - 1 light (max_depth <= 16)

// PathVertex (proj/include/proxima/transport.hpp:17-28); 128 B.
struct alignas(16) PV {
  V3 p, n, wi, thr;
  double pdf_fwd;
  int mat, prim, emitter, flag;
  double pad;
};

struct StatsView {
  const double* max_ratio;   // [4000]
  const double* sum_est;     // [4000]
  const double* sum_sq;      // [4000]
  const long long* est_count;  // [4000]
};

struct Mapper {  // SubspaceMapper (proj/include/proxima/subspace.hpp:23-50)
  V3 bmin, bmax;
};

#if defined(__CUDACC__)

__device__ __forceinline__ bool specmat(const SceneView& S, const PV& v) {
  return v.mat >= 0 && S.materials[v.mat].specular;
}

// ---- subspace labels (proj/src/subspace.cpp:21-55) ----
__device__ __forceinline__ int grid_axis(double v, double lo, double hi) {
  double extent = hi - lo;
  if (!(extent > 0.0)) return 0;
  int i = static_cast<int>((v - lo) / extent * 4);
  return i < 0 ? 0 : (i > 3 ? 3 : i);
}
__device__ __forceinline__ int grid_cell(const Mapper& M, const V3& p) {
  int ix = grid_axis(p.x, M.bmin.x, M.bmax.x);
  int iy = grid_axis(p.y, M.bmin.y, M.bmax.y);
  int iz = grid_axis(p.z, M.bmin.z, M.bmax.z);
  return (ix * 4 + iy) * 4 + iz;
}
__device__ __forceinline__ int octant(const V3& v) {
  return (v.x > 0.0 ? 1 : 0) | (v.y > 0.0 ? 2 : 0) | (v.z > 0.0 ? 4 : 0);
}
__device__ __forceinline__ int classify_specular(const Mapper& M, const PV& v) {
  return (grid_cell(M, v.p) * 8 + octant(v.n)) % 100;
}
__device__ __forceinline__ int classify_control(const Mapper& M, const PV* hc, bool has_dir, const V3& dir) {
  if (hc == nullptr) return 0;
  int slot = has_dir ? octant(dir) : 8;
  int raw = grid_cell(M, hc->p) * 9 + slot;
  return 1 + raw % 9;
}
__device__ __forceinline__ int classify_eye(const Mapper& M, const V3& p, const V3& dir) {
  return (grid_cell(M, p) * 8 + octant(dir)) % 32;
}
__device__ __forceinline__ int bucket_index(int u, int c, int s) { return ((u - 1) * 10 + c) * 100 + s; }

// ---- measure conversion (transport.cpp:92-99) ----
__device__ __forceinline__ double to_area_density(double pdf_w, const V3& from, const V3& to, const V3& n_to) {
  V3 d = to - from;
  double dist2 = dot(d, d);
  if (dist2 <= 0.0) return 0.0;
  double cos_to = fabs(dot(n_to, d)) / sqrt(dist2);
  return pdf_w * cos_to / dist2;
}

__device__ __forceinline__ double light_direction_pdf(const V3& n, const V3& d) {
  double c = dot(n, d);
  return c > 0.0 ? c / kPi : 0.0;
}

__device__ __forceinline__ PV surface_vertex(const SceneView& S, const Hit& h, const V3& wi) {
  PV v;
  v.p = h.p;
  v.n = h.n;
  v.wi = wi;
  v.thr = v3(1.0);
  v.pdf_fwd = 0.0;
  v.mat = h.material;
  v.prim = h.prim;
  v.emitter = h.emitter;
  v.flag = S.materials[h.material].specular ? kSpecular : kDiffuse;
  v.pad = 0.0;
  return v;
}

// Pixel ray (scene.cpp:116-125); u, v are the jitter draws.
__device__ __forceinline__ V3 camera_dir(const SceneView& S, int px, int py, double u, double v) {
  double sx = (2.0 * ((px + u) / S.width) - 1.0) * S.tan_half * S.aspect;
  double sy = (1.0 - 2.0 * ((py + v) / S.height)) * S.tan_half;
  return normalize(S.cam_fwd + sx * S.cam_right + sy * S.cam_up);
}

// extend_walk (transport.cpp:37-56). `out` holds n vertices already; returns the count.
__device__ __forceinline__ int extend_walk(const SceneView& S, PV* out, size_t stride, int n, V3 beta,
                                           V3 dir, double pdf_dir, int max_vertices, Rng& rng) {
  PV prev = out[(n - 1) * stride];
  while (n < max_vertices) {
    Hit hit;
    if (!intersect(S, prev.p, dir, hit)) break;
    PV v = surface_vertex(S, hit, -dir);
    v.pdf_fwd = to_area_density(pdf_dir, prev.p, v.p, v.n);
    v.thr = beta;
    out[n * stride] = v;
    ++n;
    if (n >= max_vertices) break;
    BsdfSample bs = sample_bsdf(S.materials[v.mat], v.n, v.wi, rng);
    if (!bs.valid || bs.pdf <= 0.0) break;
    beta = beta * bs.value * (fabs(dot(bs.wo, v.n)) / bs.pdf);
    if (near_zero(beta)) break;
    dir = bs.wo;
    pdf_dir = bs.pdf;
    prev = v;
  }
  return n;
}

// trace_light_subpath (transport.cpp:111-135)
__device__ __forceinline__ int trace_light_subpath(const SceneView& S, int max_vertices, Rng& rng, PV* out,
                                                   size_t stride) {
  if (max_vertices < 1) return 0;
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
  out[0] = y0;
  if (max_vertices == 1) return 1;
  V3 d = sample_cosine_hemisphere(lp.n, rng);
  double pdf_dir = light_direction_pdf(lp.n, d);
  if (pdf_dir <= 0.0) return 1;
  V3 beta = y0.thr * lp.radiance * (dot(d, lp.n) / pdf_dir);
  return extend_walk(S, out, stride, 1, beta, d, pdf_dir, max_vertices, rng);
}

// trace_eye_subpath (transport.cpp:137-166). The jitter draws are taken v first, then u:
// the reference build evaluates generate_ray's two rng arguments right to left.
__device__ __forceinline__ int trace_eye_subpath(const SceneView& S, int px, int py, int max_vertices, Rng& rng,
                                                 PV* out, size_t stride) {
  if (max_vertices < 1) return 0;
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
  out[0] = z0;
  if (max_vertices == 1) return 1;
  double jv = rng.next_double();
  double ju = rng.next_double();
  V3 dir = camera_dir(S, px, py, ju, jv);
  Hit hit;
  if (!intersect(S, S.cam_pos, dir, hit)) return 1;
  PV z1 = surface_vertex(S, hit, -dir);
  z1.pdf_fwd = 1.0;
  z1.thr = v3(1.0);
  out[stride] = z1;
  if (max_vertices == 2) return 2;
  BsdfSample bs = sample_bsdf(S.materials[z1.mat], z1.n, z1.wi, rng);
  if (!bs.valid || bs.pdf <= 0.0) return 2;
  V3 beta = bs.value * (fabs(dot(bs.wo, z1.n)) / bs.pdf);
  return extend_walk(S, out, stride, 2, beta, bs.wo, bs.pdf, max_vertices, rng);
}

// geometry_term (transport.cpp:168-176)
__device__ __forceinline__ double geometry_term(const SceneView& S, const PV& a, const PV& b) {
  V3 d = b.p - a.p;
  double dist2 = dot(d, d);
  if (dist2 <= 0.0) return 0.0;
  V3 dir = d / sqrt(dist2);
  double g = fabs(dot(a.n, dir)) * fabs(dot(b.n, dir)) / dist2;
  if (g <= 0.0) return 0.0;
  return visible(S, a.p, b.p) ? g : 0.0;
}

// A full path light[0..s-1] + eye[t-1..0] (transport.hpp:37-44) read through strided views.
// Strides are in bytes so the vertices can also live in shared memory at a padded stride.
struct FullPath {
  const char* L;
  size_t ls;
  const char* E;
  size_t es;
  int s, t;
  __device__ __forceinline__ const PV& vtx(int i) const {
    return i < s ? *reinterpret_cast<const PV*>(L + i * ls) : *reinterpret_cast<const PV*>(E + (s + t - 1 - i) * es);
  }
};

__device__ __forceinline__ FullPath make_fp(const PV* L, size_t ls, const PV* E, size_t es, int s, int t) {
  return FullPath{reinterpret_cast<const char*>(L), ls * sizeof(PV), reinterpret_cast<const char*>(E),
                  es * sizeof(PV), s, t};
}

// Memoised step densities of one full path (see header comment).
struct PathTable {
  double F[kMaxPath];
  double R[kMaxPath];
  double ld_pdfw, ld_area;
  unsigned fmask, rmask;
  bool ld_done, ld_ok;
};

// bsdf_step of strategy_pdf (transport.cpp:226-234) / proxy_weight_density (proxy.cpp:469-477).
__device__ __forceinline__ double bsdf_step_v(const SceneView& S, const PV& v, const PV& vf, const PV& vt) {
  V3 wi = normalize(vf.p - v.p);
  V3 wo_dir = vt.p - v.p;
  double len = length(wo_dir);
  if (len <= 0.0) return 0.0;
  double pdf_w = pdf_bsdf(S.materials[v.mat], v.n, wi, wo_dir / len);
  return to_area_density(pdf_w, v.p, vt.p, vt.n);
}

__device__ __forceinline__ double bsdf_step(const SceneView& S, const FullPath& fp, int at, int from, int to) {
  return bsdf_step_v(S, fp.vtx(at), fp.vtx(from), fp.vtx(to));
}

// Per-sub-path step densities shared by every connection of a pixel (strided by pixel):
//   LF[i] = step(y[i-1] <- y[i-2] -> y[i])  i in [2, nl-1]   (light forward)
//   LR[j] = step(y[j+1] <- y[j+2] -> y[j])  j in [0, nl-3]   (light reverse)
//   EF[m] = step(e[m+1] <- e[m+2] -> e[m])  m in [0, ne-3]   (eye, light direction)
//   ER[m] = step(e[m-1] <- e[m-2] -> e[m])  m in [2, ne-1]   (eye, eye direction)
//   ld    = light_direction density y0 -> y1 (ld_ok = 0: strategy returns 0)
struct PathCache {
  double* LF;
  double* LR;
  double* EF;
  double* ER;
  double* ld;
  int* ld_ok;
  int n;  // stride (pixels)
};

__device__ __forceinline__ double tabF(const SceneView& S, const FullPath& fp, PathTable& T, int i) {
  if (!(T.fmask & (1u << i))) {
    T.F[i] = bsdf_step(S, fp, i - 1, i - 2, i);
    T.fmask |= 1u << i;
  }
  return T.F[i];
}
__device__ __forceinline__ double tabR(const SceneView& S, const FullPath& fp, PathTable& T, int j) {
  if (!(T.rmask & (1u << j))) {
    T.R[j] = bsdf_step(S, fp, j + 1, j + 2, j);
    T.rmask |= 1u << j;
  }
  return T.R[j];
}
// Light-direction density y0 -> y1. ok=false means "return 0" (len <= 0 or pdf_w <= 0).
__device__ __forceinline__ void tabLD(const FullPath& fp, PathTable& T) {
  if (T.ld_done) return;
  T.ld_done = true;
  const PV& y0 = fp.vtx(0);
  const PV& y1 = fp.vtx(1);
  V3 d = y1.p - y0.p;
  double len = length(d);
  T.ld_ok = false;
  if (len <= 0.0) return;
  double pdf_w = light_direction_pdf(y0.n, d / len);
  if (pdf_w <= 0.0) return;
  T.ld_ok = true;
  T.ld_area = to_area_density(pdf_w, y0.p, y1.p, y1.n);
}

// Pre-fills the memo table of connection (s, t) of pixel i from the per-sub-path caches;
// only the junction steps (F(s), F(s+1), R(s-2), R(s-1)) and, for s = 1 or 0, the
// light-direction factor remain to be evaluated. Values are the same function of the same
// vertices, so every strategy density is bit-identical to the uncached table.
__device__ __forceinline__ void table_init_cached(PathTable& T, const PathCache& C, int i, int s, int t) {
  T.fmask = 0u;
  T.rmask = 0u;
  T.ld_done = false;
  T.ld_ok = false;
  const int n_v = s + t;
  const size_t n = static_cast<size_t>(C.n);
  for (int k = 2; k <= s - 1; ++k) {
    T.F[k] = C.LF[k * n + i];
    T.fmask |= 1u << k;
  }
  for (int k = s + 2; k <= n_v - 1; ++k) {
    T.F[k] = C.EF[(n_v - 1 - k) * n + i];
    T.fmask |= 1u << k;
  }
  for (int j = 0; j <= s - 3; ++j) {
    T.R[j] = C.LR[j * n + i];
    T.rmask |= 1u << j;
  }
  for (int j = s; j <= n_v - 3; ++j) {
    T.R[j] = C.ER[(n_v - 1 - j) * n + i];
    T.rmask |= 1u << j;
  }
  if (s >= 2) {
    T.ld_done = true;
    T.ld_ok = C.ld_ok[i] != 0;
    T.ld_area = C.ld[i];
  }
}

// Same as table_init_cached with the per-sub-path steps held in (shared-memory) arrays of
// one pixel: LF/LR indexed by light vertex, EF/ER by eye vertex.
__device__ __forceinline__ void table_init_local(PathTable& T, const double* LF, const double* LR, const double* EF,
                                                 const double* ER, double ld, int ld_ok, int s, int t) {
  T.fmask = 0u;
  T.rmask = 0u;
  T.ld_done = false;
  T.ld_ok = false;
  const int n_v = s + t;
  for (int k = 2; k <= s - 1; ++k) {
    T.F[k] = LF[k];
    T.fmask |= 1u << k;
  }
  for (int k = s + 2; k <= n_v - 1; ++k) {
    T.F[k] = EF[n_v - 1 - k];
    T.fmask |= 1u << k;
  }
  for (int j = 0; j <= s - 3; ++j) {
    T.R[j] = LR[j];
    T.rmask |= 1u << j;
  }
  for (int j = s; j <= n_v - 3; ++j) {
    T.R[j] = ER[n_v - 1 - j];
    T.rmask |= 1u << j;
  }
  if (s >= 2) {
    T.ld_done = true;
    T.ld_ok = ld_ok != 0;
    T.ld_area = ld;
  }
}

__device__ __forceinline__ void table_init(PathTable& T) {
  T.fmask = 0u;
  T.rmask = 0u;
  T.ld_done = false;
  T.ld_ok = false;
}

// Evaluates the junction steps of connection (s, t) eagerly, at one point of the code for
// every lane: F(s), F(s+1), R(s-2), R(s-1) and the light-direction factor when it involves
// an eye vertex (s <= 1). Together with the cached sub-path steps the table is then
// complete, so the strategy loops below never branch into a pdf evaluation (the lazy
// version ran at 2/32 active lanes). Same function, same inputs: bit-identical values.
__device__ __forceinline__ void table_fill_junctions(const SceneView& S, const FullPath& fp, PathTable& T) {
  const int s = fp.s, n_v = fp.s + fp.t;
  if (s >= 2 && s <= n_v - 1) tabF(S, fp, T, s);
  if (s >= 1 && s + 1 <= n_v - 1) tabF(S, fp, T, s + 1);
  if (s >= 2 && s - 2 <= n_v - 3) tabR(S, fp, T, s - 2);
  if (s >= 1 && s - 1 <= n_v - 3) tabR(S, fp, T, s - 1);
  if (n_v >= 2) tabLD(fp, T);
}

// strategy_pdf (transport.cpp:206-253) on the memoised factors.
__device__ __forceinline__ double strategy_pdf(const SceneView& S, const FullPath& fp, PathTable& T, int s) {
  const int n_v = fp.s + fp.t;
  const int t = n_v - s;
  if (s < 0 || t < 2) return 0.0;
  if (s >= 1) {
    if (fp.vtx(s).flag != kDiffuse) return 0.0;
    if (s >= 2 && fp.vtx(s - 1).flag != kDiffuse) return 0.0;
    if (fp.vtx(0).emitter < 0) return 0.0;
  }
  double p = 1.0;
  if (s >= 1) p *= 1.0 / S.total_emitter_area;
  if (s >= 2) {
    tabLD(fp, T);
    if (!T.ld_ok) return 0.0;
    p *= T.ld_area;
  }
  for (int i = 2; i < s; ++i) {
    double step = tabF(S, fp, T, i);
    if (step <= 0.0) return 0.0;
    p *= step;
  }
  for (int j = n_v - 3; j >= s; --j) {
    double step = tabR(S, fp, T, j);
    if (step <= 0.0) return 0.0;
    p *= step;
  }
  return p;
}

// proxy_weight_density (proxy.cpp:430-531) on the memoised factors.
__device__ __forceinline__ double proxy_weight_density(const SceneView& S, const Mapper& M, const StatsView& st,
                                                       const FullPath& fp, PathTable& T) {
  const int n = fp.s + fp.t;
  if (n < 4) return 0.0;
  if (fp.vtx(n - 1).flag != kCamera) return 0.0;
  int k = 1;
  while (n - 1 - k >= 1 && specmat(S, fp.vtx(n - 1 - k))) ++k;
  const int jz = n - 1 - k;
  if (jz < 2) return 0.0;
  const PV& zv = fp.vtx(jz);
  if (zv.mat < 0 || specmat(S, zv)) return 0.0;
  const int jy = jz - 1;
  if (!specmat(S, fp.vtx(jy))) return 0.0;
  int u = 0;
  while (jy - u >= 0 && specmat(S, fp.vtx(jy - u))) ++u;
  if (u < 1 || u > 4) return 0.0;
  const int ti = jy - u;
  if (ti < 0) return 0.0;
  const int ci = ti - 1;
  const PV* hc = nullptr;
  bool has_wc = false;
  V3 wc = v3(0.0);
  if (ci >= 0) {
    hc = &fp.vtx(ci);
    if (hc->emitter < 0) return 0.0;
    if (ci >= 1) {
      wc = normalize(hc->p - fp.vtx(ci - 1).p);
      has_wc = true;
    }
    if (fp.vtx(0).emitter < 0) return 0.0;
  } else {
    if (fp.vtx(ti).emitter < 0) return 0.0;
  }
  double p = 1.0;
  for (int j = n - 3; j >= jz; --j) {
    double step = tabR(S, fp, T, j);
    if (step <= 0.0) return 0.0;
    p *= step;
  }
  if (ci >= 0) {
    p *= 1.0 / S.total_emitter_area;
    if (ci >= 1) {
      tabLD(fp, T);
      if (!T.ld_ok) return 0.0;
      p *= T.ld_area;
    }
    for (int i = 2; i <= ci; ++i) {
      double step = tabF(S, fp, T, i);
      if (step <= 0.0) return 0.0;
      p *= step;
    }
  }
  {
    double step = tabR(S, fp, T, jy - 1);
    if (step <= 0.0) return 0.0;
    p *= step;
  }
  for (int m = jy - 1; m > ti; --m) {
    double step = tabR(S, fp, T, m - 1);
    if (step <= 0.0) return 0.0;
    p *= step;
  }
  const int key = bucket_index(u, classify_control(M, hc, has_wc, wc), classify_specular(M, fp.vtx(jy)));
  const long long cnt = st.est_count[key];
  if (cnt <= 0) return 0.0;
  const double m1 = st.sum_est[key] / static_cast<double>(cnt);
  if (!(m1 > 0.0)) return 0.0;
  double config_density;
  if (cnt >= 16) {
    const double m2 = st.sum_sq[key] / static_cast<double>(cnt);
    if (!(m2 > 0.0)) return 0.0;
    config_density = m1 / m2;
  } else {
    config_density = 1.0 / m1;
  }
  return p * config_density;
}

// reciprocal_mis_weight (proxy.cpp:533-546). cur_s < 0 selects the proxy strategy.
__device__ __forceinline__ double reciprocal_mis_weight_t(const SceneView& S, const Mapper& M, const StatsView& st,
                                                          const FullPath& fp, PathTable& T, int cur_s,
                                                          bool use_stats) {
  const double p_proxy = use_stats ? proxy_weight_density(S, M, st, fp, T) : 0.0;
  const double num = cur_s < 0 ? p_proxy : strategy_pdf(S, fp, T, cur_s);
  if (num <= 0.0) return 0.0;
  const int n_v = fp.s + fp.t;
  double denom = 0.0;
  for (int sp = 0; sp <= n_v - 2; ++sp) denom += strategy_pdf(S, fp, T, sp);
  denom += p_proxy;
  return num / denom;
}

// reciprocal_mis_weight on a COMPLETE table (cached sub-path steps + table_fill_junctions),
// written without early exits so a warp's lanes (different (s, t), different n_v) stay
// converged: every strategy density is the same left-to-right product as strategy_pdf
// (transport.cpp:218-253) and is replaced by 0 when a flag check fails or a factor is
// <= 0, exactly where strategy_pdf returns 0. Sum order and the final division are the
// reference's (proxy.cpp:536-545), so the weight is bit-identical.
__device__ __forceinline__ double mis_weight_full(const SceneView& S, const Mapper& M, const StatsView& st,
                                                  const FullPath& fp, PathTable& T, int cur_s, bool use_stats) {
  const double p_proxy = use_stats ? proxy_weight_density(S, M, st, fp, T) : 0.0;
  const int n_v = fp.s + fp.t;
  unsigned diffuse = 0u;
  for (int i = 0; i < n_v; ++i) diffuse |= (fp.vtx(i).flag == kDiffuse ? 1u : 0u) << i;
  const bool emit0 = fp.vtx(0).emitter >= 0;
  const double inv_area = 1.0 / S.total_emitter_area;
  const double ld = T.ld_ok ? T.ld_area : 0.0;
  double num = 0.0, denom = 0.0;
  for (int sp = 0; sp <= n_v - 2; ++sp) {
    bool ok = true;
    if (sp >= 1) ok = ((diffuse >> sp) & 1u) && (sp < 2 || ((diffuse >> (sp - 1)) & 1u)) && emit0;
    double p = 1.0;
    if (sp >= 1) p *= inv_area;
    if (sp >= 2) {
      ok = ok && T.ld_ok;
      p *= ld;
    }
    for (int i = 2; i < sp; ++i) {
      const double v = T.F[i];
      ok = ok && v > 0.0;
      p *= v;
    }
    for (int j = n_v - 3; j >= sp; --j) {
      const double v = T.R[j];
      ok = ok && v > 0.0;
      p *= v;
    }
    p = ok ? p : 0.0;
    if (sp == cur_s) num = p;
    denom += p;
  }
  if (cur_s < 0) num = p_proxy;
  if (num <= 0.0) return 0.0;
  denom += p_proxy;
  return num / denom;
}

__device__ __forceinline__ double reciprocal_mis_weight(const SceneView& S, const Mapper& M, const StatsView& st,
                                                        const FullPath& fp, int cur_s, bool use_stats) {
  PathTable T;
  table_init(T);
  return reciprocal_mis_weight_t(S, M, st, fp, T, cur_s, use_stats);
}

// connection_contribution (transport.cpp:187-196) incl. junction_kernels (:70-88).
__device__ __forceinline__ V3 connection_contribution(const SceneView& S, const FullPath& fp) {
  if (fp.s < 1 || fp.t < 2) return v3(0.0);
  const PV& y = fp.vtx(fp.s - 1);
  const PV& z = fp.vtx(fp.s);
  if (z.flag != kDiffuse) return v3(0.0);
  V3 d = z.p - y.p;
  double len = length(d);
  if (len <= 0.0) return v3(0.0);
  V3 dir = d / len;
  V3 f_light;
  if (fp.s == 1) {
    f_light = emitted(S, y.emitter, y.n, dir);
  } else {
    if (y.flag != kDiffuse) return v3(0.0);
    f_light = eval_bsdf(S.materials[y.mat], y.n, y.wi, dir);
  }
  V3 f_eye = eval_bsdf(S.materials[z.mat], z.n, z.wi, -dir);
  if (near_zero(f_light) || near_zero(f_eye)) return v3(0.0);
  double g = geometry_term(S, y, z);
  if (g <= 0.0) return v3(0.0);
  return y.thr * f_light * g * f_eye * z.thr;
}

// weighted_bdpt_value (proxy.cpp:621-643): all standard strategies of one px-sample.
__device__ __forceinline__ V3 weighted_bdpt_value(const SceneView& S, const Mapper& M, const StatsView& st,
                                                  bool use_stats, const PV* eye, size_t es, int n_eye,
                                                  const PV* light, size_t ls, int n_light) {
  V3 radiance = v3(0.0);
  for (int t = 2; t <= n_eye; ++t) {
    const PV& z = eye[(t - 1) * es];
    if (z.emitter >= 0) {
      V3 le = z.thr * emitted(S, z.emitter, z.n, z.wi);
      if (!near_zero(le)) {
        FullPath fp = make_fp(light, ls, eye, es, 0, t);
        radiance += le * reciprocal_mis_weight(S, M, st, fp, 0, use_stats);
      }
    }
    for (int s = 1; s <= n_light && s + t <= S.max_depth + 1; ++s) {
      FullPath fp = make_fp(light, ls, eye, es, s, t);
      V3 c = connection_contribution(S, fp);
      if (near_zero(c)) continue;
      radiance += c * reciprocal_mis_weight(S, M, st, fp, s, use_stats);
    }
  }
  return radiance;
}

#endif  // __CUDACC__

}  // namespace pxg
