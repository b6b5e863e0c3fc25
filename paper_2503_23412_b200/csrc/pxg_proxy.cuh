// pxg_proxy.cuh — proxy sampling on the device: dropout, the supporting mixture, the
// incomplete-path target density, the reciprocal (Russian-roulette-and-split) tree,
// the proxy retrace and the proxy connection. Restates proj/src/proxy.cpp:28-603 and
// proj/include/proxima/recip.hpp:49-138 with the reference's operation and draw order.
#pragma once

#include "pxg_path.cuh"

namespace pxg {

constexpr int kMaxLight = 16;  // light sub-path vertices (max_depth - 1 <= 15) + repair slack

// IncompleteLightSubPath (proj/include/proxima/proxy.hpp:27-42). Prefix vertices are
// stored separately (IncPool::prefix, kMaxLight per entry).
struct IncHdr {
  PV spec_end;
  V3 cdir;
  double prefix_pdf;
  double inverse_p, inverse_p_m2;
  int u, n_prefix, has_cdir, c_label;
  int s_label, key, walk, end;
  int dflag_last, valid, pad0, pad1;
};

struct IncView {
  const IncHdr* hdr;
  const PV* prefix;  // [entry][kMaxLight]
};

// Errors raised by the estimator (the reference throws std::runtime_error).
enum { kErrNone = 0, kErrIntegrand = 1, kErrSupport = 2, kErrSplit = 3, kErrRatio = 4, kErrPool = 5 };

struct RecipFrame {
  double ans;
  double sgn;
  long long rem;
};

// Resumable state of one reciprocal run (recip::estimate_reciprocal, recip.hpp:131-138).
// The DFS itself is k_recip_dfs_warp (pxg_stage_kernels.cuh): main_tree (recip.hpp:89-97)
// unrolled onto an explicit frame stack over precomputed nodes, nesting the partial sums
// exactly like the recursion (frame d holds ans = g/B + sgn * child values so far and the
// number of children still to expand), so the estimate is bit-identical.
struct RunState {
  long long depth, cost, avail;  // avail: nodes 0..avail-1 have precomputed (g, n)
  double ret;
  int entering, truncated, done, err;
};

// stochastic_split (recip.hpp:49-56) of node k on its own split stream.
PXD long long split_count(double g, Rng& split_rng, int& err) {
  const double r = fabs(g);
  if (!(r >= 0.0) || !isfinite(r)) {
    err = kErrSplit;
    return 0;
  }
  const double fl = floor(r);
  const double frac = r - fl;
  long long n = static_cast<long long>(fl);
  if (frac > 0.0 && split_rng.bernoulli(frac)) ++n;
  return n;
}

#if defined(__CUDACC__)

__device__ __forceinline__ const PV* inc_control(const IncHdr& h, const PV* prefix) {
  return h.n_prefix > 0 ? &prefix[h.n_prefix - 1] : nullptr;
}

// dropout (proxy.cpp:59-94) of the prefix v[0..n) of a traced light walk (stride 1).
// Writes the header and prefix vertices; returns false when the shape is not eligible.
__device__ __forceinline__ bool dropout(const Mapper& M, const PV* v, int n, IncHdr& h, PV* prefix_out) {
  if (n < 2) return false;
  if (v[n - 1].flag != kSpecular) return false;
  int u = 0;
  while (u < n && v[n - 1 - u].flag == kSpecular) ++u;
  if (u < 1 || u > 4) return false;
  const int terminal = n - 1 - u;
  h.u = u;
  h.spec_end = v[n - 1];
  h.dflag_last = v[terminal].flag;
  h.n_prefix = terminal;
  h.has_cdir = 0;
  h.cdir = v3(0.0);
  if (terminal > 0) {
    const PV& hc = v[terminal - 1];
    if (hc.emitter < 0) return false;
    if (terminal >= 2) {
      h.cdir = -hc.wi;
      h.has_cdir = 1;
    }
  } else if (v[terminal].flag != kLight) {
    return false;
  }
  double pp = 1.0;
  for (int i = 0; i < terminal; ++i) pp *= v[i].pdf_fwd;
  h.prefix_pdf = pp;
  if (!(pp > 0.0)) return false;
  if (prefix_out)
    for (int i = 0; i < terminal; ++i) prefix_out[i] = v[i];
  h.s_label = classify_specular(M, h.spec_end);
  h.c_label = classify_control(M, terminal > 0 ? &v[terminal - 1] : nullptr, h.has_cdir != 0, h.cdir);
  h.key = bucket_index(u, h.c_label, h.s_label);
  h.inverse_p = 0.0;
  h.inverse_p_m2 = 0.0;
  return true;
}

__device__ __forceinline__ PV vertex_from_hit(const SceneView& S, const Hit& hit, const V3& wi) {
  return surface_vertex(S, hit, wi);
}

__device__ __forceinline__ double sphere_cosine_pdf(const V3& n, const V3& d) {
  return fabs(dot(n, d)) / (2.0 * kPi);
}

struct Cand {
  PV g[4];
  double q;
  bool escaped;
};

// Visibility of segment (a, b) as the reference evaluates it (visible(a, b), scene.hpp:86-87).
// `seg` names the segment within one node evaluation (0-3: support chain, 4: control -> g0,
// 5-9: target chain), so the reciprocal-node wavefront can trace them all as one queue and
// replay the same code with the results (k_recip_eval_wave).
struct VisDirect {
  const SceneView* S;
  __device__ __forceinline__ bool operator()(int, const V3& a, const V3& b) const { return visible(*S, a, b); }
};

// The two terms of support_pdf (proxy.cpp:153-209): q_fs (the from-specular strand) and
// q_other (light-area or from-control strand; only for u == 1).
template <class Vis>
__device__ __forceinline__ void support_terms_v(const SceneView& S, const IncHdr& h, const PV* prefix, const PV* g,
                                                const Vis& vis, double& q_fs_out, double& q_other_out) {
  const int u = h.u;
  const PV* hc = inc_control(h, prefix);
  const PV& y = h.spec_end;
  double q_fs = 1.0;
  {
    const PV* before = nullptr;
    const PV* prev = &y;
    for (int j = 0; j < u; ++j) {
      const PV& nxt = g[j];
      V3 d = nxt.p - prev->p;
      double len = length(d);
      if (len <= 0.0) {
        q_fs = 0.0;
        break;
      }
      V3 dir = d / len;
      double pdf_w = (j == 0) ? sphere_cosine_pdf(y.n, dir)
                              : pdf_bsdf(S.materials[prev->mat], prev->n, normalize(before->p - prev->p), dir);
      if (pdf_w <= 0.0 || !vis(j, prev->p, nxt.p)) {
        q_fs = 0.0;
        break;
      }
      q_fs *= to_area_density(pdf_w, prev->p, nxt.p, nxt.n);
      before = prev;
      prev = &nxt;
    }
  }
  q_fs_out = q_fs;
  q_other_out = 0.0;
  if (u > 1) return;
  double q_other = 0.0;
  if (hc == nullptr) {
    if (g[0].emitter >= 0) q_other = 1.0 / S.total_emitter_area;
  } else {
    V3 d = g[0].p - hc->p;
    double len = length(d);
    if (len > 0.0) {
      V3 dir = d / len;
      double pdf_w = h.has_cdir ? pdf_bsdf(S.materials[hc->mat], hc->n, -h.cdir, dir)
                                : light_direction_pdf(hc->n, dir);
      if (pdf_w > 0.0 && vis(4, hc->p, g[0].p)) q_other = to_area_density(pdf_w, hc->p, g[0].p, g[0].n);
    }
  }
  q_other_out = q_other;
}

// support_pdf from its terms, in the reference's operation order.
__device__ __forceinline__ double support_combine(int u, double q_fs, double q_other) {
  return u > 1 ? q_fs : 0.5 * (q_other + q_fs);
}

template <class Vis>
__device__ __forceinline__ double support_pdf_v(const SceneView& S, const IncHdr& h, const PV* prefix, const PV* g,
                                                const Vis& vis) {
  double q_fs, q_other;
  support_terms_v(S, h, prefix, g, vis, q_fs, q_other);
  return support_combine(h.u, q_fs, q_other);
}

__device__ __forceinline__ double support_pdf(const SceneView& S, const IncHdr& h, const PV* prefix, const PV* g) {
  return support_pdf_v(S, h, prefix, g, VisDirect{&S});
}

// support_sample (proxy.cpp:211-269)
__device__ __forceinline__ void support_sample(const SceneView& S, const IncHdr& h, const PV* prefix, Rng& rng,
                                               Cand& c) {
  const int u = h.u;
  c.escaped = false;
  c.q = 0.0;
  const PV* hc = inc_control(h, prefix);
  const PV& y = h.spec_end;
  const int strand = (u == 1) ? static_cast<int>(rng.next_below(2)) : 0;
  if (strand == 1 && hc == nullptr) {
    LightPoint lp = sample_light_point(S, rng);
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
    c.g[0] = v;
  } else if (strand == 1) {
    V3 dir;
    if (h.has_cdir) {
      BsdfSample bs = sample_bsdf(S.materials[hc->mat], hc->n, -h.cdir, rng);
      if (!bs.valid || bs.pdf <= 0.0) {
        c.escaped = true;
        c.q = 1.0;
        return;
      }
      dir = bs.wo;
    } else {
      dir = sample_cosine_hemisphere(hc->n, rng);
    }
    Hit hit;
    if (!intersect(S, hc->p, dir, hit)) {
      c.escaped = true;
      c.q = 1.0;
      return;
    }
    c.g[0] = vertex_from_hit(S, hit, -dir);
  } else {
    const PV* prev = &y;
    for (int j = 0; j < u; ++j) {
      V3 dir;
      if (j == 0) {
        V3 axis = rng.next_double() < 0.5 ? y.n : -y.n;
        dir = sample_cosine_hemisphere(axis, rng);
      } else {
        BsdfSample bs = sample_bsdf(S.materials[prev->mat], prev->n, prev->wi, rng);
        if (!bs.valid || bs.pdf <= 0.0) {
          c.escaped = true;
          c.q = 1.0;
          return;
        }
        dir = bs.wo;
      }
      Hit hit;
      if (!intersect(S, prev->p, dir, hit)) {
        c.escaped = true;
        c.q = 1.0;
        return;
      }
      c.g[j] = vertex_from_hit(S, hit, -dir);
      prev = &c.g[j];
    }
  }
  c.q = support_pdf(S, h, prefix, c.g);
  if (!(c.q > 0.0)) {
    c.escaped = true;
    c.q = 1.0;
  }
}

// target_density (proxy.cpp:106-151); g has exactly u vertices.
template <class Vis>
__device__ __forceinline__ double target_density_v(const SceneView& S, const IncHdr& h, const PV* prefix, const PV* g,
                                                   const Vis& vis) {
  const int u = h.u;
  for (int i = 0; i + 1 < u; ++i)
    if (!specmat(S, g[i])) return 0.0;
  if (specmat(S, g[u - 1])) return 0.0;
  const PV* hc = inc_control(h, prefix);
  if (hc == nullptr && g[u - 1].emitter < 0) return 0.0;
  // chain: [control] g_{u-1} ... g_0 endpoint
  const PV* chain[6];
  int m = 0;
  if (hc) chain[m++] = hc;
  for (int i = u - 1; i >= 0; --i) chain[m++] = &g[i];
  chain[m++] = &h.spec_end;
  double f = hc ? 1.0 : 1.0 / S.total_emitter_area;
  {
    const PV& a = *chain[0];
    const PV& b = *chain[1];
    V3 d = b.p - a.p;
    double len = length(d);
    if (len <= 0.0) return 0.0;
    V3 dir = d / len;
    double pdf_w = (!hc || !h.has_cdir) ? light_direction_pdf(a.n, dir)
                                        : pdf_bsdf(S.materials[a.mat], a.n, -h.cdir, dir);
    if (pdf_w <= 0.0 || !vis(5, a.p, b.p)) return 0.0;
    f *= to_area_density(pdf_w, a.p, b.p, b.n);
  }
  for (int k = 1; k + 1 < m; ++k) {
    const PV& a = *chain[k];
    const PV& b = *chain[k + 1];
    V3 wi = normalize(chain[k - 1]->p - a.p);
    V3 d = b.p - a.p;
    double len = length(d);
    if (len <= 0.0) return 0.0;
    double pdf_w = pdf_bsdf(S.materials[a.mat], a.n, wi, d / len);
    if (pdf_w <= 0.0 || !vis(5 + k, a.p, b.p)) return 0.0;
    f *= to_area_density(pdf_w, a.p, b.p, b.n);
  }
  return f;
}

__device__ __forceinline__ double target_density(const SceneView& S, const IncHdr& h, const PV* prefix, const PV* g) {
  return target_density_v(S, h, prefix, g, VisDirect{&S});
}


// recip::Walk::draw_g (recip.hpp:69-77) for the proxy integrand.
__device__ __forceinline__ double draw_g(const SceneView& S, const IncHdr& h, const PV* prefix, double bound,
                                         Rng& rng, int& err) {
  Cand c;
  support_sample(S, h, prefix, rng, c);
  const double qx = c.q;
  const double fx = c.escaped ? 0.0 : target_density(S, h, prefix, c.g);
  if (!isfinite(fx) || fx < 0.0) err = kErrIntegrand;
  else if (!isfinite(qx) || qx <= 0.0) err = kErrSupport;
  return 1.0 - fx / (bound * qx);
}

// retrace_proxy (proxy.cpp:271-319). g receives u vertices; returns density (> 0) or 0.
__device__ __forceinline__ double retrace_proxy(const SceneView& S, const IncHdr& h, const PV* prefix, const PV& z,
                                                Rng& rng, PV* g) {
  const int u = h.u;
  V3 d0 = z.p - h.spec_end.p;
  double l0 = length(d0);
  if (l0 <= 0.0) return 0.0;
  PV cur = h.spec_end;
  V3 wi = d0 / l0;
  double density = 1.0;
  for (int step = 0; step < u; ++step) {
    BsdfSample bs = sample_bsdf(S.materials[cur.mat], cur.n, wi, rng);
    if (!bs.valid || bs.pdf <= 0.0) return 0.0;
    Hit hit;
    if (!intersect(S, cur.p, bs.wo, hit)) return 0.0;
    PV v = vertex_from_hit(S, hit, -bs.wo);
    density *= to_area_density(bs.pdf, cur.p, v.p, v.n);
    const bool terminal = step == u - 1;
    if (!terminal) {
      if (!specmat(S, v)) return 0.0;
    } else {
      if (specmat(S, v)) return 0.0;
      if (h.dflag_last == kLight) {
        if (v.emitter < 0) return 0.0;
        v.flag = kLight;
      }
    }
    v.pdf_fwd = to_area_density(bs.pdf, cur.p, v.p, v.n);
    g[step] = v;
    wi = v.wi;
    cur = v;
  }
  if (!(density > 0.0)) return 0.0;
  for (int j = 0; j + 1 < u; ++j) g[j].wi = normalize(g[j + 1].p - g[j].p);
  const PV* hc = inc_control(h, prefix);
  g[u - 1].wi = hc ? normalize(hc->p - g[u - 1].p) : v3(0.0);
  return density;
}

// proxy_connect (proxy.cpp:548-603). eye: the pixel's eye sub-path (strided view) cut at
// tp vertices. lv: scratch for the repaired light sub-path (kMaxLight).
__device__ __forceinline__ V3 proxy_connect(const SceneView& S, const Mapper& M, const StatsView& st,
                                            const PV* eye, size_t es, int t, const IncHdr& h, const PV* prefix,
                                            Rng& rng, PV* lv) {
  if (t < 2) return v3(0.0);
  const PV& z = eye[(t - 1) * es];
  if (z.flag != kDiffuse) return v3(0.0);
  for (int i = 1; i + 1 < t; ++i)
    if (eye[i * es].flag != kSpecular) return v3(0.0);
  if (!(h.inverse_p > 0.0) || !(h.prefix_pdf > 0.0)) return v3(0.0);
  PV g[4];
  const double density = retrace_proxy(S, h, prefix, z, rng, g);
  if (!(density > 0.0)) return v3(0.0);
  // repair (proxy.cpp:96-104)
  int s = 0;
  for (int i = 0; i < h.n_prefix; ++i) lv[s++] = prefix[i];
  for (int i = h.u - 1; i >= 0; --i) lv[s++] = g[i];
  lv[s++] = h.spec_end;

  V3 d01 = lv[1].p - lv[0].p;
  double l01 = length(d01);
  if (l01 <= 0.0 || lv[0].emitter < 0) return v3(0.0);
  V3 value = emitted(S, lv[0].emitter, lv[0].n, d01 / l01);
  if (near_zero(value)) return v3(0.0);
  for (int i = 0; i + 1 < s; ++i) {
    double gt = geometry_term(S, lv[i], lv[i + 1]);
    if (gt <= 0.0) return v3(0.0);
    value = value * gt;
  }
  double gj = geometry_term(S, lv[s - 1], z);
  if (gj <= 0.0) return v3(0.0);
  value = value * gj;
  for (int i = 1; i < s; ++i) {
    V3 wi = normalize(lv[i - 1].p - lv[i].p);
    V3 to = i + 1 < s ? lv[i + 1].p : z.p;
    V3 wo = normalize(to - lv[i].p);
    V3 fk = eval_bsdf(S.materials[lv[i].mat], lv[i].n, wi, wo);
    if (near_zero(fk)) return v3(0.0);
    value = value * fk;
  }
  V3 fz = eval_bsdf(S.materials[z.mat], z.n, z.wi, normalize(lv[s - 1].p - z.p));
  if (near_zero(fz)) return v3(0.0);
  value = value * fz * z.thr;
  FullPath fp = make_fp(lv, 1, eye, es, s, t);
  const double w = reciprocal_mis_weight(S, M, st, fp, -1, true);
  if (!(w > 0.0)) return v3(0.0);
  return value * (h.inverse_p * w / (h.prefix_pdf * density));
}

#endif  // __CUDACC__

}  // namespace pxg
