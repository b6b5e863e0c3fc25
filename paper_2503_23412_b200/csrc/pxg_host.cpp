// pxg_host.cpp — one-time host work of pxg_create: Scene::finalize and the BVH build.
//
// finalize mirrors proj/src/scene.cpp:234-252 with the reference's fp64 operation order
// (compiled with -ffp-contract=off) so the emitter areas, their running sums, the scene
// bbox that the subspace grid is built on, and the camera basis are bit-identical.
//
// The BVH is this library's own: a binned-SAH binary tree whose nodes store both child
// boxes in fp32 (64 B per node), rounded outward and padded so that the fp32 slab test is
// conservative for every fp64 hit (see pxg_scene.cuh). The reference's median-split BVH
// (scene.cpp:254-295) is private and only affects its traversal order, not hit ids.
#include "pxg_host.h"

#include <algorithm>
#include <atomic>
#include <thread>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numbers>
#include <stdexcept>

namespace pxg {

namespace {

struct D3 {
  double x, y, z;
};
inline D3 add(D3 a, D3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline D3 sub(D3 a, D3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline D3 mul(D3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double dot3(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline D3 cross3(D3 a, D3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
inline double len3(D3 a) { return std::sqrt(dot3(a, a)); }
inline D3 norm3(D3 a) { return mul(a, 1.0 / len3(a)); }
inline D3 vmin(D3 a, D3 b) { return {std::min(a.x, b.x), std::min(a.y, b.y), std::min(a.z, b.z)}; }
inline D3 vmax(D3 a, D3 b) { return {std::max(a.x, b.x), std::max(a.y, b.y), std::max(a.z, b.z)}; }
inline D3 ld(const double* p) { return {p[0], p[1], p[2]}; }
inline double comp(D3 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : v.z); }

// Primitive::area (scene.cpp:107-114)
double prim_area(int shape, D3 a, D3 b, D3 c, double r) {
  switch (shape) {
    case 0: return 4.0 * std::numbers::pi * r * r;
    case 1: return 0.5 * len3(cross3(sub(b, a), sub(c, a)));
    default: return len3(cross3(b, c));
  }
}

// primitive_bounds (scene.cpp:74-89)
void prim_bounds(int shape, D3 a, D3 b, D3 c, double r, D3& lo, D3& hi) {
  if (shape == 0) {
    lo = sub(a, D3{r, r, r});
    hi = add(a, D3{r, r, r});
  } else if (shape == 1) {
    lo = vmin(a, vmin(b, c));
    hi = vmax(a, vmax(b, c));
  } else {
    D3 ab = add(a, b), ac = add(a, c), abc = add(add(a, b), c);
    lo = vmin(vmin(a, ab), vmin(ac, abc));
    hi = vmax(vmax(a, ab), vmax(ac, abc));
  }
}

struct BPrim {
  D3 lo, hi, cen;
  int id;
};

struct Box {
  D3 lo{1e300, 1e300, 1e300}, hi{-1e300, -1e300, -1e300};
  void grow(const D3& l, const D3& h) {
    lo = vmin(lo, l);
    hi = vmax(hi, h);
  }
  double area() const {
    if (hi.x < lo.x) return 0.0;
    D3 e = sub(hi, lo);
    return 2.0 * (e.x * e.y + e.y * e.z + e.z * e.x);
  }
};

struct Builder {
  std::vector<BPrim>& prims;
  std::vector<HostNode>& nodes;
  std::vector<int>& order;
  double pad;
  int max_depth_seen = 0;

  static float down(double v, double pad) {
    float f = static_cast<float>(v - pad);
    return std::nextafter(f, -INFINITY);
  }
  static float up(double v, double pad) {
    float f = static_cast<float>(v + pad);
    return std::nextafter(f, INFINITY);
  }

  void set_child(HostNode& n, int k, const Box& b, int code) {
    float* lo = k == 0 ? n.lo0 : n.lo1;
    float* hi = k == 0 ? n.hi0 : n.hi1;
    lo[0] = down(b.lo.x, pad); lo[1] = down(b.lo.y, pad); lo[2] = down(b.lo.z, pad);
    hi[0] = up(b.hi.x, pad); hi[1] = up(b.hi.y, pad); hi[2] = up(b.hi.z, pad);
    (k == 0 ? n.c0 : n.c1) = code;
  }

  int leaf_code(int first, int count) {
    for (int i = 0; i < count; ++i) order.push_back(prims[first + i].id);
    int base = static_cast<int>(order.size()) - count;
    return ~(base * 16 + count);
  }

  // Builds [first, first+count) and returns the child code referencing it.
  int leaf_max = 1;  // measured best on C2 (fp64 primitive tests dominate); PXG_LEAF overrides

  // Binned SAH split of [first, first+count): partitions the range, returns mid and the
  // child boxes. PXG_SAH_BINS overrides the bin count (tuning experiments).
  static constexpr int kMaxBins = 64;
  // Bins of one range for all three axes at once: one pass over the primitives (chunks of a
  // large range binned on worker threads and merged), the SAH sweep per axis, then one
  // partition pass; the child boxes come from the sweep (unions of primitive boxes, exact).
  struct Bins {
    Box bb[3][kMaxBins];
    int cnt[3][kMaxBins] = {};
  };
  static void bin_range(const BPrim* p, int count, const D3& clo, const double* scale, int nb, Bins& B) {
    for (int i = 0; i < count; ++i) {
      const BPrim& q = p[i];
      const double c[3] = {q.cen.x, q.cen.y, q.cen.z};
      const double l[3] = {clo.x, clo.y, clo.z};
      for (int a = 0; a < 3; ++a) {
        const int b = std::min(nb - 1, std::max(0, static_cast<int>((c[a] - l[a]) * scale[a])));
        B.bb[a][b].grow(q.lo, q.hi);
        ++B.cnt[a][b];
      }
    }
  }

  void split(int first, int count, int& mid, Box& lb, Box& rb) {
    static const int kBins = std::getenv("PXG_SAH_BINS") ? std::max(2, std::min(kMaxBins, std::atoi(std::getenv("PXG_SAH_BINS")))) : 16;
    const BPrim* P = prims.data() + first;
    Box cb;
    for (int i = 0; i < count; ++i) cb.grow(P[i].cen, P[i].cen);
    double scale[3];
    bool ok[3];
    for (int a = 0; a < 3; ++a) {
      const double lo = comp(cb.lo, a), hi = comp(cb.hi, a);
      ok[a] = hi > lo;
      scale[a] = ok[a] ? kBins / (hi - lo) : 0.0;
    }
    Bins B;
    constexpr int kParBin = 1 << 16;
    if (count >= kParBin) {
      const int T = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
      std::vector<Bins> part(T);
      std::vector<std::thread> th;
      const int chunk = (count + T - 1) / T;
      for (int t = 0; t < T; ++t) {
        const int s0 = t * chunk, s1 = std::min(count, s0 + chunk);
        if (s0 >= s1) break;
        th.emplace_back([&, t, s0, s1]() { bin_range(P + s0, s1 - s0, cb.lo, scale, kBins, part[t]); });
      }
      for (auto& x : th) x.join();
      for (const Bins& q : part)
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < kBins; ++b) {
            if (q.cnt[a][b]) B.bb[a][b].grow(q.bb[a][b].lo, q.bb[a][b].hi);
            B.cnt[a][b] += q.cnt[a][b];
          }
    } else {
      bin_range(P, count, cb.lo, scale, kBins, B);
    }
    mid = -1;
    double best_cost = INFINITY;
    int best_axis = -1, best_bin = -1;
    Box best_l, best_r;
    for (int axis = 0; axis < 3; ++axis) {
      if (!ok[axis]) continue;
      Box left[kMaxBins];
      int lc[kMaxBins];
      Box acc;
      int ac = 0;
      for (int b = 0; b < kBins; ++b) {
        if (B.cnt[axis][b]) acc.grow(B.bb[axis][b].lo, B.bb[axis][b].hi);
        ac += B.cnt[axis][b];
        left[b] = acc;
        lc[b] = ac;
      }
      Box racc;
      int rc = 0;
      for (int b = kBins - 1; b >= 1; --b) {
        if (B.cnt[axis][b]) racc.grow(B.bb[axis][b].lo, B.bb[axis][b].hi);
        rc += B.cnt[axis][b];
        if (lc[b - 1] == 0 || rc == 0) continue;
        double cost = left[b - 1].area() * lc[b - 1] + racc.area() * rc;
        if (cost < best_cost) {
          best_cost = cost;
          best_axis = axis;
          best_bin = b;
          best_l = left[b - 1];
          best_r = racc;
        }
      }
    }
    if (best_axis >= 0) {
      const double lo = comp(cb.lo, best_axis), sc = scale[best_axis];
      auto it = std::partition(prims.begin() + first, prims.begin() + first + count, [&](const BPrim& p) {
        int b = std::min(kBins - 1, std::max(0, static_cast<int>((comp(p.cen, best_axis) - lo) * sc)));
        return b < best_bin;
      });
      mid = static_cast<int>(it - prims.begin());
      if (mid == first || mid == first + count) mid = -1;
    }
    if (mid >= 0) {
      lb = best_l;
      rb = best_r;
      return;
    }
    mid = first + count / 2;  // degenerate centroids: split by position
    for (int i = first; i < mid; ++i) lb.grow(prims[i].lo, prims[i].hi);
    for (int i = mid; i < first + count; ++i) rb.grow(prims[i].lo, prims[i].hi);
  }

  int build(int first, int count, const Box& bounds, int depth) {
    max_depth_seen = std::max(max_depth_seen, depth);
    if (count <= leaf_max || depth >= 56) {
      if (count <= 15) return leaf_code(first, count);
    }
    int mid;
    Box lb, rb;
    split(first, count, mid, lb, rb);
    const int idx = static_cast<int>(nodes.size());
    nodes.push_back(HostNode{});
    int cl = build(first, mid - first, lb, depth + 1);
    int cr = build(mid, first + count - mid, rb, depth + 1);
    set_child(nodes[idx], 0, lb, cl);
    set_child(nodes[idx], 1, rb, cr);
    return idx;
  }

  // Parallel build (same tree as build(), node indices in a different order): the top
  // levels are split here; every subtree below depth kParDepth (or smaller than kParMin
  // primitives) is deferred, built by a worker thread into its own vectors, and spliced in.
  struct Pending {
    int first, count, depth, parent, side;
    Box bounds;
  };
  static constexpr int kParDepth = 5, kParMin = 2048;

  int plan(int first, int count, const Box& bounds, int depth, int parent, int side, std::vector<Pending>& pend) {
    max_depth_seen = std::max(max_depth_seen, depth);
    if (parent >= 0 && (depth >= kParDepth || count <= kParMin)) {
      pend.push_back(Pending{first, count, depth, parent, side, bounds});
      return 0;  // patched after the splice
    }
    if (count <= leaf_max || depth >= 56) {
      if (count <= 15) return leaf_code(first, count);
    }
    int mid;
    Box lb, rb;
    split(first, count, mid, lb, rb);
    const int idx = static_cast<int>(nodes.size());
    nodes.push_back(HostNode{});
    int cl = plan(first, mid - first, lb, depth + 1, idx, 0, pend);
    int cr = plan(mid, first + count - mid, rb, depth + 1, idx, 1, pend);
    set_child(nodes[idx], 0, lb, cl);
    set_child(nodes[idx], 1, rb, cr);
    return idx;
  }

  void build_parallel(int n, const Box& all) {
    std::vector<Pending> pend;
    plan(0, n, all, 0, -1, 0, pend);  // nodes is empty, so the root lands in slot 0
    struct Part {
      std::vector<HostNode> nodes;
      std::vector<int> order;
      int root = 0, depth = 0;
    };
    std::vector<Part> parts(pend.size());
    std::atomic<size_t> next{0};
    auto work = [&]() {
      for (size_t t; (t = next.fetch_add(1)) < pend.size();) {
        Part& P = parts[t];
        Builder sub{prims, P.nodes, P.order, pad};
        sub.leaf_max = leaf_max;
        P.root = sub.build(pend[t].first, pend[t].count, pend[t].bounds, pend[t].depth);
        P.depth = sub.max_depth_seen;
      }
    };
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned i = 1; i < hw && i < pend.size(); ++i) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    for (size_t t = 0; t < pend.size(); ++t) {
      const Part& P = parts[t];
      const int node_off = static_cast<int>(nodes.size()), order_off = static_cast<int>(order.size());
      auto remap = [&](int code) {
        if (code >= 0) return code + node_off;
        const int x = ~code;
        return ~((((x >> 4) + order_off) << 4) | (x & 15));
      };
      for (HostNode nd : P.nodes) {
        nd.c0 = remap(nd.c0);
        nd.c1 = remap(nd.c1);
        nodes.push_back(nd);
      }
      order.insert(order.end(), P.order.begin(), P.order.end());
      HostNode& par = nodes[pend[t].parent];
      (pend[t].side == 0 ? par.c0 : par.c1) = remap(P.root);
      max_depth_seen = std::max(max_depth_seen, P.depth);
    }
  }
};

// Collapses the binary BVH into a 4-wide one: each wide node takes up to four descendants,
// always opening the internal child with the largest box surface (the usual collapse
// heuristic). Child boxes are copied from the binary nodes, so they stay conservative.
struct Collapser {
  const std::vector<HostNode>& bin;
  std::vector<HostNode4>& out;

  struct Child {
    float lo[3], hi[3];
    int code;
  };

  static float area(const Child& c) {
    if (c.hi[0] < c.lo[0]) return -1.f;
    const float ex = c.hi[0] - c.lo[0], ey = c.hi[1] - c.lo[1], ez = c.hi[2] - c.lo[2];
    return ex * ey + ey * ez + ez * ex;
  }

  Child child_of(int node, int k) const {
    const HostNode& n = bin[node];
    Child c;
    for (int a = 0; a < 3; ++a) {
      c.lo[a] = k == 0 ? n.lo0[a] : n.lo1[a];
      c.hi[a] = k == 0 ? n.hi0[a] : n.hi1[a];
    }
    c.code = k == 0 ? n.c0 : n.c1;
    return c;
  }

  int build(int node) {
    Child ch[4];
    int m = 0;
    ch[m++] = child_of(node, 0);
    ch[m++] = child_of(node, 1);
    while (m < 4) {
      int best = -1;
      float best_area = -1.f;
      for (int k = 0; k < m; ++k)
        if (ch[k].code >= 0 && area(ch[k]) > best_area) {
          best = k;
          best_area = area(ch[k]);
        }
      if (best < 0) break;
      const int b = ch[best].code;
      ch[best] = child_of(b, 0);
      ch[m++] = child_of(b, 1);
    }
    const int idx = static_cast<int>(out.size());
    out.push_back(HostNode4{});
    int codes[4];
    for (int k = 0; k < 4; ++k) {
      if (k < m && ch[k].code >= 0) codes[k] = build(ch[k].code);
      else codes[k] = k < m ? ch[k].code : ~0;
    }
    HostNode4& w = out[idx];
    for (int k = 0; k < 4; ++k) {
      for (int a = 0; a < 3; ++a) {
        w.lo[a][k] = k < m ? ch[k].lo[a] : 1e30f;
        w.hi[a][k] = k < m ? ch[k].hi[a] : -1e30f;
      }
      w.child[k] = codes[k];
    }
    return idx;
  }
};

// Quantises a 4-wide node's child boxes to 8 bits per plane: origin = the lower corner of
// the children's union (fp32), grid step 2^e per axis with 255 * 2^e >= extent, lower planes
// rounded down and upper planes rounded up, so every decoded box contains its fp32 box
// (checked exactly in double). Empty children (lo > hi) keep their codes, which test nothing.
HostNode4Q quantize_node(const HostNode4& w) {
  HostNode4Q q{};
  float ulo[3] = {INFINITY, INFINITY, INFINITY}, uhi[3] = {-INFINITY, -INFINITY, -INFINITY};
  bool valid[4];
  for (int k = 0; k < 4; ++k) {
    valid[k] = w.lo[0][k] <= w.hi[0][k] && w.lo[1][k] <= w.hi[1][k] && w.lo[2][k] <= w.hi[2][k];
    if (!valid[k]) continue;
    for (int a = 0; a < 3; ++a) {
      ulo[a] = std::min(ulo[a], w.lo[a][k]);
      uhi[a] = std::max(uhi[a], w.hi[a][k]);
    }
  }
  for (int a = 0; a < 3; ++a) {
    if (!(ulo[a] <= uhi[a])) ulo[a] = uhi[a] = 0.f;
    q.origin[a] = ulo[a];
    const double ext = static_cast<double>(uhi[a]) - static_cast<double>(ulo[a]);
    int e = -126;
    if (ext > 0.0) e = std::max(-126, std::ilogb(ext / 255.0) - 1);  // then at most a few steps up
    while (e < 127 && std::ldexp(255.0, e) < ext) ++e;
    q.exps |= static_cast<unsigned>(e + 127) << (8 * a);
    const double step = std::ldexp(1.0, e);
    for (int k = 0; k < 4; ++k) {
      unsigned lo = 255u, hi = 0u;
      if (valid[k]) {
        const double l = std::floor((static_cast<double>(w.lo[a][k]) - ulo[a]) / step);
        const double u = std::ceil((static_cast<double>(w.hi[a][k]) - ulo[a]) / step);
        lo = static_cast<unsigned>(std::max(0.0, std::min(255.0, l)));
        hi = static_cast<unsigned>(std::max(0.0, std::min(255.0, u)));
        if (!(static_cast<double>(ulo[a]) + lo * step <= w.lo[a][k] && static_cast<double>(ulo[a]) + hi * step >= w.hi[a][k]))
          throw std::runtime_error("quantize_node: box not contained");
      }
      q.qlo[a] |= lo << (8 * k);
      q.qhi[a] |= hi << (8 * k);
    }
  }
  for (int k = 0; k < 4; ++k) {
    q.child[k] = w.child[k];
    if (w.child[k] < 0) q.exps |= 1u << (24 + k);  // bits 24-27: child k is a leaf (or empty: never hit)
  }
  return q;
}

}  // namespace

void finalize_scene(const SceneDesc& d, SceneHost& h) {
  const int n = d.n_prims;
  if (n <= 0) throw std::runtime_error("scene: no primitives defined");
  if (d.n_emitters <= 0) throw std::runtime_error("scene: scene must contain at least one emitter");
  if (d.width <= 0 || d.height <= 0) throw std::runtime_error("scene: resolution must be positive");
  h.prim_emitter.assign(n, -1);
  h.prim_mat.assign(d.material, d.material + n);
  h.prim_shape.assign(d.shape, d.shape + n);
  for (int i = 0; i < n; ++i) {
    if (d.material[i] < 0 || d.material[i] >= d.n_materials)
      throw std::runtime_error("scene: unknown material");
    if (d.shape[i] < 0 || d.shape[i] > 2) throw std::runtime_error("scene: unknown shape");
  }
  // emitters, areas and running sums in the reference order
  double total = 0.0;
  h.emitter_cum.resize(d.n_emitters);
  for (int e = 0; e < d.n_emitters; ++e) {
    const int p = d.emitter_prim[e];
    if (p < 0 || p >= n) throw std::runtime_error("scene: emitter references unknown primitive");
    h.prim_emitter[p] = e;
    total += prim_area(d.shape[p], ld(d.a + 3 * p), ld(d.b + 3 * p), ld(d.c + 3 * p), d.radius[p]);
  }
  // sample_light_point re-sums areas in emitter order with its own accumulator; the
  // running values are identical to the finalize sum's prefixes.
  double acc = 0.0;
  for (int e = 0; e < d.n_emitters; ++e) {
    const int p = d.emitter_prim[e];
    acc += prim_area(d.shape[p], ld(d.a + 3 * p), ld(d.b + 3 * p), ld(d.c + 3 * p), d.radius[p]);
    h.emitter_cum[e] = acc;
  }
  // an emitter listed twice keeps the later index (emitter_of_primitive overwrite order)
  h.total_emitter_area = total;
  D3 bmin{1e30, 1e30, 1e30}, bmax{-1e30, -1e30, -1e30};
  h.prim_geo.assign(3 * static_cast<size_t>(n), 0.0);
  h.prim_center.assign(4 * static_cast<size_t>(n), 0.0);
  h.prim_abc.assign(9 * static_cast<size_t>(n), 0.0);
  std::vector<BPrim> bp(n);
  double scale = 0.0;
  for (int i = 0; i < n; ++i) {
    D3 a = ld(d.a + 3 * i), b = ld(d.b + 3 * i), c = ld(d.c + 3 * i);
    const double r = d.radius[i];
    D3 lo, hi;
    prim_bounds(d.shape[i], a, b, c, r, lo, hi);
    bmin = vmin(bmin, lo);
    bmax = vmax(bmax, hi);
    bp[i] = BPrim{lo, hi, mul(add(lo, hi), 0.5), i};
    scale = std::max({scale, std::fabs(lo.x), std::fabs(lo.y), std::fabs(lo.z), std::fabs(hi.x),
                      std::fabs(hi.y), std::fabs(hi.z)});
    D3 e1 = d.shape[i] == 1 ? sub(b, a) : b;
    D3 e2 = d.shape[i] == 1 ? sub(c, a) : c;
    double* g = &h.prim_abc[9 * static_cast<size_t>(i)];
    if (d.shape[i] == 0) {
      g[0] = a.x; g[1] = a.y; g[2] = a.z; g[3] = r;
      double* cc = &h.prim_center[4 * static_cast<size_t>(i)];
      cc[0] = a.x; cc[1] = a.y; cc[2] = a.z; cc[3] = r;
    } else {
      g[0] = a.x; g[1] = a.y; g[2] = a.z;
      g[3] = e1.x; g[4] = e1.y; g[5] = e1.z;
      g[6] = e2.x; g[7] = e2.y; g[8] = e2.z;
      // primitive_normal: triangle normalize(cross(b - a, c - a)); rectangle normalize(cross(b, c))
      D3 nn = norm3(cross3(e1, e2));
      h.prim_geo[3 * i] = nn.x; h.prim_geo[3 * i + 1] = nn.y; h.prim_geo[3 * i + 2] = nn.z;
    }
  }
  h.bbox_min[0] = bmin.x; h.bbox_min[1] = bmin.y; h.bbox_min[2] = bmin.z;
  h.bbox_max[0] = bmax.x; h.bbox_max[1] = bmax.y; h.bbox_max[2] = bmax.z;

  // camera basis (scene.cpp:116-125)
  D3 pos = ld(d.cam_position), look = ld(d.cam_look_at), up = ld(d.cam_up);
  D3 fwd = norm3(sub(look, pos));
  D3 right = norm3(cross3(fwd, up));
  D3 cup = cross3(right, fwd);
  const double v[12] = {pos.x, pos.y, pos.z, fwd.x, fwd.y, fwd.z, right.x, right.y, right.z, cup.x, cup.y, cup.z};
  std::memcpy(h.cam, v, sizeof(v));
  h.tan_half = std::tan(d.fov_y * std::numbers::pi / 360.0);
  h.aspect = static_cast<double>(d.width) / d.height;
  scale = std::max({scale, std::fabs(pos.x), std::fabs(pos.y), std::fabs(pos.z), 1.0});

  // BVH
  h.nodes.clear();
  h.order.clear();
  h.nodes.reserve(2 * static_cast<size_t>(n) / 3 + 2);
  h.order.reserve(n);
  const double pad = 1e-5 * scale;
  Builder B{bp, h.nodes, h.order, pad};
  if (const char* lm = std::getenv("PXG_LEAF")) B.leaf_max = std::max(1, std::min(15, std::atoi(lm)));
  Box all;
  for (auto& p : bp) all.grow(p.lo, p.hi);
  if (n <= 4) {
    // the root is always an internal node: one leaf child and one empty child
    h.nodes.push_back(HostNode{});
    int code = B.leaf_code(0, n);
    B.set_child(h.nodes[0], 0, all, code);
    HostNode& r = h.nodes[0];
    r.lo1[0] = r.lo1[1] = r.lo1[2] = 1e30f;
    r.hi1[0] = r.hi1[1] = r.hi1[2] = -1e30f;
    r.c1 = ~0;
    h.bvh_depth = 1;
  } else {
    B.build_parallel(n, all);
    h.bvh_depth = B.max_depth_seen;
  }
  h.nodes4.clear();
  h.nodes4.reserve(h.nodes.size() / 2 + 2);
  Collapser{h.nodes, h.nodes4}.build(0);
  // Quantised nodes halve the bytes per visit: a win once the node array outgrows the L1
  // working set (C4: 43 MB of 128 B nodes, +5.5%; C3: 4.5 MB, +3.3% since the near / far
  // plane selection of node4q_test); on the smallest scenes the 128 B nodes stay as fast or
  // faster (C2, 1 MB: -0.5% quantised). PXG_NODEQ=0/1 forces the choice.
  {
    const char* e = std::getenv("PXG_NODEQ");
    h.nodeq = e ? std::atoi(e) != 0 : h.nodes4.size() * sizeof(HostNode4) > (2u << 20);
  }
  h.nodes4q.clear();
  if (h.nodeq) {
    h.nodes4q.resize(h.nodes4.size());
    for (size_t k = 0; k < h.nodes4.size(); ++k) h.nodes4q[k] = quantize_node(h.nodes4[k]);
  }
  // leaf-ordered exact records
  h.recs.resize(n);
  for (int k = 0; k < n; ++k) {
    const int i = h.order[k];
    HostRec& r = h.recs[k];
    const double* g = &h.prim_abc[9 * static_cast<size_t>(i)];
    for (int j = 0; j < 9; ++j) r.v[j] = g[j];
    if (d.shape[i] == 0) {
      r.v[3] = d.radius[i];
      r.v[4] = r.v[5] = r.v[6] = r.v[7] = r.v[8] = 0.0;
    }
    r.shape = d.shape[i];
    r.id = i;
  }
}

}  // namespace pxg
