// ORACLE / TEST INFRASTRUCTURE ONLY. Imported by tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs; never by the product path.
//
// This file is the CPU restatement of the reference hot path
// `proxima::render_proxy_bdpt` (proj/src/proxy.cpp:647-834) that the GPU is checked
// against. It is linked with the UNMODIFIED reference sources (proj/src/*.cpp, built by
// oracle/Makefile) and calls only their public functions for the leaves (traversal,
// BSDFs, sub-paths, dropout, support sampling, reciprocal runs, proxy_connect ...).
//
// Two documented deviations from the reference loop, both required for any parallel
// implementation:
//   (1) streams the reference draws sequentially — pool walks + reservoir + all
//       estimate_inverse_p calls on `pool_rng` (proxy.cpp:691-721) and the 20,000
//       pretrace walks on one stream (proxy.cpp:669) — are re-keyed per unit of work
//       (walk, reservoir key, probe set, reciprocal run) with the PXG_KIND_* streams of
//       include/pxg_philox.h. Pixel streams (proxy.cpp:664-666) and proxy streams
//       (proxy.cpp:759-760) keep the reference's own ids.
//   (2) Algorithm R (proxy.cpp:703-709) is replaced by the distributionally identical
//       priority reservoir: keep the `pool_budget` smallest i.i.d. 64-bit keys; kept
//       entries are ordered by (walk, prefix end). kappa is unchanged.
// Everything else — the sequential B-bound semantics, the per-cell gate order, the
// pixel-order gamma accumulation — follows the reference exactly.
//
// Built twice: with the Philox shadow rng.hpp (parity oracle, liboracle.so) and with the
// reference's own PCG rng.hpp and ORC_PCG defined (liboracle_pcg.so: only the unmodified
// reference entry points, used to time the reference CPU path as shipped).

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "proxima/proxy.hpp"
#include "proxima/recip.hpp"
#include "proxima/scene.hpp"
#include "proxima/subspace.hpp"
#include "proxima/transport.hpp"

#define ORC_API extern "C" __attribute__((visibility("default")))

using namespace proxima;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}

struct OrcScene {
  Scene scene;
};

// Runs fn(i) for i in [0, n) on `threads` workers; deterministic because every unit
// writes only its own outputs. The first exception is rethrown on the caller.
void parallel_for(int n, int threads, const std::function<void(int)>& fn) {
  if (threads <= 1 || n < 2) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int> next{0};
  std::exception_ptr err;
  std::mutex mu;
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&]() {
      for (;;) {
        int i = next.fetch_add(1);
        if (i >= n) break;
        try {
          fn(i);
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu);
          if (!err) err = std::current_exception();
          next.store(n);
        }
      }
    });
  }
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace

extern "C" {

struct OrcParams {
  int enabled;
  int pool_budget;
  int recip_repeats;
  int freeze_iteration;
  long long recursion_cap;
  int pretrace_paths;
  int light_walks;
  double gate_high;
  double gate_low;
  double gate_threshold;
};

// Dense bucket index of StatsKey{u,c,s}: ((u-1)*10 + c)*100 + s, 4000 buckets.
struct OrcTrace {
  int n_passes_cap;      // capacity of the per-pass arrays below
  double* pass_val;      // [pass][px][3] final per-pixel sample value
  double* pass_bdpt;     // [pass][px][3] standard-strategy value (before the proxy term)
  double* pass_c;        // [pass][px][3] proxy_connect value (speculative: gate not applied)
  int* pass_flags;       // [pass][px] bit0 tp>=2, bit1 attempted, bit2 gate passed, bit3 contributed
  int trace_pass;        // pass whose sub-path primitive ids are recorded (-1: none)
  int* eye_prims;        // [px][max_depth+1] primitive id per eye vertex, -1 pad (camera = -1)
  int* light_prims;      // [px][max_depth-1]
  int pool_cap;          // capacity per pass of the pool arrays
  long long* pool_raw;   // [pass]
  int* pool_n;           // [pass] entries kept after the reciprocal estimate
  int* pool_walk;        // [pass][pool_cap]
  int* pool_end;         // [pass][pool_cap]
  int* pool_key;         // [pass][pool_cap] dense bucket index
  double* pool_inv_p;    // [pass][pool_cap]
  double* pool_inv_p_m2; // [pass][pool_cap]
  double* pool_bound;    // [pass][pool_cap] B used by the reciprocal runs
  double* pretrace_max;  // [4000] bucket max f/q after the pretrace
  long long* pretrace_cnt;  // [4000]
  double* stats_out;     // [4000][3] max_ratio, sum_est, sum_est_sq at the end
  long long* stats_cnt;  // [4000][2] ratio_count, est_count at the end
  double* gamma_rows;    // [32][100] at the end
  long long* diag;       // [4000][5] retrace_attempts, accepts, recip_runs, truncated, failed
  long long* diag_pool;  // [2] pool_raw, pool_kept
};

ORC_API const char* orc_last_error() { return g_err.c_str(); }

ORC_API void* orc_scene_load(const char* json_text) {
  try {
    auto* s = new OrcScene{load_scene_from_string(json_text)};
    return s;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

ORC_API void orc_scene_free(void* h) { delete static_cast<OrcScene*>(h); }

ORC_API int orc_scene_info(void* h, int* ints /*[6]*/, double* dbl /*[7]*/) {
  const Scene& sc = static_cast<OrcScene*>(h)->scene;
  ints[0] = sc.camera.width;
  ints[1] = sc.camera.height;
  ints[2] = sc.settings.max_depth;
  ints[3] = static_cast<int>(sc.primitives.size());
  ints[4] = static_cast<int>(sc.emitters.size());
  ints[5] = sc.settings.spp;
  dbl[0] = sc.total_emitter_area;
  dbl[1] = sc.bbox_min.x; dbl[2] = sc.bbox_min.y; dbl[3] = sc.bbox_min.z;
  dbl[4] = sc.bbox_max.x; dbl[5] = sc.bbox_max.y; dbl[6] = sc.bbox_max.z;
  return 0;
}

// Scene::intersect (proj/src/scene.cpp:127-150) on n rays [ox oy oz dx dy dz].
ORC_API int orc_intersect(void* h, int n, const double* rays, const double* tmax, int* prim,
                          double* t, int threads) {
  try {
    const Scene& sc = static_cast<OrcScene*>(h)->scene;
    parallel_for(n, threads, [&](int i) {
      const double* r = rays + 6 * static_cast<size_t>(i);
      Ray ray{{r[0], r[1], r[2]}, {r[3], r[4], r[5]}};
      auto hit = sc.intersect(ray, tmax ? tmax[i] : 1e30);
      prim[i] = hit ? hit->primitive : -1;
      t[i] = hit ? hit->t : 0.0;
    });
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Scene::occluded (proj/src/scene.cpp:170-177) on n segments [from xyz, to xyz].
ORC_API int orc_occluded(void* h, int n, const double* seg, int* occ, int threads) {
  try {
    const Scene& sc = static_cast<OrcScene*>(h)->scene;
    parallel_for(n, threads, [&](int i) {
      const double* s = seg + 6 * static_cast<size_t>(i);
      occ[i] = sc.occluded({s[0], s[1], s[2]}, {s[3], s[4], s[5]}) ? 1 : 0;
    });
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Unmodified reference renderers (proj/src/transport.cpp:374-386).
ORC_API int orc_render_bdpt(void* h, int spp, unsigned long long seed, double* rgb) {
  try {
    Image img = render_bdpt(static_cast<OrcScene*>(h)->scene, spp, seed);
    std::memcpy(rgb, img.pixels.data(), img.pixels.size() * sizeof(Vec3));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

ORC_API int orc_render_pt(void* h, int spp, unsigned long long seed, double* rgb) {
  try {
    Image img = render_pt(static_cast<OrcScene*>(h)->scene, spp, seed);
    std::memcpy(rgb, img.pixels.data(), img.pixels.size() * sizeof(Vec3));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

static ProxyParams to_params(const OrcParams* p) {
  ProxyParams pp;
  if (!p) return pp;
  pp.enabled = p->enabled != 0;
  pp.pool_budget = p->pool_budget;
  pp.recip_repeats = p->recip_repeats;
  pp.freeze_iteration = p->freeze_iteration;
  pp.recursion_cap = p->recursion_cap;
  pp.pretrace_paths = p->pretrace_paths;
  pp.light_walks = p->light_walks;
  pp.gate_high = p->gate_high;
  pp.gate_low = p->gate_low;
  pp.gate_threshold = p->gate_threshold;
  return pp;
}

// The unmodified reference `render_proxy_bdpt` (proj/src/proxy.cpp:647-834): the
// statistical oracle, and (PCG build) the CPU path the reference arm times.
ORC_API int orc_render_proxy_ref(void* h, int spp, unsigned long long seed, const OrcParams* p,
                                 double* rgb, long long* pool_raw_kept) {
  try {
    ProxyDiagnostics diag;
    Image img = render_proxy_bdpt(static_cast<OrcScene*>(h)->scene, spp, seed, to_params(p),
                                  &diag);
    std::memcpy(rgb, img.pixels.data(), img.pixels.size() * sizeof(Vec3));
    if (pool_raw_kept) {
      pool_raw_kept[0] = diag.pool_raw;
      pool_raw_kept[1] = diag.pool_kept;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Runs `copies` independent unmodified reference renders on `copies` threads (distinct
// seeds seed+i); used to time the single-threaded reference on every host core.
ORC_API int orc_render_proxy_ref_mt(void* h, int spp, unsigned long long seed, const OrcParams* p,
                                    int copies, double* rgb0, double* rgb_all) {
  try {
    const Scene& sc = static_cast<OrcScene*>(h)->scene;
    ProxyParams pp = to_params(p);
    std::vector<Image> imgs(copies);
    parallel_for(copies, copies, [&](int i) {
      imgs[i] = render_proxy_bdpt(sc, spp, seed + static_cast<unsigned long long>(i), pp);
    });
    if (rgb0) std::memcpy(rgb0, imgs[0].pixels.data(), imgs[0].pixels.size() * sizeof(Vec3));
    if (rgb_all)
      for (int i = 0; i < copies; ++i)
        std::memcpy(rgb_all + static_cast<size_t>(i) * imgs[i].pixels.size() * 3, imgs[i].pixels.data(),
                    imgs[i].pixels.size() * sizeof(Vec3));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Copy of a loaded scene rendered at another resolution (same geometry, camera pose and
// settings; Camera::width / height are plain members, proj/include/proxima/scene.hpp:43-44).
ORC_API void* orc_scene_with_resolution(void* h, int width, int height) {
  try {
    auto* src = static_cast<OrcScene*>(h);
    auto* c = new OrcScene(*src);
    c->scene.camera.width = width;
    c->scene.camera.height = height;
    return c;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// `copies` independent unmodified reference renders of `spp` passes on `copies` threads,
// copy i of scene hs[i] with seed seed+i, each with a pass_done callback (the reference's
// progressive-render hook, proj/include/proxima/proxy.hpp:197-200) that records the time since
// the common start: pass_end[i * spp + p] = seconds at the end of pass p of copy i. The
// steady-state time of one pass is pass_end[p] - pass_end[p-1] for p >= 1 (pass 0 also holds
// the render's one-time pretrace and the gate's first pass).
ORC_API int orc_render_proxy_ref_timed(void* const* hs, int spp, unsigned long long seed, const OrcParams* p,
                                       int copies, double* pass_end) {
  try {
    ProxyParams pp = to_params(p);
    const auto t0 = std::chrono::steady_clock::now();
    parallel_for(copies, copies, [&](int i) {
      const Scene& sc = static_cast<OrcScene*>(hs[i])->scene;
      auto cb = [&, i](int done, const Image&) {
        pass_end[static_cast<size_t>(i) * spp + (done - 1)] =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return true;
      };
      render_proxy_bdpt(sc, spp, seed + static_cast<unsigned long long>(i), pp, nullptr, cb);
    });
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"

#ifndef ORC_PCG

namespace {

constexpr int kBuckets = 4000;

int bucket_index(const StatsKey& k) { return ((k.u - 1) * 10 + k.c) * 100 + k.s; }

bool near_zero3(const Vec3& v) { return v.x == 0.0 && v.y == 0.0 && v.z == 0.0; }

uint64_t unit_stream(int pass, int walk) {
  return (static_cast<uint64_t>(pass) << 32) | static_cast<uint32_t>(walk);
}

// Restates pretrace_statistics (proj/src/subspace.cpp:190-218) with one stream per walk
// (deviation 1). Bucket maxima and counts do not depend on the visiting order, so the
// per-thread partial tables merge exactly.
SubspaceStats pretrace_rekeyed(const Scene& scene, int n_paths, uint64_t seed,
                               const SubspaceMapper& mapper, int threads) {
  if (n_paths < 1000)
    throw std::invalid_argument("pretrace_statistics: need at least 1000 paths");
  const int chunks = std::max(1, threads) * 4;
  std::vector<SubspaceStats> part(chunks);
  parallel_for(chunks, threads, [&](int c) {
    for (int i = c; i < n_paths; i += chunks) {
      Rng rng = Rng::keyed(seed, PXG_KIND_PRETRACE, 0, static_cast<uint64_t>(i));
      SubPath walk = trace_light_subpath(scene, 7, rng);
      const int n = static_cast<int>(walk.vertices.size());
      for (int end = 2; end <= n; ++end) {
        if (walk.vertices[end - 1].flag != VertexFlag::kSpecular) continue;
        SubPath prefix;
        prefix.kind = SubPathKind::kLight;
        prefix.vertices.assign(walk.vertices.begin(), walk.vertices.begin() + end);
        auto inc = dropout(prefix, mapper);
        if (!inc) continue;
        StatsKey key{inc->u, inc->c_label, inc->s_label};
        for (int probe = 0; probe < 2; ++probe) {
          SupportCandidate cand = support_sample(*inc, scene, rng);
          if (!cand.valid || cand.q <= 0.0) continue;
          double f = cand.escaped ? 0.0 : target_density(*inc, cand.g, scene);
          part[c].update_ratio(key, f / cand.q);
        }
      }
    }
  });
  SubspaceStats stats;
  for (auto& p : part) stats.merge(p);
  return stats;
}

struct PoolCand {
  uint64_t key;
  int walk;
  int end;
  IncompleteLightSubPath inc;
};

// Restates weighted_bdpt_value (proj/src/proxy.cpp:621-643): every standard strategy
// with the reciprocal-aware weight.
Vec3 weighted_bdpt(const Scene& scene, const SubPath& eye, const SubPath& light,
                   const SubspaceMapper& mapper, const SubspaceStats& stats) {
  const int max_depth = scene.settings.max_depth;
  Vec3 radiance(0.0);
  const int n_eye = static_cast<int>(eye.vertices.size());
  const int n_light = static_cast<int>(light.vertices.size());
  for (int t = 2; t <= n_eye; ++t) {
    Vec3 le = eye_hit_emission(eye, t, scene);
    if (!near_zero3(le)) {
      FullPath fp = make_full_path(light, 0, eye, t);
      radiance += le * reciprocal_mis_weight(fp, StrategyId{0, t, false}, scene, mapper, stats);
    }
    for (int s = 1; s <= n_light && s + t <= max_depth + 1; ++s) {
      FullPath fp = make_full_path(light, s, eye, t);
      Vec3 c = connection_contribution(fp, scene);
      if (near_zero3(c)) continue;
      radiance += c * reciprocal_mis_weight(fp, StrategyId{s, t, false}, scene, mapper, stats);
    }
  }
  return radiance;
}

struct PixelOut {
  Vec3 bdpt;
  Vec3 c;
  double u_gate = 0.0;
  double q_sel = 0.0;
  int t_label = -1;
  int chosen = -1;
  int key = -1;
  int flags = 0;  // bit0 tp>=2 (gate drawn), bit1 attempted (s_rep fits), bit2 z_norm > 0
};

}  // namespace

extern "C" {

// The restated render loop. Returns the mean image in rgb[n_px*3].
ORC_API int orc_render(void* h, int spp, unsigned long long seed, const OrcParams* op,
                       int threads, double* rgb, OrcTrace* tr) {
  try {
    const Scene& scene = static_cast<OrcScene*>(h)->scene;
    const ProxyParams params = to_params(op);
    if (spp <= 0) spp = scene.settings.spp;
    const int width = scene.camera.width;
    const int height = scene.camera.height;
    const int n_px = width * height;
    const int max_depth = scene.settings.max_depth;

    const SubspaceMapper mapper = SubspaceMapper::for_scene(scene);
    SubspaceStats stats;
    GammaMatrix gamma =
        GammaMatrix::uniform(mapper.t_count, mapper.s_count, params.freeze_iteration);
    std::vector<Rng> pixel_rng;
    pixel_rng.reserve(n_px);
    for (int i = 0; i < n_px; ++i) pixel_rng.emplace_back(seed, static_cast<uint64_t>(i));

    if (params.enabled) {
      stats = pretrace_rekeyed(scene, std::max(params.pretrace_paths, 1000), seed, mapper,
                               threads);
      if (tr && tr->pretrace_max) {
        for (const auto& [k, b] : stats.buckets) {
          tr->pretrace_max[bucket_index(k)] = b.max_ratio;
          tr->pretrace_cnt[bucket_index(k)] = b.ratio_count;
        }
      }
    }

    const int light_walks = params.light_walks > 0 ? params.light_walks : n_px;
    const int grid_w = (width + 9) / 10;
    const int grid_h = (height + 9) / 10;
    const int n_cells = grid_w * grid_h;
    std::vector<double> grid_proxy(n_cells, 0.0), grid_total(n_cells, 0.0);
    std::vector<Vec3> acc(n_px, Vec3(0.0));
    std::vector<PixelOut> px(n_px);
    std::vector<long long> diag(static_cast<size_t>(kBuckets) * 5, 0);
    long long diag_raw = 0, diag_kept = 0;

    for (int pass = 0; pass < spp; ++pass) {
      // ---- Stage 1 (proxy.cpp:684-736) ----
      std::vector<IncompleteLightSubPath> pool;
      std::vector<std::vector<int>> by_label(mapper.s_count);
      std::vector<int> pool_walk, pool_end;
      std::vector<double> pool_bound;
      double kappa = 1.0;
      if (params.enabled) {
        std::vector<std::vector<PoolCand>> per_walk(light_walks);
        parallel_for(light_walks, threads, [&](int w) {
          Rng rng = Rng::keyed(seed, PXG_KIND_POOL_WALK, 0, unit_stream(pass, w));
          SubPath walk = trace_light_subpath(scene, max_depth - 1, rng);
          const int n = static_cast<int>(walk.vertices.size());
          for (int end = 2; end <= n; ++end) {
            if (walk.vertices[end - 1].flag != VertexFlag::kSpecular) continue;
            SubPath prefix;
            prefix.kind = SubPathKind::kLight;
            prefix.vertices.assign(walk.vertices.begin(), walk.vertices.begin() + end);
            auto inc = dropout(prefix, mapper);
            if (!inc) continue;
            Rng kr = Rng::keyed(seed, PXG_KIND_RESERVOIR, static_cast<uint32_t>(end),
                                unit_stream(pass, w));
            uint64_t hi = kr.next_u32();
            uint64_t key = (hi << 32) | kr.next_u32();
            per_walk[w].push_back(PoolCand{key, w, end, std::move(*inc)});
          }
        });
        long long raw = 0;
        for (auto& v : per_walk) raw += static_cast<long long>(v.size());
        // Priority reservoir (deviation 2): the budget smallest keys, ties by (walk, end).
        std::vector<PoolCand*> all;
        all.reserve(static_cast<size_t>(raw));
        for (auto& v : per_walk)
          for (auto& c : v) all.push_back(&c);
        auto by_key = [](const PoolCand* a, const PoolCand* b) {
          if (a->key != b->key) return a->key < b->key;
          if (a->walk != b->walk) return a->walk < b->walk;
          return a->end < b->end;
        };
        if (static_cast<long long>(all.size()) > params.pool_budget) {
          std::nth_element(all.begin(), all.begin() + params.pool_budget, all.end(), by_key);
          all.resize(params.pool_budget);
        }
        std::sort(all.begin(), all.end(), [](const PoolCand* a, const PoolCand* b) {
          if (a->walk != b->walk) return a->walk < b->walk;
          return a->end < b->end;
        });
        kappa = raw > 0 ? std::min(1.0, static_cast<double>(params.pool_budget) /
                                            static_cast<double>(raw))
                        : 1.0;
        diag_raw += raw;
        if (tr && tr->pool_raw && pass < tr->n_passes_cap) tr->pool_raw[pass] = raw;

        // estimate_inverse_p (proxy.cpp:380-428), restated: probes and the bound are
        // sequential in pool order (B of entry k sees the probes of entries <= k);
        // reciprocal runs are independent given B and run in parallel.
        const int n_ent = static_cast<int>(all.size());
        std::vector<double> bound(n_ent, 0.0);
        for (int k = 0; k < n_ent; ++k) {
          IncompleteLightSubPath& inc = all[k]->inc;
          const StatsKey key = inc.key();
          if (params.recip_repeats >= 1) {
            for (int i = 0; i < 4; ++i) {
              // one stream per probe (PROBE, end | i << 8) so the four probes run in parallel
              Rng pr = Rng::keyed(seed, PXG_KIND_PROBE,
                                  static_cast<uint32_t>(all[k]->end) | (static_cast<uint32_t>(i) << 8),
                                  unit_stream(pass, all[k]->walk));
              SupportCandidate cand = support_sample(inc, scene, pr);
              if (!cand.valid || !(cand.q > 0.0)) continue;
              double f = cand.escaped ? 0.0 : target_density(inc, cand.g, scene);
              stats.update_ratio(key, f / cand.q);
            }
          }
          bound[k] = stats.b_bound(key);
        }
        const int R = params.recip_repeats;
        std::vector<recip::ReciprocalRun> runs(static_cast<size_t>(n_ent) * std::max(R, 1));
        parallel_for(n_ent * std::max(R, 0), threads, [&](int j) {
          const int k = j / R, r = j % R;
          if (!(bound[k] > 0.0)) return;
          const IncompleteLightSubPath& inc = all[k]->inc;
          recip::IntegrandOracle<SupportCandidate> f_oracle = [&](const SupportCandidate& c) {
            return c.escaped ? 0.0 : target_density(inc, c.g, scene);
          };
          // Deviation (3): node k of the tree (DFS pre-order == k-th draw_g call) draws its
          // support sample from stream (RECIP_NODE, k) and its split decision from
          // (RECIP_SPLIT, k): the sampler re-keys the walk's Rng, which recip::Walk hands
          // to stochastic_split right after draw_g (recip.hpp:69-97).
          const uint64_t stream = pxg_recip_stream(static_cast<uint32_t>(pass), static_cast<uint32_t>(all[k]->walk),
                                                   static_cast<uint32_t>(all[k]->end), static_cast<uint32_t>(r));
          uint32_t node = 0;
          recip::SupportSampler<SupportCandidate> sampler{
              [&](Rng& rr) {
                Rng nr = Rng::keyed(seed, PXG_KIND_RECIP_NODE, node, stream);
                SupportCandidate c = support_sample(inc, scene, nr);
                rr = Rng::keyed(seed, PXG_KIND_RECIP_SPLIT, node, stream);
                ++node;
                return c;
              },
              [](const SupportCandidate& c) { return c.q; }};
          recip::ReciprocalConfig cfg;
          cfg.bound = bound[k];
          cfg.recursion_cap = params.recursion_cap;
          Rng rr = Rng::keyed(seed, PXG_KIND_RECIP_SPLIT, 0, stream);
          runs[static_cast<size_t>(k) * R + r] = recip::estimate_reciprocal(f_oracle, sampler, cfg, rr);
        });
        for (int k = 0; k < n_ent; ++k) {
          IncompleteLightSubPath& inc = all[k]->inc;
          const StatsKey key = inc.key();
          const int bi = bucket_index(key);
          bool valid = false;
          if (R >= 1 && bound[k] > 0.0) {
            double sum = 0.0, sum_sq = 0.0;
            int truncated = 0;
            for (int r = 0; r < R; ++r) {
              const auto& run = runs[static_cast<size_t>(k) * R + r];
              sum += run.estimate;
              sum_sq += run.estimate * run.estimate;
              if (run.truncated) ++truncated;
            }
            double mean = sum / R;
            double m2 = sum_sq / R;
            diag[bi * 5 + 3] += truncated;
            if (std::isfinite(mean) && mean > 0.0) {
              valid = true;
              inc.inverse_p = mean;
              inc.inverse_p_m2 = m2;
              stats.update_estimate(key, mean);
            }
          }
          diag[bi * 5 + 2] += R;
          if (!valid) {
            ++diag[bi * 5 + 4];
            continue;
          }
          pool.push_back(inc);
          pool_walk.push_back(all[k]->walk);
          pool_end.push_back(all[k]->end);
          pool_bound.push_back(bound[k]);
        }
        diag_kept += static_cast<long long>(pool.size());
        for (int i = 0; i < static_cast<int>(pool.size()); ++i)
          by_label[pool[i].s_label].push_back(i);
        if (tr && tr->pool_n && pass < tr->n_passes_cap) {
          const int m = std::min(static_cast<int>(pool.size()), tr->pool_cap);
          tr->pool_n[pass] = static_cast<int>(pool.size());
          for (int i = 0; i < m; ++i) {
            const size_t o = static_cast<size_t>(pass) * tr->pool_cap + i;
            tr->pool_walk[o] = pool_walk[i];
            tr->pool_end[o] = pool_end[i];
            tr->pool_key[o] = bucket_index(pool[i].key());
            tr->pool_inv_p[o] = pool[i].inverse_p;
            tr->pool_inv_p_m2[o] = pool[i].inverse_p_m2;
            tr->pool_bound[o] = pool_bound[i];
          }
        }
      }

      // ---- Stage 2, phase A: independent per pixel (proxy.cpp:739-793) ----
      const bool record_prims = tr && tr->trace_pass == pass && tr->eye_prims;
      parallel_for(height, threads, [&](int y) {
        for (int x = 0; x < width; ++x) {
          const int idx = y * width + x;
          PixelOut& o = px[idx];
          o = PixelOut{};
          Rng& rng = pixel_rng[idx];
          SubPath eye = trace_eye_subpath(scene, x, y, max_depth + 1, rng);
          SubPath light = trace_light_subpath(scene, max_depth - 1, rng);
          if (record_prims) {
            for (int k = 0; k <= max_depth; ++k)
              tr->eye_prims[static_cast<size_t>(idx) * (max_depth + 1) + k] =
                  k < static_cast<int>(eye.vertices.size()) ? eye.vertices[k].primitive : -2;
            for (int k = 0; k < max_depth - 1; ++k)
              tr->light_prims[static_cast<size_t>(idx) * (max_depth - 1) + k] =
                  k < static_cast<int>(light.vertices.size()) ? light.vertices[k].primitive : -2;
          }
          o.bdpt = weighted_bdpt(scene, eye, light, mapper, stats);
          if (!(params.enabled && !pool.empty())) continue;
          int tp = 0;
          const int n_eye = static_cast<int>(eye.vertices.size());
          for (int i = 1; i < n_eye; ++i) {
            if (eye.vertices[i].flag == VertexFlag::kDiffuse) {
              tp = i + 1;
              break;
            }
            if (eye.vertices[i].flag != VertexFlag::kSpecular) break;
          }
          if (tp < 2) continue;
          o.flags |= 1;
          // Speculative: every draw after the gate draw happens in the same order
          // whether or not the gate passes; phase B discards failed gates.
          Rng prox_rng(seed, (uint64_t(2) << 32) + static_cast<uint64_t>(pass) * n_px + idx);
          o.u_gate = prox_rng.next_double();
          const PathVertex& z = eye.vertices[tp - 1];
          const int t_label = mapper.classify_eye(z.p, -z.wi);
          double z_norm = 0.0;
          for (int sl = 0; sl < mapper.s_count; ++sl)
            if (!by_label[sl].empty()) z_norm += gamma.pmf(t_label, sl);
          if (!(z_norm > 0.0)) continue;
          o.flags |= 4;
          double uu = prox_rng.next_double() * z_norm;
          int chosen = -1;
          double cdf = 0.0;
          for (int sl = 0; sl < mapper.s_count; ++sl) {
            if (by_label[sl].empty()) continue;
            chosen = sl;
            cdf += gamma.pmf(t_label, sl);
            if (uu < cdf) break;
          }
          const double row_p = gamma.pmf(t_label, chosen) / z_norm;
          const auto& bucket = by_label[chosen];
          const IncompleteLightSubPath& inc =
              pool[bucket[prox_rng.next_below(static_cast<uint32_t>(bucket.size()))]];
          const int s_rep = static_cast<int>(inc.prefix.size()) + inc.u + 1;
          o.t_label = t_label;
          o.chosen = chosen;
          o.key = bucket_index(inc.key());
          o.q_sel = row_p / static_cast<double>(bucket.size());
          if (s_rep + tp <= max_depth + 1) {
            o.flags |= 2;
            SubPath eye_prefix;
            eye_prefix.kind = SubPathKind::kEye;
            eye_prefix.vertices.assign(eye.vertices.begin(), eye.vertices.begin() + tp);
            o.c = proxy_connect(eye_prefix, inc, scene, mapper, stats, prox_rng);
          }
        }
      });

      // ---- Stage 2, phase B: per 10x10 cell in scan order (proxy.cpp:761-817) ----
      std::vector<Vec3> val(n_px);
      std::vector<double> gamma_val(n_px, 0.0);
      std::vector<char> contributed(n_px, 0);
      std::vector<std::vector<long long>> cell_diag(n_cells);
      parallel_for(n_cells, threads, [&](int cell) {
        const int cx = cell % grid_w, cy = cell / grid_w;
        for (int y = cy * 10; y < std::min(height, cy * 10 + 10); ++y) {
          for (int x = cx * 10; x < std::min(width, cx * 10 + 10); ++x) {
            const int idx = y * width + x;
            const PixelOut& o = px[idx];
            Vec3 v = o.bdpt;
            int fl = o.flags & 1;
            if (o.flags & 1) {
              double gate = params.gate_high;
              if (pass > 0) {
                double share = grid_total[cell] > 0.0 ? grid_proxy[cell] / grid_total[cell] : 0.0;
                gate = share > params.gate_threshold ? params.gate_high : params.gate_low;
              }
              if (gate > 0.0 && o.u_gate < gate && (o.flags & 4)) {
                fl |= 4;
                if (o.flags & 2) {
                  fl |= 2;
                  if (cell_diag[cell].empty()) cell_diag[cell].assign(kBuckets * 2, 0);
                  ++cell_diag[cell][o.key * 2 + 0];
                  if (!near_zero3(o.c)) {
                    fl |= 8;
                    ++cell_diag[cell][o.key * 2 + 1];
                    Vec3 contrib = o.c / (static_cast<double>(light_walks) * kappa * gate * o.q_sel);
                    v += contrib;
                    gamma_val[idx] = luminance(o.c) / o.q_sel;
                    contributed[idx] = 1;
                    grid_proxy[cell] += luminance(contrib);
                  }
                }
              }
            }
            acc[idx] += v;
            val[idx] = v;
            grid_total[cell] += luminance(v);
            if (tr && pass < tr->n_passes_cap) {
              const size_t o3 = (static_cast<size_t>(pass) * n_px + idx) * 3;
              if (tr->pass_val) { tr->pass_val[o3] = v.x; tr->pass_val[o3 + 1] = v.y; tr->pass_val[o3 + 2] = v.z; }
              if (tr->pass_bdpt) { tr->pass_bdpt[o3] = o.bdpt.x; tr->pass_bdpt[o3 + 1] = o.bdpt.y; tr->pass_bdpt[o3 + 2] = o.bdpt.z; }
              if (tr->pass_c) { tr->pass_c[o3] = o.c.x; tr->pass_c[o3 + 1] = o.c.y; tr->pass_c[o3 + 2] = o.c.z; }
              if (tr->pass_flags) tr->pass_flags[static_cast<size_t>(pass) * n_px + idx] = fl;
            }
          }
        }
      });
      for (auto& cd : cell_diag) {
        if (cd.empty()) continue;
        for (int b = 0; b < kBuckets; ++b) {
          diag[b * 5 + 0] += cd[b * 2 + 0];
          diag[b * 5 + 1] += cd[b * 2 + 1];
        }
      }
      // ---- phase C: gamma accumulation in pixel scan order (proxy.cpp:807-808) ----
      for (int idx = 0; idx < n_px; ++idx)
        if (contributed[idx])
          gamma.record_contribution(px[idx].t_label, px[idx].chosen, gamma_val[idx]);
      gamma.end_iteration();
    }

    for (int i = 0; i < n_px; ++i) {
      Vec3 m = acc[i] / static_cast<double>(spp > 0 ? spp : 1);
      rgb[3 * i] = m.x;
      rgb[3 * i + 1] = m.y;
      rgb[3 * i + 2] = m.z;
    }
    if (tr) {
      if (tr->stats_out) {
        for (const auto& [k, b] : stats.buckets) {
          const int bi = bucket_index(k);
          tr->stats_out[bi * 3 + 0] = b.max_ratio;
          tr->stats_out[bi * 3 + 1] = b.sum_est;
          tr->stats_out[bi * 3 + 2] = b.sum_est_sq;
          tr->stats_cnt[bi * 2 + 0] = b.ratio_count;
          tr->stats_cnt[bi * 2 + 1] = b.est_count;
        }
      }
      if (tr->gamma_rows) std::memcpy(tr->gamma_rows, gamma.rows.data(), gamma.rows.size() * sizeof(double));
      if (tr->diag) std::memcpy(tr->diag, diag.data(), diag.size() * sizeof(long long));
      if (tr->diag_pool) { tr->diag_pool[0] = diag_raw; tr->diag_pool[1] = diag_kept; }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Reciprocal estimator on the two-point fixture (proj/tests/test_recip.cpp:16-23):
// f = {1, 3}, q = 1/2, B = bound. Run i uses stream (seed, RECIP kind, sub 0, i).
ORC_API int orc_recip_twopoint(int n, double bound, long long cap, unsigned long long seed,
                               double* est, long long* cost, int* truncated) {
  try {
    recip::IntegrandOracle<int> f = [](const int& x) { return x == 0 ? 1.0 : 3.0; };
    recip::ReciprocalConfig cfg;
    cfg.bound = bound;
    cfg.recursion_cap = cap;
    for (int i = 0; i < n; ++i) {
      // node-keyed streams as in the render loop (deviation 3), stream = run index
      uint32_t node = 0;
      recip::SupportSampler<int> q{[&](Rng& rr) {
                                     Rng nr = Rng::keyed(seed, PXG_KIND_RECIP_NODE, node, static_cast<uint64_t>(i));
                                     int x = nr.next_double() < 0.5 ? 0 : 1;
                                     rr = Rng::keyed(seed, PXG_KIND_RECIP_SPLIT, node, static_cast<uint64_t>(i));
                                     ++node;
                                     return x;
                                   },
                                   [](const int&) { return 0.5; }};
      Rng rng = Rng::keyed(seed, PXG_KIND_RECIP_SPLIT, 0, static_cast<uint64_t>(i));
      auto run = recip::estimate_reciprocal(f, q, cfg, rng);
      est[i] = run.estimate;
      cost[i] = run.cost;
      truncated[i] = run.truncated ? 1 : 0;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- Replay parity (SURVEY §8c mode ii): the device's vertices rescored by the reference.
// The vertex record mirrors pxg_vertex / the device PathVertex (include/pxg.h).
struct OrcVertex {
  double p[3], n[3], wi[3], thr[3];
  double pdf_fwd;
  int material, primitive, emitter, flag;
  double reserved;
};

// One pixel's proxy connection inputs (the pool entry the device picked).
struct OrcProxyIn {
  int tp;          // eye cut (eye vertices [0, tp))
  int u, n_prefix, has_cdir;
  double cdir[3];
  double prefix_pdf, inverse_p;
};

// Rescored values: prefix / retrace densities (proxy_pdf_components), subspace labels,
// the reciprocal-aware MIS weight and the proxy_connect value of the device's path.
struct OrcProxyOut {
  double prefix_pdf, retrace_density, weight;
  double c[3];
  int s_label, c_label, pad0, pad1;
};

static PathVertex to_vertex(const Scene& scene, const OrcVertex& v) {
  PathVertex o;
  o.p = Vec3(v.p[0], v.p[1], v.p[2]);
  o.n = Vec3(v.n[0], v.n[1], v.n[2]);
  o.wi = Vec3(v.wi[0], v.wi[1], v.wi[2]);
  o.throughput = Vec3(v.thr[0], v.thr[1], v.thr[2]);
  o.pdf_fwd = v.pdf_fwd;
  o.material = v.material >= 0 ? &scene.materials[static_cast<size_t>(v.material)] : nullptr;
  o.primitive = v.primitive;
  o.emitter = v.emitter;
  o.flag = static_cast<VertexFlag>(v.flag);
  return o;
}

static SubspaceStats stats_from_dense(const double* s3) {
  SubspaceStats st;
  for (int k = 0; k < kBuckets; ++k) {
    const long long cnt = static_cast<long long>(s3[3 * k + 2]);
    if (cnt <= 0) continue;
    BucketStats b;
    b.sum_est = s3[3 * k];
    b.sum_est_sq = s3[3 * k + 1];
    b.est_count = cnt;
    st.buckets[StatsKey{k / 1000 + 1, (k / 100) % 10, k % 100}] = b;
  }
  return st;
}

// weighted_bdpt_value (proj/src/proxy.cpp:621-643) of the device's sub-paths:
// eye[i*eye_stride + k], k < n_eye[i]; light likewise; stats3 = the pass's snapshot
// (pxg_dump_paths). out[i*3] = the standard-strategy sum.
ORC_API int orc_replay_bdpt(void* h, int n, const OrcVertex* eye, const int* n_eye, int eye_stride,
                            const OrcVertex* light, const int* n_light, int light_stride, const double* stats3,
                            int threads, double* out) {
  try {
    const Scene& scene = static_cast<OrcScene*>(h)->scene;
    const SubspaceMapper mapper = SubspaceMapper::for_scene(scene);
    const SubspaceStats stats = stats_from_dense(stats3);
    parallel_for(n, threads, [&](int i) {
      SubPath e, l;
      e.kind = SubPathKind::kEye;
      l.kind = SubPathKind::kLight;
      for (int k = 0; k < n_eye[i]; ++k) e.vertices.push_back(to_vertex(scene, eye[static_cast<size_t>(i) * eye_stride + k]));
      for (int k = 0; k < n_light[i]; ++k)
        l.vertices.push_back(to_vertex(scene, light[static_cast<size_t>(i) * light_stride + k]));
      Vec3 v = weighted_bdpt(scene, e, l, mapper, stats);
      out[3 * i] = v.x;
      out[3 * i + 1] = v.y;
      out[3 * i + 2] = v.z;
    });
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

static OrcVertex from_vertex(const Scene& scene, const PathVertex& v) {
  OrcVertex o;
  std::memset(&o, 0, sizeof(o));
  const Vec3* src[4] = {&v.p, &v.n, &v.wi, &v.throughput};
  double* dst[4] = {o.p, o.n, o.wi, o.thr};
  for (int k = 0; k < 4; ++k) {
    dst[k][0] = src[k]->x;
    dst[k][1] = src[k]->y;
    dst[k][2] = src[k]->z;
  }
  o.pdf_fwd = v.pdf_fwd;
  o.material = v.material ? static_cast<int>(v.material - scene.materials.data()) : -1;
  o.primitive = v.primitive;
  o.emitter = v.emitter;
  o.flag = static_cast<int>(v.flag);
  return o;
}

// The first pass's sub-paths of pixels [0, n) as the render loop traces them
// (proj/src/proxy.cpp:742-744: eye then light sub-path on the pixel stream Rng(seed, idx)),
// in the replay vertex layout: pins the replay evaluator against the restated loop on the CPU.
ORC_API int orc_trace_subpaths(void* h, unsigned long long seed, int n, OrcVertex* eye, int* n_eye, int eye_stride,
                               OrcVertex* light, int* n_light, int light_stride, int threads) {
  try {
    const Scene& scene = static_cast<OrcScene*>(h)->scene;
    const int width = scene.camera.width;
    const int max_depth = scene.settings.max_depth;
    parallel_for(n, threads, [&](int idx) {
      Rng rng(seed, static_cast<uint64_t>(idx));
      SubPath e = trace_eye_subpath(scene, idx % width, idx / width, max_depth + 1, rng);
      SubPath l = trace_light_subpath(scene, max_depth - 1, rng);
      n_eye[idx] = static_cast<int>(e.vertices.size());
      n_light[idx] = static_cast<int>(l.vertices.size());
      for (int k = 0; k < n_eye[idx] && k < eye_stride; ++k)
        eye[static_cast<size_t>(idx) * eye_stride + k] = from_vertex(scene, e.vertices[k]);
      for (int k = 0; k < n_light[idx] && k < light_stride; ++k)
        light[static_cast<size_t>(idx) * light_stride + k] = from_vertex(scene, l.vertices[k]);
    });
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The proxy connection of the device's path: px[i*kMaxLight + ..] holds the picked entry's
// prefix [0, n_prefix), the retraced block g (reference order) [n_prefix, n_prefix+u) and the
// specular endpoint at n_prefix+u. Recomputes proxy_pdf_components (proj/src/proxy.cpp:321-378),
// the labels dropout assigns (proxy.cpp:87-89) and the value proxy_connect forms after its
// retrace (proxy.cpp:562-602, with the recomputed retrace density), all with the reference's
// functions.
ORC_API int orc_replay_proxy(void* h, int n, const OrcVertex* eye, int eye_stride, const OrcVertex* px, int px_stride,
                             const OrcProxyIn* in, const double* stats3, int threads, OrcProxyOut* out) {
  try {
    const Scene& scene = static_cast<OrcScene*>(h)->scene;
    const SubspaceMapper mapper = SubspaceMapper::for_scene(scene);
    const SubspaceStats stats = stats_from_dense(stats3);
    parallel_for(n, threads, [&](int i) {
      const OrcProxyIn& a = in[i];
      OrcProxyOut& o = out[i];
      std::memset(&o, 0, sizeof(o));
      const OrcVertex* pv = px + static_cast<size_t>(i) * px_stride;
      IncompleteLightSubPath inc;
      for (int k = 0; k < a.n_prefix; ++k) inc.prefix.push_back(to_vertex(scene, pv[k]));
      inc.specular_end = to_vertex(scene, pv[a.n_prefix + a.u]);
      if (a.has_cdir) inc.control_dir = Vec3(a.cdir[0], a.cdir[1], a.cdir[2]);
      inc.u = a.u;
      inc.prefix_pdf = a.prefix_pdf;
      inc.inverse_p = a.inverse_p;
      inc.s_label = mapper.classify_specular(inc.specular_end);
      inc.c_label = mapper.classify_control(inc.control(), inc.control_dir);
      o.s_label = inc.s_label;
      o.c_label = inc.c_label;
      std::vector<PathVertex> g;
      for (int j = 0; j < a.u; ++j) g.push_back(to_vertex(scene, pv[a.n_prefix + j]));
      SubPath e;
      e.kind = SubPathKind::kEye;
      for (int k = 0; k < a.tp; ++k) e.vertices.push_back(to_vertex(scene, eye[static_cast<size_t>(i) * eye_stride + k]));
      const PathVertex& z = e.vertices[a.tp - 1];
      ProxyPdfComponents comps = proxy_pdf_components(inc, g, z, scene);
      o.prefix_pdf = comps.prefix_pdf;
      o.retrace_density = comps.retrace_density;
      if (!(comps.retrace_density > 0.0)) return;
      // proxy_connect after retrace_proxy (proxy.cpp:562-602)
      SubPath rep = repair(inc, g);
      const auto& lv = rep.vertices;
      const int s = static_cast<int>(lv.size());
      const int t = a.tp;
      Vec3 d01 = lv[1].p - lv[0].p;
      double l01 = length(d01);
      if (l01 <= 0.0 || lv[0].emitter < 0) return;
      Vec3 value = scene.emitted(lv[0].emitter, lv[0].n, d01 / l01);
      if (near_zero3(value)) return;
      for (int k = 0; k + 1 < s; ++k) {
        double gt = geometry_term(lv[k], lv[k + 1], scene);
        if (gt <= 0.0) return;
        value *= gt;
      }
      double gj = geometry_term(lv[s - 1], z, scene);
      if (gj <= 0.0) return;
      value *= gj;
      for (int k = 1; k < s; ++k) {
        Vec3 wi = normalize(lv[k - 1].p - lv[k].p);
        Vec3 to = k + 1 < s ? lv[k + 1].p : z.p;
        Vec3 wo = normalize(to - lv[k].p);
        Vec3 fk = eval_bsdf(*lv[k].material, lv[k].n, wi, wo);
        if (near_zero3(fk)) return;
        value = value * fk;
      }
      Vec3 fz = eval_bsdf(*z.material, z.n, z.wi, normalize(lv[s - 1].p - z.p));
      if (near_zero3(fz)) return;
      value = value * fz * z.throughput;
      FullPath fp;
      fp.light = lv;
      fp.eye = e.vertices;
      fp.s = s;
      fp.t = t;
      const double w = reciprocal_mis_weight(fp, StrategyId{s, t, true}, scene, mapper, stats);
      o.weight = w;
      if (!(w > 0.0)) return;
      Vec3 c = value * (inc.inverse_p * w / (inc.prefix_pdf * comps.retrace_density));
      o.c[0] = c.x;
      o.c[1] = c.y;
      o.c[2] = c.z;
    });
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The reference's dropout, support_pdf, target_density and support_sample on caller-supplied
// vertices (proj/src/proxy.cpp:59-269): the checker of pxg_proxy_probe. Draw j uses the stream
// Rng::keyed(seed, 3 /* PROBE */, 0, j), like the device probe.
ORC_API int orc_proxy_probe(void* h, int n_walk, const OrcVertex* walk, int n_cand, const OrcVertex* cand,
                            int n_draws, unsigned long long seed, int* info, double* prefix_pdf, double* q,
                            double* f, OrcVertex* draw_cand, double* draw_q, int* draw_escaped) {
  try {
    const Scene& scene = static_cast<OrcScene*>(h)->scene;
    const SubspaceMapper mapper = SubspaceMapper::for_scene(scene);
    SubPath sp;
    sp.kind = SubPathKind::kLight;
    for (int k = 0; k < n_walk; ++k) sp.vertices.push_back(to_vertex(scene, walk[k]));
    for (int k = 0; k < 8; ++k) info[k] = 0;
    *prefix_pdf = 0.0;
    auto inc = dropout(sp, mapper);
    if (!inc) return 0;
    info[0] = 1;
    info[1] = inc->u;
    info[2] = static_cast<int>(inc->prefix.size());
    info[3] = inc->control_dir.has_value() ? 1 : 0;
    info[4] = inc->c_label;
    info[5] = inc->s_label;
    info[6] = ((inc->u - 1) * 10 + inc->c_label) * 100 + inc->s_label;
    info[7] = static_cast<int>(sp.vertices[inc->prefix.size()].flag);
    *prefix_pdf = inc->prefix_pdf;
    const int u = inc->u;
    for (int i = 0; i < n_cand; ++i) {
      std::vector<PathVertex> g;
      for (int k = 0; k < u; ++k) g.push_back(to_vertex(scene, cand[static_cast<size_t>(i) * u + k]));
      q[i] = support_pdf(*inc, g, scene);
      f[i] = target_density(*inc, g, scene);
    }
    for (int j = 0; j < n_draws; ++j) {
      Rng rng = Rng::keyed(seed, 3, 0, static_cast<uint64_t>(j));
      SupportCandidate c = support_sample(*inc, scene, rng);
      draw_q[j] = c.q;
      draw_escaped[j] = c.escaped ? 1 : 0;
      for (int k = 0; k < u; ++k) {
        OrcVertex z;
        std::memset(&z, 0, sizeof(z));
        draw_cand[static_cast<size_t>(j) * u + k] =
            (!c.escaped && k < static_cast<int>(c.g.size())) ? from_vertex(scene, c.g[k]) : z;
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Philox stream check: first n draws of Rng::keyed(seed, kind, sub, stream).
ORC_API void orc_rng_draws(unsigned long long seed, unsigned kind, unsigned sub,
                           unsigned long long stream, int n, unsigned* out) {
  Rng r = Rng::keyed(seed, kind, sub, stream);
  for (int i = 0; i < n; ++i) out[i] = r.next_u32();
}

}  // extern "C"

#endif  // ORC_PCG
