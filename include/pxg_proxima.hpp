// pxg_proxima.hpp — drop-in C++ entry point for the reference code base.
//
// A proxima maintainer adds this header to the reference build and links libpxg.so; the
// function below has the exact signature of proxima::render_proxy_bdpt
// (proj/include/proxima/proxy.hpp:197-200) and the same semantics: spp <= 0 uses
// scene.settings.spp, one pass = one sample per pixel, pass_done receives the running
// mean after every pass and returning false stops the render, diagnostics is filled in
// place, and failures throw std::runtime_error (validation failures: the reference's
// messages) — the C ABI's error codes never leak.
//
// Only this header depends on the reference's types; libpxg itself is plain C ABI.
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "proxima/image.hpp"
#include "proxima/proxy.hpp"
#include "proxima/scene.hpp"
#include "pxg.h"

namespace proxima {

inline void pxg_throw(int rc, const pxg_ctx* ctx) {
  if (rc != PXG_OK) throw std::runtime_error(pxg_last_error(ctx));
}

// Flattens a finalized proxima::Scene into the C ABI descriptor. The vectors own the
// arrays the descriptor points to and must outlive pxg_create.
struct PxgSceneArrays {
  std::vector<int> shape, material, emitter_prim;
  std::vector<double> a, b, c, radius, materials, emitter_radiance;
  pxg_scene_desc desc{};

  explicit PxgSceneArrays(const Scene& s) {
    const size_t n = s.primitives.size();
    shape.resize(n);
    material.resize(n);
    a.resize(3 * n);
    b.resize(3 * n);
    c.resize(3 * n);
    radius.resize(n);
    for (size_t i = 0; i < n; ++i) {
      const Primitive& p = s.primitives[i];
      shape[i] = p.shape == Primitive::Shape::kSphere ? 0 : (p.shape == Primitive::Shape::kTriangle ? 1 : 2);
      material[i] = p.material;
      const Vec3* v[3] = {&p.a, &p.b, &p.c};
      std::vector<double>* dst[3] = {&a, &b, &c};
      for (int k = 0; k < 3; ++k) {
        (*dst[k])[3 * i] = v[k]->x;
        (*dst[k])[3 * i + 1] = v[k]->y;
        (*dst[k])[3 * i + 2] = v[k]->z;
      }
      radius[i] = p.radius;
    }
    for (const Material& m : s.materials) {
      const double row[7] = {m.base_color.x, m.base_color.y, m.base_color.z, m.metallic,
                             m.roughness, m.transmission, m.ior};
      materials.insert(materials.end(), row, row + 7);
    }
    for (const Emitter& e : s.emitters) {
      emitter_prim.push_back(e.primitive);
      emitter_radiance.insert(emitter_radiance.end(), {e.radiance.x, e.radiance.y, e.radiance.z});
    }
    desc.n_prims = static_cast<int>(n);
    desc.shape = shape.data();
    desc.material = material.data();
    desc.a = a.data();
    desc.b = b.data();
    desc.c = c.data();
    desc.radius = radius.data();
    desc.n_materials = static_cast<int>(s.materials.size());
    desc.materials = materials.data();
    desc.n_emitters = static_cast<int>(s.emitters.size());
    desc.emitter_prim = emitter_prim.data();
    desc.emitter_radiance = emitter_radiance.data();
    const Vec3* cam[3] = {&s.camera.position, &s.camera.look_at, &s.camera.up};
    double* out[3] = {desc.cam_position, desc.cam_look_at, desc.cam_up};
    for (int k = 0; k < 3; ++k) {
      out[k][0] = cam[k]->x;
      out[k][1] = cam[k]->y;
      out[k][2] = cam[k]->z;
    }
    desc.fov_y = s.camera.fov_y;
    desc.width = s.camera.width;
    desc.height = s.camera.height;
    desc.max_depth = s.settings.max_depth;
  }
};

inline pxg_params pxg_params_from(const ProxyParams& p) {
  pxg_params q;
  q.enabled = p.enabled ? 1 : 0;
  q.pool_budget = p.pool_budget;
  q.recip_repeats = p.recip_repeats;
  q.freeze_iteration = p.freeze_iteration;
  q.recursion_cap = p.recursion_cap;
  q.pretrace_paths = p.pretrace_paths;
  q.light_walks = p.light_walks;
  q.gate_high = p.gate_high;
  q.gate_low = p.gate_low;
  q.gate_threshold = p.gate_threshold;
  return q;
}

// Passes in flight in the pipelined pass_done loop (< PXG_SNAPSHOT_SLOTS).
constexpr int kPxgPipelineAhead = 3;

inline void pxg_fill_diagnostics(pxg_ctx* ctx, ProxyDiagnostics* diagnostics) {
  std::vector<long long> rows(4000 * 5);
  std::vector<int> touched(4000);
  long long pool[2];
  pxg_throw(pxg_read_diag(ctx, rows.data(), touched.data(), pool), ctx);
  for (int k = 0; k < 4000; ++k) {
    if (!touched[k]) continue;
    ProxyDiagRow& r = diagnostics->rows[StatsKey{k / 1000 + 1, (k / 100) % 10, k % 100}];
    r.retrace_attempts += rows[5 * k];
    r.retrace_accepts += rows[5 * k + 1];
    r.recip_runs += rows[5 * k + 2];
    r.recip_truncated += rows[5 * k + 3];
    r.estimates_failed += rows[5 * k + 4];
  }
  diagnostics->pool_raw += pool[0];
  diagnostics->pool_kept += pool[1];
}

// The render loop of proxima::render_proxy_bdpt (proj/src/proxy.cpp:683-833) over a context.
//  * no callback: all passes are enqueued at once (Stage 1 runs a batch ahead of Stage 2);
//  * a callback: passes k+1 .. k+kPxgPipelineAhead-1 are already enqueued while pass_done sees
//    the device snapshot of the mean after pass k, so the GPU never drains while the host reads
//    back and runs the callback; an early stop returns that snapshot (bitwise the k-pass image,
//    proj/tests/test_proxy.cpp:1096-1105) and the passes rendered beyond it are discarded;
//  * a callback and diagnostics: one pass at a time, so the counters never include a pass
//    beyond an early stop.
inline Image pxg_render_loop(pxg_ctx* ctx, int w, int h, int spp, ProxyDiagnostics* diagnostics,
                             const std::function<bool(int, const Image&)>& pass_done) {
  pxg_throw(pxg_set_pass_limit(ctx, spp), ctx);
  std::vector<double> rgb(static_cast<size_t>(w) * h * 3);
  auto to_image = [&]() {
    Image img(w, h);
    for (size_t i = 0; i < img.pixels.size(); ++i) img.pixels[i] = Vec3(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
    return img;
  };
  int done = 0;
  if (!pass_done) {
    pxg_throw(pxg_render_passes(ctx, spp), ctx);
    pxg_throw(pxg_read_mean(ctx, rgb.data(), &done), ctx);
  } else if (!diagnostics) {
    const int ahead = spp < kPxgPipelineAhead ? spp : kPxgPipelineAhead;
    for (int j = 0; j < ahead; ++j) {
      pxg_throw(pxg_render_passes_async(ctx, 1), ctx);
      pxg_throw(pxg_snapshot_mean(ctx, j % PXG_SNAPSHOT_SLOTS), ctx);
    }
    for (int k = 1; k <= spp; ++k) {
      const int j = k + ahead - 1;  // next pass to enqueue (0-based)
      if (j < spp) {
        pxg_throw(pxg_render_passes_async(ctx, 1), ctx);
        pxg_throw(pxg_snapshot_mean(ctx, j % PXG_SNAPSHOT_SLOTS), ctx);
      }
      pxg_throw(pxg_read_snapshot(ctx, (k - 1) % PXG_SNAPSHOT_SLOTS, rgb.data(), &done), ctx);
      if (!pass_done(done, to_image())) break;
    }
  } else {
    for (int pass = 0; pass < spp; ++pass) {
      pxg_throw(pxg_render_pass(ctx), ctx);
      pxg_throw(pxg_read_mean(ctx, rgb.data(), &done), ctx);
      if (!pass_done(done, to_image())) break;
    }
    pxg_throw(pxg_read_mean(ctx, rgb.data(), &done), ctx);
  }
  if (diagnostics) pxg_fill_diagnostics(ctx, diagnostics);
  return to_image();
}

// A finalised scene on the GPU side (validation, emitter tables and the BVH built once), the
// counterpart of the reference's Scene after Scene::finalize (proj/src/scene.cpp:234-252):
// repeated render calls on one scene upload it without rebuilding.
class PxgScene {
 public:
  explicit PxgScene(const Scene& s) : w_(s.camera.width), h_(s.camera.height), spp_(s.settings.spp) {
    PxgSceneArrays arrays(s);
    pxg_throw(pxg_scene_create(&arrays.desc, &scene_), nullptr);
  }
  ~PxgScene() { pxg_scene_destroy(scene_); }
  PxgScene(const PxgScene&) = delete;
  PxgScene& operator=(const PxgScene&) = delete;
  const pxg_scene* get() const { return scene_; }
  int width() const { return w_; }
  int height() const { return h_; }
  int spp() const { return spp_; }

 private:
  pxg_scene* scene_ = nullptr;
  int w_, h_, spp_;
};

// render_proxy_bdpt on an already finalised GPU scene.
inline Image render_proxy_bdpt_gpu(const PxgScene& scene, int spp, uint64_t seed, const ProxyParams& params = {},
                                   ProxyDiagnostics* diagnostics = nullptr,
                                   const std::function<bool(int, const Image&)>& pass_done = {},
                                   int device = 0) {
  if (spp <= 0) spp = scene.spp();
  const pxg_params p = pxg_params_from(params);
  pxg_ctx* ctx = nullptr;
  pxg_throw(pxg_create_from_scene(scene.get(), &p, seed, device, nullptr, &ctx), nullptr);
  struct Guard {
    pxg_ctx* c;
    ~Guard() { pxg_destroy(c); }
  } guard{ctx};
  return pxg_render_loop(ctx, scene.width(), scene.height(), spp, diagnostics, pass_done);
}

// Same signature and behaviour as proxima::render_proxy_bdpt, computed on the GPU.
inline Image render_proxy_bdpt_gpu(const Scene& scene, int spp, uint64_t seed, const ProxyParams& params = {},
                                   ProxyDiagnostics* diagnostics = nullptr,
                                   const std::function<bool(int, const Image&)>& pass_done = {},
                                   int device = 0) {
  if (spp <= 0) spp = scene.settings.spp;
  PxgSceneArrays arrays(scene);
  const pxg_params p = pxg_params_from(params);
  pxg_ctx* ctx = nullptr;
  pxg_throw(pxg_create(&arrays.desc, &p, seed, device, nullptr, &ctx), nullptr);
  struct Guard {
    pxg_ctx* c;
    ~Guard() { pxg_destroy(c); }
  } guard{ctx};
  return pxg_render_loop(ctx, scene.camera.width, scene.camera.height, spp, diagnostics, pass_done);
}

// Same signature and behaviour as proxima::render_pt (proj/include/proxima/transport.hpp:88),
// computed on the GPU (per pixel identical to the reference on the same RNG streams).
inline Image render_pt_gpu(const Scene& scene, int spp, uint64_t seed, int device = 0) {
  if (spp <= 0) spp = scene.settings.spp;
  PxgSceneArrays arrays(scene);
  pxg_params p;
  pxg_default_params(&p);
  p.enabled = 0;
  pxg_ctx* ctx = nullptr;
  pxg_throw(pxg_create(&arrays.desc, &p, seed, device, nullptr, &ctx), nullptr);
  struct Guard {
    pxg_ctx* c;
    ~Guard() { pxg_destroy(c); }
  } guard{ctx};
  const int w = scene.camera.width, h = scene.camera.height;
  std::vector<double> rgb(static_cast<size_t>(w) * h * 3);
  pxg_throw(pxg_render_pt(ctx, spp, seed, 1, rgb.data()), ctx);
  Image img(w, h);
  for (size_t i = 0; i < img.pixels.size(); ++i) img.pixels[i] = Vec3(rgb[3 * i], rgb[3 * i + 1], rgb[3 * i + 2]);
  return img;
}

}  // namespace proxima
