// ORACLE / TEST INFRASTRUCTURE ONLY.
// Exercises include/pxg_proxima.hpp exactly as a reference maintainer would: the
// reference's own Scene (loaded by the unmodified reference loader) goes into
// render_proxy_bdpt_gpu, and the result is compared with the unmodified reference
// render_bdpt on the same Philox streams (proxy off, proj/tests/test_proxy.cpp:1053-1079);
// render_pt_gpu against the unmodified reference render_pt.
// Usage: dropin_test scene.json spp seed            parity checks (exit 0 = pass)
//        dropin_test scene.json spp seed --time     end-to-end timing of the pipelined pass_done
//                                                   loop on a finalised scene (one JSON line)
#include <chrono>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>

#include "pxg_proxima.hpp"
#include "proxima/transport.hpp"

int main(int argc, char** argv) {
  if (argc < 4) return 2;
  std::ifstream in(argv[1]);
  std::stringstream buf;
  buf << in.rdbuf();
  proxima::Scene scene = proxima::load_scene_from_string(buf.str());
  const int spp = std::atoi(argv[2]);
  const uint64_t seed = std::strtoull(argv[3], nullptr, 10);
  if (argc > 4 && std::strcmp(argv[4], "--time") == 0) {
    // the reference's load_scene finalises once; render calls then start from the finalised scene
    proxima::PxgScene gs(scene);
    proxima::ProxyParams def;
    double mean_sum = 0.0;
    auto cb = [&](int, const proxima::Image& img) {
      mean_sum += img.pixels[0].x;
      return true;
    };
    proxima::render_proxy_bdpt_gpu(gs, 2, seed, def, nullptr, cb);  // warm-up (allocator, pinned staging)
    const auto t0 = std::chrono::steady_clock::now();
    proxima::Image img = proxima::render_proxy_bdpt_gpu(gs, spp, seed, def, nullptr, cb);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const double px = static_cast<double>(scene.camera.width) * scene.camera.height;
    std::printf("{\"e2e_msamples_s\": %.4f, \"spp\": %d, \"wall_s\": %.4f, \"width\": %d, \"height\": %d, "
                "\"path\": \"render_proxy_bdpt_gpu(PxgScene, spp, seed, {}, nullptr, pass_done) from C++\", "
                "\"finite\": %d}\n",
                px * spp / s / 1e6, spp, s, scene.camera.width, scene.camera.height,
                std::isfinite(img.pixels[0].x) && std::isfinite(mean_sum) ? 1 : 0);
    return 0;
  }
  proxima::ProxyParams off;
  off.enabled = false;
  proxima::Image gpu = proxima::render_proxy_bdpt_gpu(scene, spp, seed, off);
  proxima::Image ref = proxima::render_bdpt(scene, spp, seed);
  double worst = 0.0;
  for (size_t i = 0; i < ref.pixels.size(); ++i) {
    const proxima::Vec3 a = gpu.pixels[i], b = ref.pixels[i];
    const double d[3] = {a.x - b.x, a.y - b.y, a.z - b.z};
    const double m[3] = {std::fabs(b.x), std::fabs(b.y), std::fabs(b.z)};
    for (int k = 0; k < 3; ++k) worst = std::fmax(worst, std::fabs(d[k]) / std::fmax(m[k], 1e-12));
  }
  // proxy on, with an early stop after 2 passes through the callback
  proxima::ProxyParams on;
  on.pretrace_paths = 2000;
  on.light_walks = 2000;
  int seen = 0;
  proxima::ProxyDiagnostics diag;
  proxima::Image p = proxima::render_proxy_bdpt_gpu(scene, spp, seed, on, &diag,
                                                    [&](int done, const proxima::Image&) {
                                                      seen = done;
                                                      return done < 2;
                                                    });
  // the pipelined pass_done loop (no diagnostics): stopping after 2 passes returns the 2-pass
  // image bitwise (proj/tests/test_proxy.cpp:1096-1105)
  int seen2 = 0;
  proxima::Image stop2 = proxima::render_proxy_bdpt_gpu(scene, spp, seed, on, nullptr,
                                                        [&](int done, const proxima::Image&) {
                                                          seen2 = done;
                                                          return done < 2;
                                                        });
  proxima::Image two = proxima::render_proxy_bdpt_gpu(scene, 2, seed, on);
  proxima::PxgScene gscene(scene);
  proxima::Image two_fin = proxima::render_proxy_bdpt_gpu(gscene, 2, seed, on);
  bool stop_bitwise = seen2 == 2;
  for (size_t i = 0; i < two.pixels.size(); ++i) {
    const proxima::Vec3 a = stop2.pixels[i], b = two.pixels[i], c = two_fin.pixels[i];
    stop_bitwise = stop_bitwise && a.x == b.x && a.y == b.y && a.z == b.z && c.x == b.x && c.y == b.y && c.z == b.z;
  }
  bool finite = true;
  for (const auto& v : p.pixels) finite = finite && std::isfinite(v.x) && std::isfinite(v.y) && std::isfinite(v.z);
  // render_pt_gpu against the unmodified reference render_pt
  proxima::Image gpt = proxima::render_pt_gpu(scene, spp, seed);
  proxima::Image rpt = proxima::render_pt(scene, spp, seed);
  double worst_pt = 0.0;
  for (size_t i = 0; i < rpt.pixels.size(); ++i) {
    const proxima::Vec3 a = gpt.pixels[i], b = rpt.pixels[i];
    const double d[3] = {a.x - b.x, a.y - b.y, a.z - b.z};
    const double m[3] = {std::fabs(b.x), std::fabs(b.y), std::fabs(b.z)};
    for (int k = 0; k < 3; ++k) worst_pt = std::fmax(worst_pt, std::fabs(d[k]) / std::fmax(m[k], 1e-12));
  }
  std::printf("bdpt_max_rel %.3e pt_max_rel %.3e passes_seen %d pool_raw %lld finite %d pipelined_stop_bitwise %d\n",
              worst, worst_pt, seen, diag.pool_raw, finite ? 1 : 0, stop_bitwise ? 1 : 0);
  return (worst < 1e-6 && worst_pt < 1e-6 && seen == 2 && finite && stop_bitwise) ? 0 : 1;
}
