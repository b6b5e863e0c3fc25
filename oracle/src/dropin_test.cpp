// ORACLE / TEST INFRASTRUCTURE ONLY.
// Exercises include/pxg_proxima.hpp exactly as a reference maintainer would: the
// reference's own Scene (loaded by the unmodified reference loader) goes into
// render_proxy_bdpt_gpu, and the result is compared with the unmodified reference
// render_bdpt on the same Philox streams (proxy off, proj/tests/test_proxy.cpp:1053-1079);
// render_pt_gpu against the unmodified reference render_pt.
// Usage: dropin_test scene.json spp seed
#include <cmath>
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
  std::printf("bdpt_max_rel %.3e pt_max_rel %.3e passes_seen %d pool_raw %lld finite %d\n", worst, worst_pt, seen,
              diag.pool_raw, finite ? 1 : 0);
  return (worst < 1e-6 && worst_pt < 1e-6 && seen == 2 && finite) ? 0 : 1;
}
