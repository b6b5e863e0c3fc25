// ORACLE / TEST INFRASTRUCTURE ONLY.
// The reference's film output and metrics (proj/src/image.cpp, proj/src/metrics.cpp) as a
// standalone program, so tests/test_film.py can pin paper_2503_23412_b200/film.py against
// them (the reference's iostream code cannot run inside the Python process: the oracle
// library carries its own static libstdc++).
// Usage: film_ref W H est.f64 ref.f64 out.pfm out.png  -> prints mape smape mse eps
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "proxima/image.hpp"

static proxima::Image load(const char* path, int w, int h) {
  std::vector<double> v(static_cast<size_t>(w) * h * 3);
  std::ifstream in(path, std::ios::binary);
  in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(double)));
  proxima::Image img(w, h);
  for (size_t i = 0; i < img.pixels.size(); ++i) img.pixels[i] = proxima::Vec3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
  return img;
}

int main(int argc, char** argv) {
  if (argc < 7) return 2;
  const int w = std::atoi(argv[1]), h = std::atoi(argv[2]);
  const proxima::Image est = load(argv[3], w, h), ref = load(argv[4], w, h);
  proxima::write_pfm(est, argv[5]);
  proxima::write_png(est, argv[6]);
  const proxima::MetricReport r = proxima::compare_images(est, ref);
  std::printf("%.17g %.17g %.17g %.17g\n", r.mape, r.smape, r.mse, r.epsilon);
  return 0;
}
