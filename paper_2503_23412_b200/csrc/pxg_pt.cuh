// pxg_pt.cuh — the reference's unidirectional path tracer on the device.
//
// render_pt / pt_radiance (proj/src/transport.cpp:272-330, 376-381): camera ray, BSDF
// sampling with next-event estimation and the two-strategy balance weights, same draw
// order (jitter v then u, light point, BSDF lobe/direction), same fp64 operation order.
// It is the converged reference for the relMSE checks of the proxy-BDPT renders (the
// reference's own acceptance test uses PT as its oracle, proj/tests/acceptance.cpp:396-402).
//
// Layout: one thread per (pixel, chunk). Chunk c is an independent render_pt(spp, seed_c)
// with seed_c = seed ^ (c * 0x9E3779B97F4A7C15) (chunk 0 is exactly render_pt(spp, seed):
// the pixel stream Rng(seed, y*W + x), samples drawn back to back on it). Each thread writes
// its pixel's mean; k_pt_reduce averages the chunks in chunk order (deterministic).
#pragma once

#include "pxg_path.cuh"

namespace pxg {

__device__ __forceinline__ uint64_t pt_chunk_seed(uint64_t seed, int chunk) {
  return seed ^ (static_cast<uint64_t>(chunk) * 0x9E3779B97F4A7C15ull);
}

// pt_radiance (transport.cpp:272-330)
__device__ __forceinline__ V3 pt_radiance(const SceneView& S, int max_depth, int px, int py, Rng& rng) {
  const double jv = rng.next_double();  // generate_ray's arguments are drawn right to left
  const double ju = rng.next_double();
  V3 o = S.cam_pos;
  V3 dir = camera_dir(S, px, py, ju, jv);
  V3 radiance = v3(0.0);
  V3 beta = v3(1.0);
  bool from_delta = true;
  double prev_pdf_w = 0.0;
  V3 prev_p = v3(0.0);
  for (int depth = 1; depth <= max_depth; ++depth) {
    Hit hit;
    if (!intersect(S, o, dir, hit)) break;
    const Material& mat = S.materials[hit.material];
    const V3 wi = -dir;
    const V3 le = emitted(S, hit.emitter, hit.n, wi);
    if (!near_zero(le)) {
      if (from_delta) {
        radiance = radiance + beta * le;
      } else {
        const double p_hit = to_area_density(prev_pdf_w, prev_p, hit.p, hit.n);
        const double p_nee = 1.0 / S.total_emitter_area;
        radiance = radiance + beta * le * (p_hit / (p_hit + p_nee));
      }
    }
    if (depth == max_depth) break;
    const bool specular = mat.specular != 0;
    if (!specular) {
      const LightPoint lp = sample_light_point(S, rng);
      const V3 d = lp.p - hit.p;
      const double dist2 = dot(d, d);
      if (dist2 > 0.0) {
        const V3 ldir = d / sqrt(dist2);
        const V3 le_nee = emitted(S, S.prim_emitter[lp.prim], lp.n, -ldir);
        if (!near_zero(le_nee)) {
          const V3 f = eval_bsdf(mat, hit.n, wi, ldir);
          if (!near_zero(f) && visible(S, hit.p, lp.p)) {
            const double g = fabs(dot(hit.n, ldir)) * fabs(dot(lp.n, ldir)) / dist2;
            const double p_bsdf = to_area_density(pdf_bsdf(mat, hit.n, wi, ldir), hit.p, lp.p, lp.n);
            const double w = lp.pdf_area / (lp.pdf_area + p_bsdf);
            radiance = radiance + beta * f * le_nee * (g * w / lp.pdf_area);
          }
        }
      }
    }
    const BsdfSample bs = sample_bsdf(mat, hit.n, wi, rng);
    if (!bs.valid || bs.pdf <= 0.0) break;
    beta = beta * bs.value * (fabs(dot(bs.wo, hit.n)) / bs.pdf);
    if (near_zero(beta)) break;
    from_delta = specular;
    prev_pdf_w = bs.pdf;
    prev_p = hit.p;
    o = hit.p;
    dir = bs.wo;
  }
  return radiance;
}

// render_image's per-pixel loop (transport.cpp:355-367) for one (pixel, chunk).
__global__ void k_render_pt(SceneView S, int max_depth, int row0, int n, int chunks, int spp, uint64_t seed,
                            double* __restrict__ out) {
  const long long gid = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= static_cast<long long>(n) * chunks) return;
  const int i = static_cast<int>(gid % n);
  const int chunk = static_cast<int>(gid / n);
  const int idx = row0 * S.width + i;
  const int x = idx % S.width, y = idx / S.width;
  Rng rng;
  rng.r = pxg_rng_make(pt_chunk_seed(seed, chunk), PXG_KIND_REF, 0, static_cast<uint64_t>(idx));
  V3 acc = v3(0.0);
  for (int s = 0; s < spp; ++s) acc = acc + pt_radiance(S, max_depth, x, y, rng);
  const V3 m = acc / static_cast<double>(spp);
  double* o = out + 3 * static_cast<size_t>(gid);
  o[0] = m.x;
  o[1] = m.y;
  o[2] = m.z;
}

__global__ void k_pt_reduce(int n, int chunks, const double* __restrict__ in, double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= 3 * n) return;
  double s = 0.0;
  for (int c = 0; c < chunks; ++c) s += in[static_cast<size_t>(c) * 3 * n + k];
  out[k] = s / chunks;
}

}  // namespace pxg
