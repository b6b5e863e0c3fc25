// ORACLE / TEST INFRASTRUCTURE ONLY — never part of the product path.
//
// Shadow of the reference header proj/include/proxima/rng.hpp:12-44. It is placed
// first on the include path when oracle/Makefile compiles the unmodified reference
// sources, so every reference translation unit draws from the Philox streams of
// include/pxg_philox.h instead of PCG32. Same members, same draw semantics
// (next_double = u32 * 2^-32, next_below = multiply-shift, bernoulli = u < p).
#pragma once

#include <cstdint>

#include "pxg_philox.h"

namespace proxima {

struct Rng {
  PxgRng r{};
  // The reference exposes `state`; one reference unit test compares it before and
  // after a call that must not draw. Here it mirrors the draw counter.
  uint64_t state = 0;

  Rng() { reseed(0, 0); }
  Rng(uint64_t seed, uint64_t stream = 0) { reseed(seed, stream); }

  // Re-keyed stream (kind != 0) used by the oracle driver where the reference draws
  // one sequential stream for independent units of work.
  static Rng keyed(uint64_t seed, uint32_t kind, uint32_t sub, uint64_t stream) {
    Rng g;
    g.r = pxg_rng_make(seed, kind, sub, stream);
    g.state = 0;
    return g;
  }

  void reseed(uint64_t seed, uint64_t stream) {
    r = pxg_rng_make(seed, PXG_KIND_REF, 0, stream);
    state = 0;
  }

  uint32_t next_u32() {
    uint32_t v = pxg_next_u32(&r);
    state = r.i;
    return v;
  }
  double next_double() { return next_u32() * 0x1p-32; }
  uint32_t next_below(uint32_t n) {
    return static_cast<uint32_t>((static_cast<uint64_t>(next_u32()) * n) >> 32);
  }
  bool bernoulli(double p) { return next_double() < p; }
};

}  // namespace proxima
