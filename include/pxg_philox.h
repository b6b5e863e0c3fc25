/* pxg_philox.h — the counter-based RNG shared by the sm_100a kernels and the CPU oracle.
 *
 * Replaces the reference's PCG32 `proxima::Rng` (proj/include/proxima/rng.hpp:12-44)
 * behind the same draw interface: next_u32, next_double = u32 * 2^-32,
 * next_below(n) = (u32 * n) >> 32, bernoulli(p) = next_double() < p.
 *
 * A stream is identified by (seed, kind, sub, stream). Draw i of a stream is word 0 of
 * Philox4x32-10 with key = (seed_lo, seed_hi) and counter = (i, kind << 24 | sub,
 * stream_lo, stream_hi). Because draw i is a pure function of (stream id, i), a GPU
 * thread and a CPU loop that consume the same stream in the same order see identical
 * numbers, and any stream can be resumed from a stored counter.
 *
 * kind 0 reproduces the reference's Rng(seed, stream) constructor (pixel streams
 * `idx`, proxy streams `(2<<32)+pass*n_px+idx`, proj/src/proxy.cpp:664-666,759-760).
 * Streams the reference draws sequentially (pool walks, reservoir, probes, reciprocal
 * runs, pretrace; proj/src/proxy.cpp:691-721, proj/src/proxy.cpp:669) are re-keyed
 * per unit with a nonzero kind so they can run in parallel.
 */
#ifndef PXG_PHILOX_H
#define PXG_PHILOX_H

#include <stdint.h>

#if defined(__CUDACC__)
#define PXG_HD __host__ __device__ __forceinline__
#else
#define PXG_HD static inline
#endif

enum {
  PXG_KIND_REF = 0,        /* reference-compatible Rng(seed, stream) */
  PXG_KIND_POOL_WALK = 1,  /* stream = pass<<32 | walk                       */
  PXG_KIND_RESERVOIR = 2,  /* stream = pass<<32 | walk, sub = prefix end      */
  PXG_KIND_PROBE = 3,      /* stream = pass<<32 | walk, sub = end | probe << 8 */
  PXG_KIND_RECIP = 4,      /* stream = pass<<32 | walk, sub = end | run << 8  */
  PXG_KIND_PRETRACE = 5,   /* stream = walk                                   */
  PXG_KIND_RECIP_NODE = 6, /* sub = tree node (DFS pre-order), stream = pxg_recip_stream() */
  PXG_KIND_RECIP_SPLIT = 7 /* sub = tree node, stream = pxg_recip_stream()     */
};

/* Stream of reciprocal run `run` of pool entry (pass, walk, end). Node k of the run's
 * Russian-roulette-and-split tree draws its support sample from (RECIP_NODE, k) and its
 * split decision from (RECIP_SPLIT, k), so every node can be evaluated independently of
 * the tree shape. Limits: pass < 2^24, walk < 2^27, end < 32, run < 256, k < 2^24. */
PXG_HD uint64_t pxg_recip_stream(uint32_t pass, uint32_t walk, uint32_t end, uint32_t run) {
  return ((uint64_t)pass << 40) | ((uint64_t)walk << 13) | ((uint64_t)(end & 31u) << 8) | (uint64_t)(run & 255u);
}

PXG_HD uint32_t pxg_mulhilo32(uint32_t a, uint32_t b, uint32_t* hi) {
#if defined(__CUDA_ARCH__)
  *hi = __umulhi(a, b);
  return a * b;
#else
  uint64_t p = (uint64_t)a * (uint64_t)b;
  *hi = (uint32_t)(p >> 32);
  return (uint32_t)p;
#endif
}

/* Philox4x32-10, first output word only. Under nvcc the function is kept out of line: one
 * copy per kernel instead of one per draw site (the fp64 kernels draw at 5-10 sites and are
 * 5,000+ instructions long; ncu shows instruction-fetch stalls second only to memory in
 * k_shade): C4 +0.75%. -DPXG_PHILOX_NOINLINE=0 inlines it again. */
#ifndef PXG_PHILOX_NOINLINE
#define PXG_PHILOX_NOINLINE 1
#endif
#if defined(__CUDACC__) && PXG_PHILOX_NOINLINE
__host__ __device__ __noinline__ static uint32_t pxg_philox_word0(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                                  uint32_t k0, uint32_t k1) {
#else
PXG_HD uint32_t pxg_philox_word0(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                 uint32_t k0, uint32_t k1) {
#endif
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, hi1;
    uint32_t lo0 = pxg_mulhilo32(M0, c0, &hi0);
    uint32_t lo1 = pxg_mulhilo32(M1, c2, &hi1);
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += W0; k1 += W1;
  }
  return c0;
}

typedef struct PxgRng {
  uint32_t k0, k1;   /* seed */
  uint32_t tag;      /* kind << 24 | sub */
  uint32_t s0, s1;   /* stream */
  uint32_t i;        /* draw counter */
} PxgRng;

PXG_HD PxgRng pxg_rng_make(uint64_t seed, uint32_t kind, uint32_t sub, uint64_t stream) {
  PxgRng r;
  r.k0 = (uint32_t)seed;
  r.k1 = (uint32_t)(seed >> 32);
  r.tag = (kind << 24) | (sub & 0xFFFFFFu);
  r.s0 = (uint32_t)stream;
  r.s1 = (uint32_t)(stream >> 32);
  r.i = 0u;
  return r;
}

PXG_HD uint32_t pxg_next_u32(PxgRng* r) {
  uint32_t v = pxg_philox_word0(r->i, r->tag, r->s0, r->s1, r->k0, r->k1);
  r->i += 1u;
  return v;
}

PXG_HD double pxg_next_double(PxgRng* r) { return (double)pxg_next_u32(r) * 0x1p-32; }

PXG_HD uint32_t pxg_next_below(PxgRng* r, uint32_t n) {
  return (uint32_t)(((uint64_t)pxg_next_u32(r) * (uint64_t)n) >> 32);
}

PXG_HD int pxg_bernoulli(PxgRng* r, double p) { return pxg_next_double(r) < p; }

#endif /* PXG_PHILOX_H */
