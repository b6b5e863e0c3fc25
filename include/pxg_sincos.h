/* pxg_sincos.h — double sin / cos that return glibc's results bit for bit.
 *
 * The reference maps a uniform draw to an angle and calls glibc (std::cos(phi),
 * std::sin(phi) with phi = 2*pi*u, u = k * 2^-32: proj/src/bsdf.cpp:63-65 (GGX visible
 * normals), proj/src/bsdf.cpp:226-227 (cosine hemisphere), proj/src/scene.cpp:199-201
 * (sphere lights)). CUDA's sin/cos are within 2 ulp of the true value and differ from glibc
 * on a large fraction of arguments, which let a few sub-path trajectories of the GPU
 * diverge from the reference's (a 1-ulp direction change that flips a grazing triangle
 * test).
 *
 * Two parts:
 * 1. pxg_sincos_dd evaluates sin and cos to ~2^-66 relative as unrounded double-doubles:
 *    Cody-Waite reduction by pi/2 held in four doubles (three 33-bit pieces, q * C_k exact
 *    for q < 2^20), a second reduction by a = j/64 with sin(a), cos(a) from a 53-entry
 *    double-double table, short Taylor polynomials on |s| <= 1/128 (tails in double), and
 *    the angle-sum formulas in double-double. hi is the correctly rounded value except on
 *    the few arguments within ~2^-13 ulp of a rounding midpoint.
 * 2. glibc 2.39 is not correctly rounded either: on ~0.14% of the 2^32 sampler angles it
 *    returns the other neighbour of the exact value, always within 0.016 ulp of a midpoint.
 *    A table built from the host's libm by csrc/pxg_sincos_gen.cpp lists every k where
 *    glibc differs from hi (per range of 2^26 k and per function, the largest midpoint
 *    distance of a listed entry: thr; per bucket of 2^12 k, a sorted run of 16-bit entries:
 *    low 12 bits of k, bit 12 sin differs, bit 13 cos differs). A draw farther than thr
 *    from a midpoint is never listed, so only ~3% of draws search their bucket.
 * pxg_sincos_2pi_glibc combines them; the generator checks every one of the 2^32 angles, so
 * the result equals glibc's on all of them by construction (tests/test_sincos.py repeats the
 * exhaustive check on the GPU box's libm and compares the device with it).
 *
 * The same code runs on the host (C/C++, compile with -ffp-contract=off) and the device
 * (nvcc --fmad=false). Valid for |x| < 2^20 * pi/2. Constants:
 * tools/gen/gen_sincos_consts.py (mpmath, 300 bits).
 */
#ifndef PXG_SINCOS_H
#define PXG_SINCOS_H

#include <math.h>
#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define PXG_SC_HD __host__ __device__ __forceinline__
#else
#define PXG_SC_HD static inline
#endif

/* pi/2 = C1 + C2 + C3 + C4 */
#define PXG_SC_C1 0x1.921fb54400000p+0
#define PXG_SC_C2 0x1.0b4611a600000p-34
#define PXG_SC_C3 0x1.3198a2e000000p-69
#define PXG_SC_C4 0x1.b839a252049c1p-104
#define PXG_SC_TWO_OVER_PI 0x1.45f306dc9c883p-1
/* (-1)^k / n! */
#define PXG_SC_F3 -0x1.5555555555555p-3
#define PXG_SC_F5 0x1.1111111111111p-7
#define PXG_SC_F7 -0x1.a01a01a01a01ap-13
#define PXG_SC_F9 0x1.71de3a556c734p-19
#define PXG_SC_F2 -0x1.0000000000000p-1
#define PXG_SC_F4 0x1.5555555555555p-5
#define PXG_SC_F6 -0x1.6c16c16c16c17p-10
#define PXG_SC_F8 0x1.a01a01a01a01ap-16
/* {sin_hi, sin_lo, cos_hi, cos_lo} of j/64, j = 0..52 */
#define PXG_SC_TAB_INIT { \
  {0x0.0p+0, 0x0.0p+0, 0x1.0000000000000p+0, 0x0.0p+0}, \
  {0x1.fffaaaaeeeed5p-7, -0x1.2ab639a9f0776p-63, 0x1.fff000155549fp-1, 0x1.28a28a03a5ef3p-55}, \
  {0x1.ffeaaaeeee86fp-6, -0x1.cd406fb224ae2p-60, 0x1.ffc00155527d3p-1, -0x1.3b54492d89b5bp-55}, \
  {0x1.7fdc01032fba9p-5, -0x1.599bdf46e997ap-59, 0x1.ff7006bfdf99fp-1, -0x1.8b3b560648d5fp-56}, \
  {0x1.ffaaaeeed4edbp-5, -0x1.2d16d32684b69p-59, 0x1.ff0015549f4d3p-1, 0x1.328387b99426fp-55}, \
  {0x1.3facb12d1755bp-4, -0x1.921915299468bp-58, 0x1.fe7034129ef6fp-1, -0x1.cbf4337c96f97p-57}, \
  {0x1.7f701032550e4p-4, 0x1.afc2d1800501ap-60, 0x1.fdc06bf7e6b9bp-1, 0x1.31902b535f8dbp-55}, \
  {0x1.bf1b78568391dp-4, 0x1.e91841dea4cc8p-58, 0x1.fcf0c800e99b1p-1, 0x1.ea3d786d186acp-57}, \
  {0x1.feaaeee86ee36p-4, -0x1.afcb2bcc6f03bp-59, 0x1.fc015527d5bd3p-1, 0x1.b68f35094efb8p-55}, \
  {0x1.1f0d3d7afceafp-3, -0x1.6ef95099769a5p-57, 0x1.faf22263c4bd3p-1, -0x1.52ace133a2769p-58}, \
  {0x1.3eb312c5d66cbp-3, 0x1.47d666b66cb91p-57, 0x1.f9c340a7cc428p-1, 0x1.c5b6b063b7462p-55}, \
  {0x1.5e44fcfa126f3p-3, -0x1.6f443063f89b6p-57, 0x1.f874c2e1eecf6p-1, -0x1.c6514e1332b16p-55}, \
  {0x1.7dc102fbaf2b5p-3, 0x1.5ab50e23c97c3p-59, 0x1.f706bdf9ece1cp-1, -0x1.698c80c36dcb4p-55}, \
  {0x1.9d252d0cec312p-3, 0x1.9c43d80b1137dp-58, 0x1.f57948cff6797p-1, 0x1.e3a0d3e03b1d4p-57}, \
  {0x1.bc6f84edc6199p-3, 0x1.9c1a56a7b0cabp-57, 0x1.f3cc7c3b3d16ep-1, -0x1.21a3ad28a3494p-57}, \
  {0x1.db9e15fb5a5d0p-3, -0x1.32e20d6cc6fc2p-57, 0x1.f20073086649fp-1, 0x1.b940416c1984bp-56}, \
  {0x1.faaeed4f31577p-3, -0x1.15d88508e32b8p-57, 0x1.f01549f7deea1p-1, 0x1.d3c1e99e5cafdp-55}, \
  {0x1.0cd00cef36436p-2, -0x1.9fb0a0c93e2b4p-56, 0x1.ee0b1fbc0f11cp-1, -0x1.bfd2380bbc3b1p-59}, \
  {0x1.1c37d64c6b876p-2, 0x1.46076fe0dcff4p-56, 0x1.ebe214f76efa8p-1, -0x1.02f9f12ba543ep-55}, \
  {0x1.2b8ddc43eb49fp-2, 0x1.1553899f2d807p-57, 0x1.e99a4c3a7cd83p-1, -0x1.2264b1bc53ce8p-55}, \
  {0x1.3ad129769d3d8p-2, 0x1.03d550487839ap-63, 0x1.e733ea0193d40p-1, -0x1.6428b3546ce13p-55}, \
  {0x1.4a00c9b0f3d20p-2, 0x1.823ba6bb08eadp-56, 0x1.e4af14b2a449cp-1, -0x1.68ca02e8a6833p-55}, \
  {0x1.591bc9fa2f597p-2, 0x1.7c74bac3fe0cbp-57, 0x1.e20bf49acd6c1p-1, -0x1.660aec7ef636bp-58}, \
  {0x1.682138a38d7f7p-2, -0x1.d889202444aadp-56, 0x1.df4ab3ebd875ep-1, -0x1.e2d8a7e6736c4p-55}, \
  {0x1.7710255764214p-2, -0x1.6ead7314bb6cep-57, 0x1.dc6b7eb995912p-1, 0x1.4b364776dcd35p-58}, \
  {0x1.85e7a12826949p-2, 0x1.8a40e9b5face0p-56, 0x1.d96e82f71a9dcp-1, 0x1.ff61bd5d2039dp-55}, \
  {0x1.94a6be9f546c5p-2, -0x1.69ce13e683f58p-56, 0x1.d653f073e4040p-1, -0x1.76236434bec37p-55}, \
  {0x1.a34c91cc50ccap-2, -0x1.a310e3b50cecdp-58, 0x1.d31bf8d8d7c06p-1, 0x1.e60dd3089cbddp-56}, \
  {0x1.b1d8305321617p-2, -0x1.ae242cb99f519p-56, 0x1.cfc6cfa52ad9fp-1, 0x1.8b5b5508f2a0dp-55}, \
  {0x1.c048b17b140a3p-2, 0x1.19fe6757e9fa7p-57, 0x1.cc54aa2b2972ep-1, 0x1.4ee162ba83a98p-57}, \
  {0x1.ce9d2e3d4a51fp-2, -0x1.2fc8a12dae298p-57, 0x1.c8c5bf8ce1a84p-1, 0x1.ab3d1a1590123p-56}, \
  {0x1.dcd4c15329c9ap-2, 0x1.0d4c6e171fd9ap-56, 0x1.c51a48b8b175ep-1, -0x1.1bbb43b9aa880p-57}, \
  {0x1.eaee8744b05f0p-2, -0x1.789b43c9b027dp-58, 0x1.c1528065b7d50p-1, -0x1.892111312e828p-55}, \
  {0x1.f8e99e76abc97p-2, 0x1.9d950af2d00a3p-58, 0x1.bd6ea310294f5p-1, 0x1.31bbcc88c109dp-56}, \
  {0x1.0362939c69955p-1, -0x1.2d8cd78397b01p-55, 0x1.b96eeef58840ep-1, 0x1.45a3cc78fade0p-58}, \
  {0x1.0a4021e9e1001p-1, -0x1.6f643a13914f6p-55, 0x1.b553a410c104ep-1, 0x1.8ff7947027a15p-58}, \
  {0x1.110d0c4b69c3bp-1, 0x1.d918998809981p-55, 0x1.b11d04162a4c6p-1, 0x1.1dd561efbc0c2p-56}, \
  {0x1.17c8e5f2eedb0p-1, 0x1.35e57102e2488p-57, 0x1.accb526f69de5p-1, 0x1.8fb6a8dd6b6ccp-55}, \
  {0x1.1e7343236574cp-1, 0x1.22a3fa4f41d5ap-56, 0x1.a85ed4373e02dp-1, 0x1.9be06385ec792p-57}, \
  {0x1.250bb93788bbbp-1, 0x1.ea3d02457bccep-56, 0x1.a3d7d0352bdcfp-1, -0x1.68dbaeca19669p-55}, \
  {0x1.2b91dea88421ep-1, -0x1.fa371db216ab0p-55, 0x1.9f368ed912f85p-1, -0x1.1d200c5791606p-55}, \
  {0x1.32054b148bc4fp-1, 0x1.f6b42095a135bp-55, 0x1.9a7b5a36a6514p-1, 0x1.722cfcc9fa7a9p-55}, \
  {0x1.386597456282bp-1, -0x1.10fada93b07a8p-56, 0x1.95a67e00cb1fdp-1, -0x1.0befda21f862dp-55}, \
  {0x1.3eb25d36cd53ap-1, -0x1.be570e1570fc0p-58, 0x1.90b84784ddaf7p-1, -0x1.0feb10ab93b87p-56}, \
  {0x1.44eb381cf386bp-1, -0x1.3ed6c1e6a5505p-55, 0x1.8bb105a5dc900p-1, 0x1.863e03e9474c1p-55}, \
  {0x1.4b0fc46aab761p-1, 0x1.0da05738cc59cp-61, 0x1.869108d77a6c6p-1, 0x1.338ffe2bfe9ddp-56}, \
  {0x1.511f9fd7b351cp-1, -0x1.5c0e861c48831p-55, 0x1.8158a31916d5dp-1, -0x1.de8b90b8228dep-57}, \
  {0x1.571a6966d59b3p-1, 0x1.c843b4d0fb197p-58, 0x1.7c0827f09e54fp-1, -0x1.c73d6d72aee68p-57}, \
  {0x1.5cffc16bf8f0dp-1, 0x1.96cb370eb578ap-55, 0x1.769fec655211fp-1, -0x1.827d5cf8c68c5p-57}, \
  {0x1.62cf49921ac79p-1, -0x1.edd9855b6241ap-55, 0x1.712046fa77678p-1, 0x1.425b0a5029c81p-55}, \
  {0x1.6888a4e134b2fp-1, -0x1.6b7d37644d5e6p-55, 0x1.6b898fa9efb5dp-1, 0x1.15ac786ccf4b2p-56}, \
  {0x1.6e2b77c40bde1p-1, -0x1.0e729857fad53p-56, 0x1.65dc1fdeb8cbap-1, -0x1.97c1b47337c77p-58}, \
  {0x1.73b7680dea578p-1, -0x1.2248306dc12a2p-56, 0x1.6018526f563dfp-1, 0x1.46ca5e0e432d0p-55}, \
}

#if defined(__CUDACC__)
__device__ const double pxg_sc_tab_dev[53][4] = PXG_SC_TAB_INIT;
#endif
static const double pxg_sc_tab_host[53][4] = PXG_SC_TAB_INIT;

typedef struct pxg_dd {
  double hi, lo;
} pxg_dd;

PXG_SC_HD pxg_dd pxg_dd_make(double hi, double lo) {
  pxg_dd r;
  r.hi = hi;
  r.lo = lo;
  return r;
}

/* |a| >= |b| or a == 0 */
PXG_SC_HD pxg_dd pxg_dd_fast_two_sum(double a, double b) {
  const double s = a + b;
  const double e = b - (s - a);
  return pxg_dd_make(s, e);
}

PXG_SC_HD pxg_dd pxg_dd_two_sum(double a, double b) {
  const double s = a + b;
  const double bb = s - a;
  const double e = (a - (s - bb)) + (b - bb);
  return pxg_dd_make(s, e);
}

PXG_SC_HD pxg_dd pxg_dd_mul(pxg_dd a, pxg_dd b) {
  const double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e = e + (a.hi * b.lo + a.lo * b.hi);
  return pxg_dd_fast_two_sum(p, e);
}

PXG_SC_HD pxg_dd pxg_dd_add(pxg_dd a, pxg_dd b) {
  pxg_dd s = pxg_dd_two_sum(a.hi, b.hi);
  s.lo = s.lo + (a.lo + b.lo);
  return pxg_dd_fast_two_sum(s.hi, s.lo);
}

PXG_SC_HD pxg_dd pxg_dd_neg(pxg_dd a) { return pxg_dd_make(-a.hi, -a.lo); }

/* sin(x), cos(x) as normalised double-doubles (|lo| <= ulp(hi)/2). */
PXG_SC_HD void pxg_sincos_dd(double x, pxg_dd* s_out, pxg_dd* c_out) {
  const double ax = fabs(x);
  const double qd = floor(ax * PXG_SC_TWO_OVER_PI + 0.5);
  const int q = (int)qd;
  /* r = ax - q * (C1 + C2 + C3 + C4); ax - q*C1 is exact (Sterbenz, or q = 0) */
  const double t1 = ax - qd * PXG_SC_C1;
  pxg_dd r = pxg_dd_two_sum(t1, -(qd * PXG_SC_C2));
  const double p34 = qd * PXG_SC_C3 + qd * PXG_SC_C4;
  r = pxg_dd_fast_two_sum(r.hi, r.lo - p34);
  /* r = a + s, a = j/64: r.hi - a is exact (Sterbenz, or j = 0) */
  const double jd = floor(fabs(r.hi) * 64.0 + 0.5);
  const int j = (int)jd;
  const double a = r.hi < 0.0 ? -jd * 0.015625 : jd * 0.015625;
  const pxg_dd s = pxg_dd_two_sum(r.hi - a, r.lo);
#if defined(__CUDA_ARCH__)
  const double* tj = pxg_sc_tab_dev[j];
  const double sah = __ldg(tj), sal = __ldg(tj + 1), cah = __ldg(tj + 2), cal = __ldg(tj + 3);
#else
  const double* tj = pxg_sc_tab_host[j];
  const double sah = tj[0], sal = tj[1], cah = tj[2], cal = tj[3];
#endif
  pxg_dd sa = pxg_dd_make(sah, sal);
  const pxg_dd ca = pxg_dd_make(cah, cal);
  if (r.hi < 0.0) sa = pxg_dd_neg(sa);
  /* sin(s) = s + s^3 P(s^2), cos(s) = 1 + s^2 Q(s^2); the tails are < 2^-14 of the result */
  const double y = s.hi, y2 = y * y;
  const double ps = y * y2 * (PXG_SC_F3 + y2 * (PXG_SC_F5 + y2 * (PXG_SC_F7 + y2 * PXG_SC_F9)));
  const double pc = y2 * (PXG_SC_F2 + y2 * (PXG_SC_F4 + y2 * (PXG_SC_F6 + y2 * PXG_SC_F8)));
  const pxg_dd ss = pxg_dd_fast_two_sum(s.hi, s.lo + ps);
  const pxg_dd cs = pxg_dd_fast_two_sum(1.0, pc);
  /* sin(a + s) = sin a cos s + cos a sin s, cos(a + s) = cos a cos s - sin a sin s */
  const pxg_dd sr = pxg_dd_add(pxg_dd_mul(sa, cs), pxg_dd_mul(ca, ss));
  const pxg_dd cr = pxg_dd_add(pxg_dd_mul(ca, cs), pxg_dd_neg(pxg_dd_mul(sa, ss)));
  pxg_dd so, co;
  switch (q & 3) {
    case 0: so = sr; co = cr; break;
    case 1: so = cr; co = pxg_dd_neg(sr); break;
    case 2: so = pxg_dd_neg(sr); co = pxg_dd_neg(cr); break;
    default: so = pxg_dd_neg(cr); co = sr; break;
  }
  if (x < 0.0) so = pxg_dd_neg(so);
  *s_out = so;
  *c_out = co;
}

/* Distance of hi + lo from the rounding boundary of hi, in ulps of hi (0 = a midpoint,
 * 0.5 = exactly representable); normal |hi| > 2^-1000. */
PXG_SC_HD double pxg_dd_round_margin(pxg_dd v) {
  uint64_t b;
#if defined(__CUDA_ARCH__)
  b = (uint64_t)__double_as_longlong(v.hi);
#else
  memcpy(&b, &v.hi, 8);
#endif
  uint64_t e = b & 0x7ff0000000000000ull;
  if (e <= (52ull << 52)) return 0.0;
  e -= 52ull << 52;
  double ulp;
#if defined(__CUDA_ARCH__)
  ulp = __longlong_as_double((long long)e);
#else
  memcpy(&ulp, &e, 8);
#endif
  return 0.5 - fabs(v.lo) / ulp;
}

/* hi's neighbour on lo's side (the value glibc returned instead of hi). */
PXG_SC_HD double pxg_dd_other_neighbour(pxg_dd v) {
  return nextafter(v.hi, v.lo > 0.0 ? INFINITY : -INFINITY);
}

/* ---- glibc agreement table (see the header comment) ---------------------------------- */
#define PXG_SC_RANGES 64
#define PXG_SC_BUCKET_BITS 12
#define PXG_SC_BUCKETS (1u << (32 - PXG_SC_BUCKET_BITS))
#define PXG_SC_MAGIC 0x32435358u /* "XSC2" */

typedef struct pxg_sincos_table {
  const double* thr;       /* [PXG_SC_RANGES][2]: sin, cos */
  const uint32_t* offset;  /* [PXG_SC_BUCKETS + 1] */
  const uint16_t* entry;   /* [offset[PXG_SC_BUCKETS]] */
} pxg_sincos_table;

/* sin(phi), cos(phi) of phi = 2.0 * pi * u with u = k * 2^-32 (the reference's draw), equal
 * to glibc's results bit for bit. */
PXG_SC_HD void pxg_sincos_2pi_glibc(double u, const pxg_sincos_table* T, double* s_out, double* c_out) {
  const double phi = 2.0 * 3.141592653589793238462643383279502884 * u;
  pxg_dd s, c;
  pxg_sincos_dd(phi, &s, &c);
  *s_out = s.hi;
  *c_out = c.hi;
  const uint32_t k = (uint32_t)(u * 4294967296.0);
#if defined(__CUDA_ARCH__)
  const double ts = __ldg(T->thr + 2 * (k >> 26)), tc = __ldg(T->thr + 2 * (k >> 26) + 1);
#else
  const double ts = T->thr[2 * (k >> 26)], tc = T->thr[2 * (k >> 26) + 1];
#endif
  if (pxg_dd_round_margin(s) > ts && pxg_dd_round_margin(c) > tc) return;
  const uint32_t b = k >> PXG_SC_BUCKET_BITS, lowk = k & ((1u << PXG_SC_BUCKET_BITS) - 1u);
#if defined(__CUDA_ARCH__)
  uint32_t e = __ldg(T->offset + b);
  const uint32_t e1 = __ldg(T->offset + b + 1);
#else
  uint32_t e = T->offset[b];
  const uint32_t e1 = T->offset[b + 1];
#endif
  for (; e < e1; ++e) {
#if defined(__CUDA_ARCH__)
    const uint32_t v = __ldg(T->entry + e);
#else
    const uint32_t v = T->entry[e];
#endif
    const uint32_t lv = v & ((1u << PXG_SC_BUCKET_BITS) - 1u);
    if (lv < lowk) continue;
    if (lv == lowk) {
      if (v & (1u << 12)) *s_out = pxg_dd_other_neighbour(s);
      if (v & (1u << 13)) *c_out = pxg_dd_other_neighbour(c);
    }
    break;
  }
}

#endif /* PXG_SINCOS_H */
