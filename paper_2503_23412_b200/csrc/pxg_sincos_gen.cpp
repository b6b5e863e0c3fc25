// pxg_sincos_gen — builds the glibc agreement table of include/pxg_sincos.h from this host's
// libm, and verifies it.
//
//   pxg_sincos_gen OUT.bin                   evaluate all 2^32 angles phi = 2*pi*(k * 2^-32),
//                                            write the table (build step, ~2 min on 8 cores)
//   pxg_sincos_gen --verify IN.bin [k0 k1]   pxg_sincos_2pi_glibc with the table == glibc
//                                            sin, cos and sincos on k in [k0, k1) (default:
//                                            all); prints one JSON line, exit 1 on any
//                                            difference
//   pxg_sincos_gen --eval KS.u32 OUT.f64      glibc sin, cos of the listed draws (parity
//                                            tests of the device code path)
//
// glibc is called through volatile function pointers so neither constant folding nor GCC's
// sin+cos -> sincos fusion changes the libm entry points compared; sincos() is checked too
// (GCC -O2 fuses the reference's adjacent std::cos(phi) / std::sin(phi) into one call).
// The angles are those of the reference's samplers: proj/src/bsdf.cpp:63-65, 226-227,
// proj/src/scene.cpp:199-201 (u = next_double() = k * 2^-32).
//
// File layout (little endian): u32 magic, u32 n_entries, f64 thr[64][2], u32 offset[2^20 + 1],
// u16 entry[n_entries].
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "pxg_sincos.h"

extern "C" void sincos(double, double*, double*);

namespace {
constexpr double kPi = 3.141592653589793238462643383279502884;
double (*volatile g_sin)(double) = std::sin;
double (*volatile g_cos)(double) = std::cos;
void (*volatile g_sincos)(double, double*, double*) = sincos;

uint64_t bits(double x) {
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return b;
}

template <typename F>
void parallel(uint64_t k0, uint64_t k1, F&& f) {
  unsigned nt = std::thread::hardware_concurrency();
  if (const char* e = std::getenv("PXG_SC_THREADS")) nt = static_cast<unsigned>(std::atoi(e));
  nt = std::max(nt, 1u);
  // chunks of 2^20 k handed out in order so each thread sees whole buckets
  const uint64_t chunk = 1ull << 20;
  std::mutex mu;
  uint64_t next = k0;
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&]() {
      for (;;) {
        uint64_t a;
        {
          std::lock_guard<std::mutex> lk(mu);
          a = next;
          next += chunk;
        }
        if (a >= k1) break;
        f(a, std::min(k1, a + chunk), mu);
      }
    });
  for (auto& x : th) x.join();
}

int generate(const char* path) {
  // flags per k: 1 sin differs, 2 cos differs; kept per bucket
  std::vector<std::vector<uint16_t>> bucket(PXG_SC_BUCKETS);
  std::vector<double> thr(2 * PXG_SC_RANGES, -1.0);
  uint64_t nsin = 0, ncos = 0, nsc = 0;
  parallel(0, 1ull << 32, [&](uint64_t a, uint64_t b, std::mutex& mu) {
    std::vector<std::pair<uint32_t, uint16_t>> found;
    std::vector<double> t(2 * PXG_SC_RANGES, -1.0);
    uint64_t ds = 0, dc = 0, dsc = 0;
    for (uint64_t k = a; k < b; ++k) {
      const double u = static_cast<double>(static_cast<uint32_t>(k)) * 0x1p-32;
      const double phi = 2.0 * kPi * u;
      pxg_dd s, c;
      pxg_sincos_dd(phi, &s, &c);
      const double gs = g_sin(phi), gc = g_cos(phi);
      double gs2, gc2;
      g_sincos(phi, &gs2, &gc2);
      dsc += bits(gs2) != bits(gs) || bits(gc2) != bits(gc);
      uint16_t f = 0;
      if (bits(gs) != bits(s.hi)) {
        if (bits(gs) != bits(pxg_dd_other_neighbour(s))) std::abort();  // glibc off by more than one neighbour
        f |= 1u << 12;
        t[2 * (k >> 26)] = std::max(t[2 * (k >> 26)], pxg_dd_round_margin(s));
        ++ds;
      }
      if (bits(gc) != bits(c.hi)) {
        if (bits(gc) != bits(pxg_dd_other_neighbour(c))) std::abort();
        f |= 1u << 13;
        t[2 * (k >> 26) + 1] = std::max(t[2 * (k >> 26) + 1], pxg_dd_round_margin(c));
        ++dc;
      }
      if (f) found.emplace_back(static_cast<uint32_t>(k), f | static_cast<uint16_t>(k & 0xfffu));
    }
    std::lock_guard<std::mutex> lk(mu);
    for (auto& [k, v] : found) bucket[k >> PXG_SC_BUCKET_BITS].push_back(v);
    for (int i = 0; i < 2 * PXG_SC_RANGES; ++i) thr[i] = std::max(thr[i], t[i]);
    nsin += ds;
    ncos += dc;
    nsc += dsc;
  });
  if (nsc) {
    std::fprintf(stderr, "pxg_sincos_gen: sincos() differs from sin()/cos() on %llu angles\n",
                 static_cast<unsigned long long>(nsc));
    return 1;
  }
  std::vector<uint32_t> off(PXG_SC_BUCKETS + 1, 0);
  std::vector<uint16_t> ent;
  for (uint32_t b = 0; b < PXG_SC_BUCKETS; ++b) {
    auto& v = bucket[b];
    std::sort(v.begin(), v.end(), [](uint16_t x, uint16_t y) { return (x & 0xfffu) < (y & 0xfffu); });
    off[b] = static_cast<uint32_t>(ent.size());
    ent.insert(ent.end(), v.begin(), v.end());
  }
  off[PXG_SC_BUCKETS] = static_cast<uint32_t>(ent.size());
  const std::string tmp = std::string(path) + ".tmp";
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) return 1;
  const uint32_t hdr[2] = {PXG_SC_MAGIC, static_cast<uint32_t>(ent.size())};
  std::fwrite(hdr, sizeof(hdr), 1, f);
  std::fwrite(thr.data(), sizeof(double), thr.size(), f);
  std::fwrite(off.data(), sizeof(uint32_t), off.size(), f);
  std::fwrite(ent.data(), sizeof(uint16_t), ent.size(), f);
  if (std::fclose(f) != 0 || std::rename(tmp.c_str(), path) != 0) return 1;
  std::printf("{\"angles\": 4294967296, \"sin_differ\": %llu, \"cos_differ\": %llu, \"entries\": %zu}\n",
              static_cast<unsigned long long>(nsin), static_cast<unsigned long long>(ncos), ent.size());
  return 0;
}

int verify(const char* path, uint64_t k0, uint64_t k1) {
  FILE* f = std::fopen(path, "rb");
  if (!f) {
    std::fprintf(stderr, "pxg_sincos_gen: cannot open %s\n", path);
    return 1;
  }
  uint32_t hdr[2];
  std::vector<double> thr(2 * PXG_SC_RANGES);
  std::vector<uint32_t> off(PXG_SC_BUCKETS + 1);
  bool ok = std::fread(hdr, sizeof(hdr), 1, f) == 1 && hdr[0] == PXG_SC_MAGIC;
  std::vector<uint16_t> ent(ok ? hdr[1] : 0);
  ok = ok && std::fread(thr.data(), sizeof(double), thr.size(), f) == thr.size() &&
       std::fread(off.data(), sizeof(uint32_t), off.size(), f) == off.size() &&
       std::fread(ent.data(), sizeof(uint16_t), ent.size(), f) == ent.size();
  std::fclose(f);
  if (!ok) {
    std::fprintf(stderr, "pxg_sincos_gen: bad table %s\n", path);
    return 1;
  }
  const pxg_sincos_table T{thr.data(), off.data(), ent.data()};
  uint64_t diff = 0, lookups = 0;
  std::vector<uint64_t> ex;
  parallel(k0, k1, [&](uint64_t a, uint64_t b, std::mutex& mu) {
    uint64_t d = 0, l = 0;
    std::vector<uint64_t> e;
    for (uint64_t k = a; k < b; ++k) {
      const double u = static_cast<double>(static_cast<uint32_t>(k)) * 0x1p-32;
      const double phi = 2.0 * kPi * u;
      double s, c, gs2, gc2;
      pxg_sincos_2pi_glibc(u, &T, &s, &c);
      const double gs = g_sin(phi), gc = g_cos(phi);
      g_sincos(phi, &gs2, &gc2);
      const bool bad = bits(s) != bits(gs) || bits(c) != bits(gc) || bits(s) != bits(gs2) || bits(c) != bits(gc2);
      d += bad;
      if (bad && e.size() < 8) e.push_back(k);
      pxg_dd sd, cd;
      pxg_sincos_dd(phi, &sd, &cd);
      l += !(pxg_dd_round_margin(sd) > thr[2 * (k >> 26)] && pxg_dd_round_margin(cd) > thr[2 * (k >> 26) + 1]);
    }
    std::lock_guard<std::mutex> lk(mu);
    diff += d;
    lookups += l;
    if (ex.size() < 8) ex.insert(ex.end(), e.begin(), e.end());
  });
  std::printf("{\"checked\": %llu, \"differ\": %llu, \"table_searches\": %llu, \"entries\": %u, \"first\": [",
              static_cast<unsigned long long>(k1 - k0), static_cast<unsigned long long>(diff),
              static_cast<unsigned long long>(lookups), hdr[1]);
  for (size_t i = 0; i < ex.size(); ++i) std::printf("%s%llu", i ? ", " : "", static_cast<unsigned long long>(ex[i]));
  std::printf("]}\n");
  return diff ? 1 : 0;
}

int eval(const char* kpath, const char* opath) {
  FILE* f = std::fopen(kpath, "rb");
  if (!f) return 1;
  std::vector<uint32_t> ks;
  uint32_t buf[4096];
  size_t got;
  while ((got = std::fread(buf, sizeof(uint32_t), 4096, f)) > 0) ks.insert(ks.end(), buf, buf + got);
  std::fclose(f);
  std::vector<double> out(2 * ks.size());
  for (size_t i = 0; i < ks.size(); ++i) {
    const double phi = 2.0 * kPi * (static_cast<double>(ks[i]) * 0x1p-32);
    out[2 * i] = g_sin(phi);
    out[2 * i + 1] = g_cos(phi);
  }
  FILE* o = std::fopen(opath, "wb");
  if (!o) return 1;
  const bool ok = std::fwrite(out.data(), sizeof(double), out.size(), o) == out.size();
  return (std::fclose(o) == 0 && ok) ? 0 : 1;
}
}  // namespace

int main(int argc, char** argv) {
  if (argc == 4 && std::strcmp(argv[1], "--eval") == 0) return eval(argv[2], argv[3]);
  if (argc >= 3 && std::strcmp(argv[1], "--verify") == 0) {
    uint64_t k0 = 0, k1 = 1ull << 32;
    if (argc >= 5) {
      k0 = std::strtoull(argv[3], nullptr, 0);
      k1 = std::min<uint64_t>(std::strtoull(argv[4], nullptr, 0), 1ull << 32);
    }
    return verify(argv[2], k0, k1);
  }
  if (argc != 2) {
    std::fprintf(stderr, "usage: pxg_sincos_gen OUT.bin | --verify IN.bin [k0 k1]\n");
    return 2;
  }
  return generate(argv[1]);
}
