// pxg_math.cuh — fp64 vector math for the path kernels.
//
// Every operator keeps the reference's evaluation order (proj/include/proxima/vec.hpp:11-71):
// dot = (ax*bx + ay*by) + az*bz, v / s = v * (1/s), normalize = v * (1/length(v)), and the
// branchless Duff ONB. The device build uses --fmad=false so no multiply-add is fused;
// together this makes a kernel vertex bit-identical to the reference vertex for the same
// random draws (up to the 1-2 ulp spread of sin/cos between CUDA and glibc).
#pragma once

#include <cmath>
#include <cstdint>

#if defined(__CUDACC__)
#define PXD __host__ __device__ __forceinline__
#else
#define PXD inline
#endif

namespace pxg {

constexpr double kPi = 3.141592653589793238462643383279502884;

struct V3 {
  double x, y, z;
};

PXD V3 v3(double s) { return {s, s, s}; }
PXD V3 v3(double x, double y, double z) { return {x, y, z}; }
PXD V3 operator-(const V3& a) { return {-a.x, -a.y, -a.z}; }
PXD V3 operator+(const V3& a, const V3& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
PXD V3 operator-(const V3& a, const V3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
PXD V3 operator*(const V3& a, const V3& b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
PXD V3 operator*(const V3& a, double s) { return {a.x * s, a.y * s, a.z * s}; }
PXD V3 operator*(double s, const V3& a) { return {a.x * s, a.y * s, a.z * s}; }
PXD V3 operator/(const V3& a, double s) { return a * (1.0 / s); }
PXD V3& operator+=(V3& a, const V3& b) { a.x += b.x; a.y += b.y; a.z += b.z; return a; }
PXD double get(const V3& v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : v.z); }

PXD double dot(const V3& a, const V3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
PXD V3 cross(const V3& a, const V3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
PXD double length_sq(const V3& v) { return dot(v, v); }
PXD double length(const V3& v) { return sqrt(dot(v, v)); }
PXD V3 normalize(const V3& v) { return v / length(v); }
PXD double luminance(const V3& c) { return 0.2126 * c.x + 0.7152 * c.y + 0.0722 * c.z; }
PXD bool near_zero(const V3& v) { return v.x == 0.0 && v.y == 0.0 && v.z == 0.0; }
PXD bool is_finite(const V3& v) { return isfinite(v.x) && isfinite(v.y) && isfinite(v.z); }
PXD V3 reflect(const V3& w, const V3& n) { return 2.0 * dot(w, n) * n - w; }
PXD double dmax(double a, double b) { return (a < b) ? b : a; }  // std::max argument order
PXD double dmin(double a, double b) { return (b < a) ? b : a; }  // std::min argument order

// Orthonormal basis (vec.hpp:59-71).
struct Frame {
  V3 n, t, b;
  PXD explicit Frame(const V3& n_) : n(n_) {
    const double sign = copysign(1.0, n.z);
    const double a = -1.0 / (sign + n.z);
    t = v3(1.0 + sign * n.x * n.x * a, sign * n.x * n.y * a, -sign * n.x);
    b = v3(n.x * n.y * a, sign + n.y * n.y * a, -n.y);
  }
  PXD V3 to_world(const V3& v) const { return v.x * t + v.y * b + v.z * n; }
  PXD V3 to_local(const V3& v) const { return {dot(v, t), dot(v, b), dot(v, n)}; }
};

}  // namespace pxg
