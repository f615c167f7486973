// ct.cuh — compile-time helpers: static_for and constexpr roots of unity.
//
// Every butterfly twiddle that is known at compile time (all of the in-register
// sub-FFTs) becomes an FFMA immediate; trivial ones (1, -i, (1-i)/sqrt2) are
// special-cased with `if constexpr` so they cost no multiplies.
#pragma once

#include <utility>

namespace rdfft {
namespace ct {

template <int I>
using ic = std::integral_constant<int, I>;

template <int B, int E, typename F, int... Is>
__host__ __device__ __forceinline__ constexpr void static_for_impl(F&& f, std::integer_sequence<int, Is...>) {
  (f(ic<B + Is>{}), ...);
}
// f(ic<i>) for i in [B, E)
template <int B, int E, typename F>
__host__ __device__ __forceinline__ constexpr void static_for(F&& f) {
  if constexpr (E > B) static_for_impl<B, E>(static_cast<F&&>(f), std::make_integer_sequence<int, E - B>{});
}

constexpr double kPi = 3.14159265358979323846264338327950288;

// sin / cos of x in [-pi/4, pi/4] by Taylor series (double, exact to rounding).
constexpr double sin_small(double x) {
  double t = x, s = x;
  for (int k = 1; k < 14; ++k) {
    t *= -x * x / ((2 * k) * (2 * k + 1));
    s += t;
  }
  return s;
}
constexpr double cos_small(double x) {
  double t = 1, s = 1;
  for (int k = 1; k < 14; ++k) {
    t *= -x * x / ((2 * k - 1) * (2 * k));
    s += t;
  }
  return s;
}
// cos(2 pi a / b) and sin(2 pi a / b) for integers, octant-reduced so that the
// exact values at multiples of pi/4 come out exactly rounded.
constexpr double cos2pi(long a, long b) {
  a %= b;
  if (a < 0) a += b;
  // reduce to first octant: angle = 2 pi a / b = (pi/4) * (8a/b)
  const long o8 = 8 * a;        // angle in units of pi/4 is o8 / b
  const long oct = o8 / b;      // octant 0..7
  const double r = (double)(o8 - oct * b) / (double)b * (kPi / 4);  // remainder angle in [0, pi/4)
  const double c = cos_small(r), s = sin_small(r);
  const double cq = cos_small(kPi / 4 - r), sq = sin_small(kPi / 4 - r);
  switch (oct) {
    case 0: return c;
    case 1: return sq;   // cos(pi/4 + r) = sin(pi/4 - r)
    case 2: return -s;   // cos(pi/2 + r)
    case 3: return -cq;  // cos(3pi/4 + r) = -cos(pi/4 - r)
    case 4: return -c;
    case 5: return -sq;
    case 6: return s;
    default: return cq;
  }
}
constexpr double sin2pi(long a, long b) { return cos2pi(a * 4 - b, 4 * b); }  // sin x = cos(x - pi/2)

// W_b^a = exp(-2 pi i a / b) = (cos, -sin)
template <long A, long B>
struct W {
  static constexpr float re = (float)cos2pi(A, B);
  static constexpr float im = (float)(-sin2pi(A, B));
};

// tan / cot of the angle of W_B^A (for the tangent-form butterflies)
template <long A, long B>
struct Wt {
  static constexpr float tan = (float)(-sin2pi(A, B) / cos2pi(A, B));  // im / re
  static constexpr float cot = (float)(cos2pi(A, B) / -sin2pi(A, B));  // re / im
};

}  // namespace ct
}  // namespace rdfft
