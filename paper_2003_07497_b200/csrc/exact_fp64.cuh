// exact_fp64.cuh — correctly rounded FP64 division and square root with a short, branch-free
// common path, for the latency-bound Adam step of the exact-order trainer (mlp.cpp:142-154).
//
// CUDA's __ddiv_rn / __dsqrt_rn are correctly rounded but wrap their fast paths in reconvergence
// regions with out-of-line slow paths; inside the Adam step of train_fp64_pipe the three divisions
// and the square root then cost ~1000 cycles per epoch, on the epoch's critical path.
//
// Here every candidate result comes from a seed (MUFU reciprocal / reciprocal square root),
// Newton refinement and one FMA correction step, and is then VERIFIED exactly:
//   division  q = RN(a/b)  iff  |a - b*q| < |b| * ulp_below(q) / 2   (no exact midpoints exist for a
//             quotient of two doubles), with a - b*q computed exactly by one FMA;
//   sqrt      s = RN(sqrt(v)) iff |v - s*s| < s * ulp_below(s)        (no midpoints either),
// using the smaller neighbour spacing (conservative at binade edges) and a 2^-40 relative safety
// margin; operands outside a safe exponent range (zeros, subnormals, huge values, inf, NaN) fail
// the check too. A caller computes its whole step on the fast path, ANDs the flags, and redoes the
// step with __ddiv_rn / __dsqrt_rn when any flag is false — so the result is the correctly
// rounded one in every case: bit-identical to the reference's IEEE division and sqrt.
#pragma once

namespace lann {

__device__ __forceinline__ double rcp_seed(double b) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
  return y;
}
__device__ __forceinline__ double rsqrt_seed(double v) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v));
  return y;
}

// |x| in [2^-900, 2^900] (finite, normal, far from under/overflow of the products below)
__device__ __forceinline__ bool safe_range(double x) {
  const unsigned hi = static_cast<unsigned>(__double2hiint(x)) & 0x7fffffffu;
  return hi >= 0x07b00000u && hi < 0x78300000u;  // biased exponent in [123, 1923)
}

// half the spacing of doubles just below positive normal x (x's ulp, halved again at a power of 2)
__device__ __forceinline__ double half_ulp_below(double x) {
  const long long bits = __double_as_longlong(x);
  const long long ex = (bits >> 52) & 0x7ff;
  const bool pow2 = (bits & 0xfffffffffffffLL) == 0;
  return __longlong_as_double((ex - 53 - (pow2 ? 1 : 0)) << 52);
}

// refined reciprocal of b (relative error ~2^-104 before rounding): depends on b only
__device__ __forceinline__ double rcp_refined(double b) {
  const double y0 = rcp_seed(b);
  const double e = __fma_rn(-b, y0, 1.0);
  const double y1 = __fma_rn(y0, __fma_rn(e, e, e), y0);
  const double e2 = __fma_rn(-b, y1, 1.0);
  return __fma_rn(y1, e2, y1);
}

// RN(a / b) given y = rcp_refined(b); ok &= the result is verified correctly rounded
__device__ __forceinline__ double div_checked(double a, double b, double y, bool& ok) {
  const double q0 = __dmul_rn(a, y);
  const double r = __fma_rn(-b, q0, a);
  const double q = __fma_rn(r, y, q0);
  const double r2 = __fma_rn(-b, q, a);  // exact for a faithful q
  const double lim = __dmul_rn(fabs(b), __dmul_rn(half_ulp_below(fabs(q)), 0.99999999999909051));
  ok = ok & safe_range(a) & safe_range(b) & safe_range(q) & (fabs(r2) < lim);  // no short circuit: branch-free
  return q;
}

// RN(sqrt(v)); ok &= verified
__device__ __forceinline__ double sqrt_checked(double v, bool& ok) {
  const double y0 = rsqrt_seed(v);
  const double t = __dmul_rn(y0, y0);
  const double e = __fma_rn(-v, t, 1.0);                                   // 1 - v y^2
  const double y = __fma_rn(__dmul_rn(y0, e), __fma_rn(0.375, e, 0.5), y0);  // y (1 + e/2 + 3e^2/8)
  const double s0 = __dmul_rn(v, y);
  const double r = __fma_rn(-s0, s0, v);
  const double s = __fma_rn(r, __dmul_rn(0.5, y), s0);
  const double r2 = __fma_rn(-s, s, v);  // exact for a faithful s
  const double lim = __dmul_rn(s, __dmul_rn(2.0 * half_ulp_below(s), 0.99999999999909051));
  ok = ok & safe_range(v) & (fabs(r2) < lim);
  return s;
}

// The ReLU and its gate (mlp.cpp:49,102): v where c > 0, else +0.0 (a NaN c gives +0.0, as the
// reference's comparison does). Two 32-bit selects on one predicate: the plain ternary compiles
// to a NaN-aware max sequence (~6 instructions) on the layer-to-layer dependency path
// (train_fp64_pipe's producers: 436 -> 384 instructions per sample, config 2 FP64 53.5 -> 51.2 ms).
__device__ __forceinline__ double gate(double c, double v) {
  const bool on = c > 0.0;
  const int hi = on ? __double2hiint(v) : 0, lo = on ? __double2loint(v) : 0;
  return __hiloint2double(hi, lo);
}

}  // namespace lann
