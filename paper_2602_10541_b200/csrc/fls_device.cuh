// fls_device.cuh -- device-side building blocks shared by the libfls kernels.
//
// Product code (CUDA path).  Nothing here is shared with oracle/ (DESIGN.md §2).
//
// Half-turn trigonometry.  The kernels carry the phase in half turns,
//     h = z / pi = sum_k (W_jk / pi) x_ik + b_j / pi,
// with W / pi and b / pi prescaled once per feature (prefactor kernel), so the phase costs d
// DFMA and no multiply by 1/pi.  Range reduction to f = h - n, n = rint(h), |f| <= 1/2, uses
// the 1.5 * 2^52 magic constant (2 DADD + 1 DADD, no F2I / I2F conversions), and
//     sin(z) = (-1)^n sin(pi f),   cos(z) = (-1)^n cos(pi f),
// with (-1)^n applied by an integer XOR on the sign bit.  sin(pi f) = f p(f^2) (7 coefficients,
// max abs error 3.97e-14) and cos(pi f) = q(f^2) (8 coefficients, 1.08e-14) are minimax fits
// produced by tools/fit_sinpoly.py.  Budget per sin: 3 DADD + 1 DMUL + 6 DFMA + 1 DMUL.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fls.h"

namespace fls {

constexpr double kPi = 3.141592653589793238462643383279502884;
constexpr double kInvPi = 0.318309886183790671537767526745028724;
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: x + kMagic rounds x to an integer
// phase-range guard (fls.h FLS_MAX_PHASE, in radians) in half turns: |h| beyond it sets bit 1 of
// the ctx error word (FLS_EUNSUPPORTED at the next fls_sync)
constexpr double kMaxHalfTurns = FLS_MAX_PHASE * kInvPi;
constexpr unsigned kErrNonFinite = 1u, kErrPhaseRange = 2u;

// Coefficients live in constant memory so DFMA reads them as c[bank][offset] operands
// (no per-iteration materialisation of 64-bit immediates).
// sin(pi f) = f * p(f^2), |f| <= 1/2 -- tools/fit_sinpoly.py 7 sin
static __constant__ double kSinC[7] = {0x1.921fb544422b9p+1, -0x1.4abbce622b70dp+2,
                                       0x1.466bc666fa76ep+1, -0x1.32d2c80461e85p-1,
                                       0x1.5076b5c39bedfp-4, -0x1.e289957d36087p-8,
                                       0x1.d3d9ca396c5b5p-12};
// cos(pi f) = q(f^2), |f| <= 1/2 -- tools/fit_sinpoly.py 8 cos
static __constant__ double kCosC[8] = {1.0, -0x1.3bd3cc9be45b0p+2, 0x1.03c1f081b29f6p+2,
                                       -0x1.55d3c7e0ba51dp+0, 0x1.e1f504256b638p-3,
                                       -0x1.a6d11187be151p-6, 0x1.f97f5b4f53910p-10,
                                       -0x1.a75f6839218cdp-14};

__device__ __forceinline__ double sinpi_core(double f, double u) {
  double p = kSinC[6];
  p = fma(p, u, kSinC[5]);
  p = fma(p, u, kSinC[4]);
  p = fma(p, u, kSinC[3]);
  p = fma(p, u, kSinC[2]);
  p = fma(p, u, kSinC[1]);
  p = fma(p, u, kSinC[0]);
  return f * p;
}

__device__ __forceinline__ double cospi_core(double u) {
  double q = kCosC[7];
  q = fma(q, u, kCosC[6]);
  q = fma(q, u, kCosC[5]);
  q = fma(q, u, kCosC[4]);
  q = fma(q, u, kCosC[3]);
  q = fma(q, u, kCosC[2]);
  q = fma(q, u, kCosC[1]);
  q = fma(q, u, kCosC[0]);
  return q;
}

// h (phase in half turns) -> f in [-1/2, 1/2] and the sign word (n odd -> 0x80000000).
// Valid for |h| < 2^51; accuracy of the caller's h is ~ulp(|h|).
__device__ __forceinline__ double halfturn(double h, int &sgn) {
  const double t = __dadd_rn(h, kMagic);
  sgn = __double2loint(t) << 31;
  const double n = __dsub_rn(t, kMagic);
  return __dsub_rn(h, n);
}

__device__ __forceinline__ double flipsign(double x, int sgn) {
  return __hiloint2double(__double2hiint(x) ^ sgn, __double2loint(x));
}

// the same reduction returning n mod 2^32 (the low word of t) instead of the sign mask
__device__ __forceinline__ double halfturn_n(double h, int &nlo) {
  const double t = __dadd_rn(h, kMagic);
  nlo = __double2loint(t);
  const double n = __dsub_rn(t, kMagic);
  return __dsub_rn(h, n);
}

// (-1)^n x: adding (n << 31) to the high word flips its sign bit exactly when n is odd (the
// carry out of bit 31 is discarded), bit-identical to the XOR form, and the shift-and-add is a
// single LEA where the XOR form needs a shift and a LOP3
__device__ __forceinline__ double addsign(double x, int nlo) {
  return __hiloint2double(__double2hiint(x) + (nlo << 31), __double2loint(x));
}

// sin(pi h) for any |h| < 2^51
__device__ __forceinline__ double sin_halfturns(double h) {
  int sgn;
  const double f = halfturn(h, sgn);
  return sinpi_core(flipsign(f, sgn), f * f);
}

// Programmatic dependent launch (sm_90+): the prefactor kernels let the assembly grid that
// follows them on the stream launch at once (pdl_trigger at entry); the assembly kernel loads
// its points, then waits for the prefactor grid's completion and memory flush (pdl_wait)
// before reading the records.  Both are no-ops when the launch has no PDL attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ bool finite(double v) {
  // exponent field all ones <=> Inf / NaN
  return (__double2hiint(v) & 0x7ff00000) != 0x7ff00000;
}

}  // namespace fls
