// fls_feat.cuh -- a1 feature draw and a2 prefactor fold as device functions, shared by the
// standalone kernels (fls_kernels.cu) and the fused single-launch assembly (fls_assemble.cuh),
// so that every path draws bit-identical W, b and records.
//
// Product code.  Paper = PAPER.md (arxiv 2602.10541), cited P:L<line>.
#pragma once
#include <stdint.h>

#include "fls_device.cuh"
#include "fls_internal.h"

namespace fls {

// a1 (Alg. 1 line 1): Philox4x64-10 (include/fls.h documents the streams)
__device__ __forceinline__ void philox4x64(uint64_t c[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t M0 = 0xD2E7470EE14C6C93ULL, M1 = 0xCA5A826395121157ULL;
    const uint64_t hi0 = __umul64hi(M0, c[0]), lo0 = M0 * c[0];
    const uint64_t hi1 = __umul64hi(M1, c[2]), lo1 = M1 * c[2];
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
}

__device__ __forceinline__ double u01(uint64_t r) {
  return (double)(r >> 11) * (1.0 / 9007199254740992.0);
}

// sigma of feature j under the multi-block basis: block q covers [ends[q-1], ends[q])
__device__ __forceinline__ double block_sigma(const FeatBlocks &fb, int64_t j) {
  int q = 0;
  while (q + 1 < fb.n && j >= fb.ends[q]) ++q;
  return fb.sigma[q];
}

// normal m (W[m / D][m % D] = sigma_{block} * normal m): Box-Muller on the pair m / 2, raw
// words (m & ~1), (m | 1) of stream 1 (cos for even m, sin for odd m)
__device__ __forceinline__ double feat_normal(int64_t m, int32_t D, const FeatBlocks &fb,
                                              uint64_t seed) {
  const double two_pi = 6.283185307179586476925286766559;
  const int64_t word0 = m & ~int64_t(1);
  uint64_t c[4] = {(uint64_t)(word0 / 4) + 1, 0, 0, 0};
  philox4x64(c, seed, 1);
  const int o = (int)(word0 % 4);
  const double u1 = u01(c[o]), u2 = u01(c[o + 1]);
  const double rad = sqrt(-2.0 * log(1.0 - u1));
  const double th = two_pi * u2;
  double sn, cs;
  sincos(th, &sn, &cs);
  return block_sigma(fb, m / D) * (rad * ((m & 1) ? sn : cs));
}

// b_j = 2 pi u_j, raw word j of stream 2
__device__ __forceinline__ double feat_bias(int64_t j, uint64_t seed) {
  const double two_pi = 6.283185307179586476925286766559;
  uint64_t c[4] = {(uint64_t)(j / 4) + 1, 0, 0, 0};
  philox4x64(c, seed, 2);
  return two_pi * u01(c[j % 4]);
}

// a2 fold of one feature into its record out[0 .. a.S) (layout: fls_internal.h PrefMode).
// Explicit _rn arithmetic: no FMA contraction, so every call site (prefactor_one,
// features_prefactor_kernel, the fused assembly prologue) rounds identically whatever the
// inliner does around it.
// NG > a.G bounds the unrolled group loops (a caller that knows the variant, e.g. the fused
// assembly kernel, passes G + 1 and saves the registers).  w: the feature's D weights (shared or
// global memory).  Latency matters here -- this fold sits on the critical path of every
// assembly step (tools/prologue_latency.py): each term runs only its |alpha| dependent
// multiplies (host-expanded factor list) and the group accumulators are registers.
template <int NG = FLS_MAX_FIELDS + 1>
__device__ inline void prefactor_rec(const PrefArgs &a, const double *w, double bj, double *out) {
  double Ps[NG], Pc[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) Ps[g] = Pc[g] = 0.0;
  for (int t = 0; t < a.n_terms; ++t) {
    const TermDev &T = a.terms[t];
    double m = T.coef;
    int order = 0;
    const int nf = T.nfac;
    if (nf >= 0) {
      for (int e = 0; e < nf; ++e) m = __dmul_rn(m, w[T.fac[e]]);
      order = nf;
    } else {
      for (int k = 0; k < a.D; ++k)
        for (int e = 0; e < T.alpha[k]; ++e) {
          m = __dmul_rn(m, w[k]);
          ++order;
        }
    }
    const int p = order & 3;  // Phi_{|alpha| mod 4}: sin, cos, -sin, -cos
    if (p & 2) m = -m;
    const int grp = T.group;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      if (grp == g) {
        if (p & 1)
          Pc[g] = __dadd_rn(Pc[g], m);
        else
          Ps[g] = __dadd_rn(Ps[g], m);
      }
    }
  }
  for (int k = 0; k < a.D; ++k) out[k] = __dmul_rn(w[k], kInvPi);
  const double bp = bj;
  double *q = out + a.D + 1;
  int used = a.D + 1;
  switch (a.pmode) {
    case PM_SIN:
#pragma unroll
      for (int g = 0; g < NG; ++g)
        if (g <= a.G) q[g] = a.scale * Ps[g];
      used += a.G + 1;
      out[a.D] = __dmul_rn(bp, kInvPi);
      break;
    case PM_COSSHIFT:  // cos z = sin(z + pi/2)  (App. F quarter-wave shift)
#pragma unroll
      for (int g = 0; g < NG; ++g)
        if (g <= a.G) q[g] = a.scale * Pc[g];
      used += a.G + 1;
      out[a.D] = __dadd_rn(__dmul_rn(bp, kInvPi), 0.5);
      break;
    case PM_FOLD: {    // Ps sin z + Pc cos z = rho sin(z + psi)
      const double ps = a.scale * Ps[0], pc = a.scale * Pc[0];
      const double rho = hypot(ps, pc);
      const double psi = atan2(pc, ps);
      q[0] = rho;
      used += 1;
      out[a.D] = __dmul_rn(__dadd_rn(bp, psi), kInvPi);
      break;
    }
    default:           // PM_SINCOS
#pragma unroll
      for (int g = 0; g < NG; ++g)
        if (g <= a.G) {
          q[2 * g] = a.scale * Ps[g];
          q[2 * g + 1] = a.scale * Pc[g];
        }
      used += 2 * (a.G + 1);
      out[a.D] = __dmul_rn(bp, kInvPi);
      break;
  }
  for (int o = used; o < a.S; ++o) out[o] = 0.0;
}

}  // namespace fls
