// fls_assemble.cuh -- the hot kernel: closed-form operator-matrix assembly (Eq. 2-3).
//
//   A_ij = sum_g c_g(x_i) (Ps_gj sin z_ij + Pc_gj cos z_ij),   z_ij = W_j . x_i + b_j
//
// (Eq. 2 folded per feature by the prefactor kernel; Eq. 3 row blocks).
// HBM-write-bound (8 B per entry) with the FP64 pipe as co-bound (d + 12 DFMA-class ops per
// entry in the sin-only family).
//
// Column-major layout A[j * lda + i] (what cuSOLVER geqrf consumes):
//   CTA = 256 threads, tile = 1024 rows x 128 features.  Thread t owns the row pairs
//   (2t, 2t+1) and (512 + 2t, 512 + 2t + 1) of the tile -- its x_i stay in registers for the
//   whole tile -- so every store instruction of a warp writes 64 consecutive rows = 512
//   contiguous bytes of one column, as one 16-byte st.global.cs per lane (streaming: the
//   output is never re-read by this kernel).  The tile's 128 per-feature records
//   [W_j/pi, b'_j/pi, P_j...] sit in shared memory and are read as warp-wide broadcasts.
#pragma once
#include "fls_device.cuh"
#include "fls_internal.h"

namespace fls {

template <int D, int G, int KM>
__global__ void __launch_bounds__(kNT) assemble_cm_kernel(const AsmArgs a) {
  constexpr int NP = (G + 1) * (KM == KM_SINCOS ? 2 : 1);
  constexpr int S = pf_stride(D, G, KM);
  static_assert(S % 2 == 0, "pf stride must be even for 16-byte smem reads");
  extern __shared__ __align__(16) double sp[];

  const int64_t j0 = (int64_t)blockIdx.y * kFC;
  const int64_t nfe64 = a.F - j0;
  const int nfe = nfe64 < kFC ? (int)nfe64 : kFC;
  {
    const double2 *src = reinterpret_cast<const double2 *>(a.pf + j0 * S);
    double2 *dst = reinterpret_cast<double2 *>(sp);
    const int n2 = nfe * (S / 2);
    for (int t = threadIdx.x; t < n2; t += kNT) dst[t] = __ldg(src + t);
  }

  // local rows (A-relative) of this thread: rbase + {0, 1, 2*kNT, 2*kNT + 1}; rbase is even.
  // The block's points map to local rows [lr0, lr1): point i = pt0 + (r - lr0).
  const int64_t rbase = (a.lr0 & ~int64_t(1)) + (int64_t)blockIdx.x * kRowsCTA + 2 * threadIdx.x;
  double x[4][D];
  double c[4][G > 0 ? G : 1];
  bool in[4];
  bool bad = false;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t r = rbase + (q >> 1) * (2 * kNT) + (q & 1);
    in[q] = (r >= a.lr0) && (r < a.lr1);
    const int64_t i = a.pt0 + (r - a.lr0);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      x[q][k] = in[q] ? __ldg(a.X + i * D + k) : 0.0;
      bad |= !finite(x[q][k]);
    }
#pragma unroll
    for (int g = 0; g < (G > 0 ? G : 1); ++g) {
      c[q][g] = (G > 0 && in[q]) ? __ldg(a.fields + i * a.nf + a.gfield[g]) : 0.0;
      bad |= !finite(c[q][g]);
    }
    if (blockIdx.y == 0 && a.rhs != nullptr && in[q]) {
      const double v = a.values ? __ldg(a.values + i) : 0.0;
      bad |= !finite(v);
      a.rhs[r] = a.weight * v;
    }
  }
  if (bad) atomicOr(a.err, 1u);
  __syncthreads();

  const bool full = a.vec && in[0] && in[1] && in[2] && in[3];
  double *colp = a.A + j0 * a.lda + rbase;
  for (int jj = 0; jj < nfe; ++jj, colp += a.lda) {
    const double *p = sp + jj * S;
    double rec[S];
#pragma unroll
    for (int s2 = 0; s2 < S / 2; ++s2) {
      const double2 v = reinterpret_cast<const double2 *>(p)[s2];
      rec[2 * s2] = v.x;
      rec[2 * s2 + 1] = v.y;
    }
    double out[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double h = rec[D];
#pragma unroll
      for (int k = 0; k < D; ++k) h = fma(rec[k], x[q][k], h);
      int sgn;
      const double f = halfturn(h, sgn);
      const double u = f * f;
      if constexpr (KM == KM_SIN) {
        double P = rec[D + 1];
#pragma unroll
        for (int g = 0; g < G; ++g) P = fma(c[q][g], rec[D + 2 + g], P);
        out[q] = P * sinpi_core(flipsign(f, sgn), u);
      } else {
        double Ps = rec[D + 1], Pc = rec[D + 2];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          Ps = fma(c[q][g], rec[D + 3 + 2 * g], Ps);
          Pc = fma(c[q][g], rec[D + 4 + 2 * g], Pc);
        }
        out[q] = flipsign(fma(Ps, sinpi_core(f, u), Pc * cospi_core(u)), sgn);
      }
    }
    (void)NP;
    if (full) {
      __stcs(reinterpret_cast<double2 *>(colp), make_double2(out[0], out[1]));
      __stcs(reinterpret_cast<double2 *>(colp + 2 * kNT), make_double2(out[2], out[3]));
    } else {
#pragma unroll
      for (int pr = 0; pr < 2; ++pr) {
        double *dst = colp + pr * (2 * kNT);
        if (a.vec && in[2 * pr] && in[2 * pr + 1]) {
          __stcs(reinterpret_cast<double2 *>(dst), make_double2(out[2 * pr], out[2 * pr + 1]));
        } else {
          if (in[2 * pr]) __stcs(dst, out[2 * pr]);
          if (in[2 * pr + 1]) __stcs(dst + 1, out[2 * pr + 1]);
        }
      }
    }
  }
}

}  // namespace fls
