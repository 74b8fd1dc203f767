// fls_asm_rm.cu -- row-major assembly A[i * lda + j] (features contiguous), for consumers that
// want rows contiguous (e.g. a row-streaming normal-equations build).  Same arithmetic per
// entry as the column-major kernel (bit-identical entries).  A warp covers 64 consecutive
// features of one row (one 16-byte store per lane); each lane keeps its two feature records
// in registers and the row's x_i is a broadcast load.
#include "fls_device.cuh"
#include "fls_internal.h"

namespace fls {

template <int D>
__global__ void __launch_bounds__(256) assemble_rm_kernel(const AsmArgs a, int G, int km, int S) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.y * kRmFeat + 2 * lane;
  constexpr int MAXREC = FLS_MAX_DIM + 2 + 2 * (FLS_MAX_FIELDS + 1);
  double rec[2][MAXREC];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const bool ok = (j + e) < a.F;
#pragma unroll
    for (int s = 0; s < MAXREC; ++s) rec[e][s] = (ok && s < S) ? __ldg(a.pf + (j + e) * S + s) : 0.0;
  }
  bool bad = false;
  for (int k8 = 0; k8 < kRmRows / 8; ++k8) {
    const int64_t r = a.lr0 + (int64_t)blockIdx.x * kRmRows + warp + 8 * k8;
    if (r >= a.lr1) break;
    const int64_t i = a.pt0 + (r - a.lr0);
    double x[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      x[k] = __ldg(a.X + i * D + k);
      bad |= !finite(x[k]);
    }
    double c[FLS_MAX_FIELDS];
#pragma unroll
    for (int g = 0; g < FLS_MAX_FIELDS; ++g) {
      c[g] = (g < G) ? __ldg(a.fields + i * a.nf + a.gfield[g]) : 0.0;
      bad |= !finite(c[g]);
    }
    if (blockIdx.y == 0 && lane == 0 && a.rhs != nullptr) {
      const double v = a.values ? __ldg(a.values + i) : 0.0;
      bad |= !finite(v);
      a.rhs[r] = a.weight * v;
    }
    double out[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      double h = rec[e][D];
#pragma unroll
      for (int k = 0; k < D; ++k) h = fma(rec[e][k], x[k], h);
      int sgn;
      const double f = halfturn(h, sgn);
      const double u = f * f;
      if (km == KM_SIN) {
        double P = rec[e][D + 1];
#pragma unroll
        for (int g = 0; g < FLS_MAX_FIELDS; ++g)
          if (g < G) P = fma(c[g], rec[e][D + 2 + g], P);
        out[e] = P * sinpi_core(flipsign(f, sgn), u);
      } else {
        double Ps = rec[e][D + 1], Pc = rec[e][D + 2];
#pragma unroll
        for (int g = 0; g < FLS_MAX_FIELDS; ++g)
          if (g < G) {
            Ps = fma(c[g], rec[e][D + 3 + 2 * g], Ps);
            Pc = fma(c[g], rec[e][D + 4 + 2 * g], Pc);
          }
        out[e] = flipsign(fma(Ps, sinpi_core(f, u), Pc * cospi_core(u)), sgn);
      }
    }
    double *dst = a.A + r * a.lda + j;
    if (a.vec && j + 1 < a.F) {
      __stcs(reinterpret_cast<double2 *>(dst), make_double2(out[0], out[1]));
    } else {
      if (j < a.F) __stcs(dst, out[0]);
      if (j + 1 < a.F) __stcs(dst + 1, out[1]);
    }
  }
  if (bad) atomicOr(a.err, 1u);
}

cudaError_t launch_assemble_rm(int D, int G, int kmode, const AsmArgs &a, cudaStream_t st) {
  const int S = pf_stride(D, G, kmode);
  const dim3 grid((unsigned)((a.lr1 - a.lr0 + kRmRows - 1) / kRmRows),
                  (unsigned)((a.F + kRmFeat - 1) / kRmFeat));
  switch (D) {
#define FLS_RM(d) \
  case d: assemble_rm_kernel<d><<<grid, 256, 0, st>>>(a, G, kmode, S); break;
    FLS_RM(1) FLS_RM(2) FLS_RM(3) FLS_RM(4) FLS_RM(5) FLS_RM(6) FLS_RM(7) FLS_RM(8)
#undef FLS_RM
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_assemble_cm_sin(int D, int G, AsmArgs *blks, int n, cudaStream_t st);
cudaError_t launch_assemble_cm_sincos(int D, int G, AsmArgs *blks, int n, cudaStream_t st);

cudaError_t launch_assemble_cm(int D, int G, int kmode, AsmArgs *blks, int n, cudaStream_t st) {
  return kmode == KM_SIN ? launch_assemble_cm_sin(D, G, blks, n, st)
                         : launch_assemble_cm_sincos(D, G, blks, n, st);
}

}  // namespace fls
