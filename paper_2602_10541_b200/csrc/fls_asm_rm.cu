// fls_asm_rm.cu -- row-major assembly A[i * lda + j] (features contiguous), for consumers that
// want rows contiguous.  The column-major kernel with the roles of rows and features swapped:
// each thread owns TWO consecutive features (their records in registers for the whole CTA),
// a CTA covers 512 features x a range of rows, and the rows' x_i (and coefficient fields) are
// staged 64 at a time in shared memory and read as warp-uniform broadcasts.  Every store
// instruction of a warp writes 64 consecutive features = 512 contiguous bytes of one row
// (16-byte st.global.cs per lane).  Same per-entry arithmetic (EntryMath) as the column-major
// kernel, so both layouts hold bit-identical entries.
#include "fls_assemble.cuh"

#ifndef FLS_RM_ROWS
#define FLS_RM_ROWS 2  // rows per iteration of the pair-store loop
#endif

namespace fls {

constexpr int kRmNT = 256;
constexpr int kRmTileF = 2 * kRmNT;   // features per CTA
constexpr int kRmChunk = 64;          // rows staged per shared-memory chunk

__device__ __forceinline__ void rm_cp_async8(double *smem, const double *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void rm_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void rm_cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int D, int G, int KM>
__global__ void __launch_bounds__(kRmNT, asm_min_blocks<D, G, KM>()) assemble_rm_kernel(const AsmArgs a) {
  using M = EntryMath<D, G, KM>;
  constexpr int S = M::S;
  constexpr int GG = G > 0 ? G : 1;
  constexpr int RS = D + GG;          // staged doubles per row
  // two staging buffers: the rows of chunk c + 1 are copied (cp.async, no registers) while
  // chunk c is computed, so the CTA never waits on a global round trip between chunks
  __shared__ __align__(16) double xs[2][kRmChunk * RS];

  const int64_t j = (int64_t)blockIdx.x * kRmTileF + 2 * threadIdx.x;
  const bool jin0 = j < a.F, jin1 = j + 1 < a.F;
  double rec0[S], rec1[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    rec0[s] = jin0 ? __ldg(a.pf + j * S + s) : 0.0;
    rec1[s] = jin1 ? __ldg(a.pf + (j + 1) * S + s) : 0.0;
  }
  const bool pair_ok = a.vec && jin1;
  // phase-range guard (FLS_MAX_PHASE): feature side from the thread's two records, row side
  // max-reduced over the staged rows (per thread, then per warp into s_xinf); exact re-check
  // only past the bound
  __shared__ unsigned long long s_xinf;
  double w1 = 0.0, bb = 0.0;
  {
    double w0 = 0.0, w1b = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      w0 += fabs(rec0[k]);
      w1b += fabs(rec1[k]);
    }
    w1 = fmax(w0, w1b);
    bb = fmax(fabs(rec0[D]), fabs(rec1[D]));
  }
  if (threadIdx.x == 0) s_xinf = 0ull;
  const int64_t r0 = a.lr0 + (int64_t)blockIdx.y * a.fpc;
  const int64_t r1 = r0 + a.fpc < a.lr1 ? r0 + a.fpc : a.lr1;
  bool bad = false;
  double xmax = 0.0;
  auto stage = [&](int64_t rc, int buf) {
    const int nrow = (r1 - rc) < kRmChunk ? (int)(r1 - rc) : kRmChunk;
    for (int t = threadIdx.x; t < nrow * RS; t += kRmNT) {
      const int rr = t / RS, k = t % RS;
      const int64_t i = a.pt0 + (rc + rr - a.lr0);
      if (k < D) rm_cp_async8(&xs[buf][t], a.X + i * D + k);
      else if (G > 0) rm_cp_async8(&xs[buf][t], a.fields + i * a.nf + a.gfield[k - D]);
      else xs[buf][t] = 0.0;
    }
    rm_cp_commit();
  };
  if (r0 < r1) stage(r0, 0);
  int buf = 0;
  for (int64_t rc = r0; rc < r1; rc += kRmChunk, buf ^= 1) {
    const int nrow = (r1 - rc) < kRmChunk ? (int)(r1 - rc) : kRmChunk;
    if (rc + kRmChunk < r1) {
      stage(rc + kRmChunk, buf ^ 1);  // its buffer was last read before the previous barrier
      rm_cp_wait<1>();
    } else {
      rm_cp_wait<0>();
    }
    __syncthreads();  // chunk rc staged by every thread
    for (int t = threadIdx.x; t < nrow * RS; t += kRmNT) {
      const double v = xs[buf][t];
      bad |= !finite(v);
      if (t % RS < D) xmax = fmax(xmax, fabs(v));
    }
    if (blockIdx.x == 0 && a.rhs != nullptr) {
      for (int rr = threadIdx.x; rr < nrow; rr += kRmNT) {
        const int64_t i = a.pt0 + (rc + rr - a.lr0);
        const double v = a.values ? __ldg(a.values + i) : 0.0;
        bad |= !finite(v);
        a.rhs[rc + rr] = a.weight * v;
      }
    }
    const double *xb = xs[buf];
    auto row = [&](int rr, double &o0, double &o1) {
      double x[D], c[GG];
#pragma unroll
      for (int k = 0; k < D; ++k) x[k] = xb[rr * RS + k];
#pragma unroll
      for (int g = 0; g < GG; ++g) c[g] = G > 0 ? xb[rr * RS + D + g] : 0.0;
      o0 = M::entry(rec0, x, c);
      o1 = M::entry(rec1, x, c);
    };
    double *dst = a.A + rc * a.lda + j;
    const int64_t lda = a.lda;
    if (pair_ok) {
      // the common case, branch-free: two rows per iteration (4 independent entries), one
      // 16-byte store per row
      constexpr int RU = FLS_RM_ROWS;
      int rr = 0;
      for (; rr + RU <= nrow; rr += RU, dst += RU * lda) {
        double o[RU][2];
#pragma unroll
        for (int u = 0; u < RU; ++u) row(rr + u, o[u][0], o[u][1]);
#pragma unroll
        for (int u = 0; u < RU; ++u)
          __stcs(reinterpret_cast<double2 *>(dst + u * lda), make_double2(o[u][0], o[u][1]));
      }
      for (; rr < nrow; ++rr, dst += lda) {
        double o0, o1;
        row(rr, o0, o1);
        __stcs(reinterpret_cast<double2 *>(dst), make_double2(o0, o1));
      }
    } else {
      for (int rr = 0; rr < nrow; ++rr, dst += lda) {
        double o0, o1;
        row(rr, o0, o1);
        if (jin0) __stcs(dst, o0);
        if (jin1) __stcs(dst + 1, o1);
      }
    }
    __syncthreads();  // chunk rc's buffer free for the chunk after next
  }
  if (bad) atomicOr(a.err, kErrNonFinite);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) xmax = fmax(xmax, __shfl_xor_sync(0xffffffffu, xmax, off));
  if ((threadIdx.x & 31) == 0) atomicMax(&s_xinf, (unsigned long long)__double_as_longlong(xmax));
  __syncthreads();
  if (fma(w1, __longlong_as_double((long long)s_xinf), bb) > kMaxHalfTurns) {
    for (int64_t r = r0; r < r1; ++r) {   // exact re-check of this thread's two features
      const int64_t i = a.pt0 + (r - a.lr0);
      double h0 = rec0[D], h1 = rec1[D];
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const double xv = __ldg(a.X + i * D + k);
        h0 = fma(rec0[k], xv, h0);
        h1 = fma(rec1[k], xv, h1);
      }
      if ((jin0 && !(fabs(h0) <= kMaxHalfTurns)) || (jin1 && !(fabs(h1) <= kMaxHalfTurns))) {
        atomicOr(a.err, kErrPhaseRange);
        break;
      }
    }
  }
}

template <int D, int G, int KM>
static cudaError_t go_rm(const AsmArgs &a0, cudaStream_t st) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  AsmArgs a = a0;
  const int64_t rows = a.lr1 - a.lr0;
  const int64_t ft = (a.F + kRmTileF - 1) / kRmTileF;
  const int64_t resident = (int64_t)sms * asm_min_blocks<D, G, KM>();
  // >= 4 waves of CTAs, >= 64 rows per CTA (a.fpc = rows per CTA in this kernel)
  int64_t g = (4 * resident + ft - 1) / ft;
  const int64_t gmax = (rows + kRmChunk - 1) / kRmChunk;
  g = g < 1 ? 1 : (g > gmax ? gmax : g);
  a.fpc = (rows + g - 1) / g;
  const dim3 grid((unsigned)ft, (unsigned)((rows + a.fpc - 1) / a.fpc));
  assemble_rm_kernel<D, G, KM><<<grid, kRmNT, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_assemble_rm(int D, int G, int kmode, const AsmArgs &a, cudaStream_t st) {
#define FLS_RM_G(d, km)                              \
  switch (G) {                                       \
    case 0: return go_rm<d, 0, km>(a, st);           \
    case 1: return go_rm<d, 1, km>(a, st);           \
    case 2: return go_rm<d, 2, km>(a, st);           \
    case 3: return go_rm<d, 3, km>(a, st);           \
    case 4: return go_rm<d, 4, km>(a, st);           \
    default: return cudaErrorInvalidValue;           \
  }
#define FLS_RM_D(km)                                 \
  switch (D) {                                       \
    case 1: FLS_RM_G(1, km)                          \
    case 2: FLS_RM_G(2, km)                          \
    case 3: FLS_RM_G(3, km)                          \
    case 4: FLS_RM_G(4, km)                          \
    case 5: FLS_RM_G(5, km)                          \
    case 6: FLS_RM_G(6, km)                          \
    case 7: FLS_RM_G(7, km)                          \
    case 8: FLS_RM_G(8, km)                          \
    default: return cudaErrorInvalidValue;           \
  }
  if (kmode == KM_SIN) {
    FLS_RM_D(KM_SIN)
  } else {
    FLS_RM_D(KM_SINCOS)
  }
#undef FLS_RM_D
#undef FLS_RM_G
}

cudaError_t launch_assemble_cm_sin(int D, int G, AsmArgs *blks, int n, cudaStream_t st, bool pdl);
cudaError_t launch_assemble_cm_sincos(int D, int G, AsmArgs *blks, int n, cudaStream_t st, bool pdl);

cudaError_t launch_assemble_cm(int D, int G, int kmode, AsmArgs *blks, int n, cudaStream_t st,
                               bool pdl) {
  return kmode == KM_SIN ? launch_assemble_cm_sin(D, G, blks, n, st, pdl)
                         : launch_assemble_cm_sincos(D, G, blks, n, st, pdl);
}

}  // namespace fls
