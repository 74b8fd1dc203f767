// microbench.cu -- roofline denominators for the assembly path, built into
// a separate libfls_microbench.so (not part of the product ABI).
//
//   mb_store_bw     store-only HBM bandwidth with the assembly kernel's exact store pattern
//                   (16-byte st.global.cs, 512 contiguous bytes per warp instruction)
//   mb_dfma_rate    register-only DFMA throughput (8 independent chains per thread)
//   mb_entry_rate   register-only throughput of the assembly kernel's per-entry arithmetic
//                   (d = 3 phase, half-turn reduction, degree-13 sin, one coefficient field),
//                   with the C5-class kernel's ILP (4 rows x 4 features per iteration)
//                   = the FP64-pipe ceiling of the C5 kernel with no memory traffic at all
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "../fls_device.cuh"

using namespace fls;

extern "C" {

__global__ void __launch_bounds__(256) store_kernel(double *A, int64_t n2, double v) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double2 *p = reinterpret_cast<double2 *>(A);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride)
    __stcs(p + i, make_double2(v, v + 1.0));
}

__global__ void __launch_bounds__(256) dfma_kernel(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[threadIdx.x] = s;  // never true; keeps the chains alive
}

// per thread: 4 rows in registers and 4 features per iteration (as the C5-class assembly
// kernel: 16 independent entries in flight), the entry arithmetic exactly as EntryMath (phase,
// half-turn reduction, (-1)^n on the argument, degree-13 sin, one coefficient field); each
// result is folded into an integer XOR (one LOP3, standing in for the kernel's store) so no
// floating-point dependency links the entries
__global__ void __launch_bounds__(256, 3) entry_kernel(double *out, int nfeat, double w0, double w1,
                                                       double w2) {
  const double x[4][3] = {{0.1 + threadIdx.x * 1e-4, 0.2, 0.3}, {0.4, 0.5 + blockIdx.x * 1e-6, 0.6},
                          {0.7, 0.8, 0.9}, {0.15, 0.25, 0.35}};
  const double c[4] = {1.1, 1.2, 1.3, 1.4};
  int bits = 0;
  double wa = w0, wb = w1, wc = w2, bp = 0.1, P0 = 2.0, P1 = 3.0;
  for (int j = 0; j < nfeat; j += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double wau = wa + 1e-3 * u, bpu = bp + 2e-3 * u;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double h = fma(wc, x[q][2], fma(wb, x[q][1], fma(wau, x[q][0], bpu)));
        int sgn;
        const double f = halfturn(h, sgn);
        const double u2 = f * f;
        const double P = fma(c[q], P1, P0);
        bits ^= __double2hiint(P * sinpi_core(flipsign(f, sgn), u2));
      }
    }
    wa += 4e-3;  // per-iteration change (the kernel's smem record loads)
    bp += 8e-3;
  }
  if (bits == 0x12345678) out[threadIdx.x] = bits;
}

// the assembly kernel's exact tile/store pattern with no arithmetic: 1024-row x 128-column
// tiles, 4 rows per thread as two 16-byte pairs, one column per iteration
__global__ void __launch_bounds__(256) tile_store_kernel(double *A, int64_t lda, int ncols, double v) {
  double *colp = A + (int64_t)blockIdx.y * 128 * lda + (int64_t)blockIdx.x * 1024 + 2 * threadIdx.x;
  const int nc = min(128, ncols - (int)blockIdx.y * 128);
  for (int j = 0; j < nc; ++j, colp += lda) {
    __stcs(reinterpret_cast<double2 *>(colp), make_double2(v, v + j));
    __stcs(reinterpret_cast<double2 *>(colp + 512), make_double2(v + 1.0, v - j));
  }
}

// contiguous streaming: each CTA writes one contiguous 256 KiB chunk
__global__ void __launch_bounds__(256) chunk_store_kernel(double *A, double v) {
  double2 *p = reinterpret_cast<double2 *>(A) + (int64_t)blockIdx.x * 16384 + threadIdx.x;
#pragma unroll 4
  for (int k = 0; k < 64; ++k) __stcs(p + k * 256, make_double2(v, v + k));
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// returns 0 on success; *gbs = bytes / s / 1e9 over `reps` launches (after one warm-up)
__attribute__((visibility("default"))) int mb_store_bw(double *A, int64_t n_doubles, int reps,
                                                       double *gbs) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 8;
  store_kernel<<<grid, 256>>>(A, n_doubles / 2, 1.0);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) store_kernel<<<grid, 256>>>(A, n_doubles / 2, 1.0 + r);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  *gbs = (double)n_doubles * 8.0 * reps / (time_ms(e0, e1) / 1e3) / 1e9;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return (int)cudaGetLastError();
}

__attribute__((visibility("default"))) int mb_dfma_rate(double *scratch, int iters, double *dfma_per_s) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 8;
  dfma_kernel<<<grid, 256>>>(scratch, 1000, 0.999, 1e-3);
  cudaEventRecord(e0);
  dfma_kernel<<<grid, 256>>>(scratch, iters, 0.999, 1e-3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  *dfma_per_s = (double)grid * 256 * iters * 8 / (time_ms(e0, e1) / 1e3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return (int)cudaGetLastError();
}

__attribute__((visibility("default"))) int mb_entry_rate(double *scratch, int nfeat, double *entries_per_s) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 8;
  entry_kernel<<<grid, 256>>>(scratch, 100, 1.0, 2.0, 3.0);
  cudaEventRecord(e0);
  entry_kernel<<<grid, 256>>>(scratch, nfeat, 1.0, 2.0, 3.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  *entries_per_s = (double)grid * 256 * 4 * nfeat / (time_ms(e0, e1) / 1e3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return (int)cudaGetLastError();
}

// rows must be a multiple of 1024, cols of 128; A holds cols * lda doubles
__attribute__((visibility("default"))) int mb_tile_store_bw(double *A, int64_t rows, int64_t lda,
                                                            int cols, int reps, double *gbs) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dim3 grid((unsigned)(rows / 1024), (unsigned)((cols + 127) / 128));
  tile_store_kernel<<<grid, 256>>>(A, lda, cols, 1.0);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) tile_store_kernel<<<grid, 256>>>(A, lda, cols, 2.0 + r);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  *gbs = (double)rows * cols * 8.0 * reps / (time_ms(e0, e1) / 1e3) / 1e9;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return (int)cudaGetLastError();
}

// n_doubles must be a multiple of 32768
__attribute__((visibility("default"))) int mb_chunk_store_bw(double *A, int64_t n_doubles, int reps,
                                                             double *gbs) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const unsigned grid = (unsigned)(n_doubles / 32768);
  chunk_store_kernel<<<grid, 256>>>(A, 1.0);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) chunk_store_kernel<<<grid, 256>>>(A, 2.0 + r);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  *gbs = (double)n_doubles * 8.0 * reps / (time_ms(e0, e1) / 1e3) / 1e9;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return (int)cudaGetLastError();
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// per-op FP64 throughput: 8 independent chains per thread of one op kind
template <int OP>
__global__ void __launch_bounds__(256) op_kernel(double *out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k + 0.25;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) x[k] = __dadd_rn(x[k], a);
      if (OP == 1) x[k] = __dmul_rn(x[k], a);
      if (OP == 2) x[k] = fma(x[k], a, b);
      if (OP == 3) x[k] = rint(x[k]) + a;          // FRND + DADD
      if (OP == 4) x[k] = (double)(__double2int_rn(x[k]) + 1);   // F2I + I2F
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// entry kernel variant: rint (FRND) + integer parity instead of the magic-constant rounding
__device__ __forceinline__ double halfturn_frnd(double h, int &sgn) {
  const double n = rint(h);
  // parity of n from the integer bits of n (n exact, |n| < 2^31): low bit of the converted int
  // computed on the integer pipe from the mantissa
  const int hi = __double2hiint(n), lo = __double2loint(n);
  const int e = ((hi >> 20) & 0x7ff) - 1023;          // n = 1.m * 2^e, e in [0, 30] when n != 0
  // units bit of n sits at mantissa bit (52 - e): in lo for e >= 21, in hi for e < 21
  const int bit = (e < 0) ? 0 : (e == 0 ? 1 : (e <= 20 ? (hi >> (20 - e)) & 1 : (lo >> (52 - e)) & 1));
  sgn = bit << 31;
  return __dsub_rn(h, n);
}

__global__ void __launch_bounds__(256) entry2_kernel(double *out, int nfeat, double w0, double w1,
                                                     double w2) {
  const double x[4][3] = {{0.1 + threadIdx.x * 1e-4, 0.2, 0.3}, {0.4, 0.5 + blockIdx.x * 1e-6, 0.6},
                          {0.7, 0.8, 0.9}, {0.15, 0.25, 0.35}};
  const double c[4] = {1.1, 1.2, 1.3, 1.4};
  double acc[4] = {0, 0, 0, 0};
  double wa = w0, wb = w1, wc = w2, bp = 0.1, P0 = 2.0, P1 = 3.0;
  for (int j = 0; j < nfeat; ++j) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double h = fma(wc, x[q][2], fma(wb, x[q][1], fma(wa, x[q][0], bp)));
      int sgn;
      const double f = halfturn_frnd(h, sgn);
      const double P = fma(c[q], P1, P0);
      acc[q] += P * sinpi_core(flipsign(f, sgn), f * f);
    }
    wa += 1e-3;
    bp += 2e-3;
  }
  const double s = acc[0] + acc[1] + acc[2] + acc[3];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// FP64 tensor path: mma.sync m8n8k4 f64 (DMMA); MODE 0 = DMMA only, 1 = DMMA + DFMA chains
// interleaved (does the tensor path run beside the FP64 ALU pipe?), 2 = the DFMA chains alone
template <int MODE>
__global__ void __launch_bounds__(256) dmma_kernel(double *out, int iters, double a, double b) {
  double acc[4][2];
  double x[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) acc[k][0] = acc[k][1] = threadIdx.x * 1e-3 + k;
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k + 0.5;
  const double av = a + threadIdx.x * 1e-9, bv = b;
  for (int i = 0; i < iters; ++i) {
    if (MODE <= 1) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        asm volatile(
            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
            : "+d"(acc[k][0]), "+d"(acc[k][1])
            : "d"(av), "d"(bv));
    }
    if (MODE >= 1) {
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += acc[k][0] + acc[k][1];
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// returns DMMA instructions/s (warp-level) and DFMA/s for the selected mode
extern "C" __attribute__((visibility("default"))) int mb_dmma_rate(int mode, double *scratch,
                                                                   int iters, double *dmma_per_s,
                                                                   double *dfma_per_s) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 8;
  auto go = [&](int it) {
    if (mode == 0) dmma_kernel<0><<<grid, 256>>>(scratch, it, 0.999, 1e-3);
    if (mode == 1) dmma_kernel<1><<<grid, 256>>>(scratch, it, 0.999, 1e-3);
    if (mode == 2) dmma_kernel<2><<<grid, 256>>>(scratch, it, 0.999, 1e-3);
  };
  go(100);
  cudaEventRecord(e0);
  go(iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  const double s = time_ms(e0, e1) / 1e3;
  const double warps = (double)grid * 8;
  *dmma_per_s = (mode <= 1) ? warps * iters * 4 / s : 0.0;
  *dfma_per_s = (mode >= 1) ? (double)grid * 256 * iters * 8 / s : 0.0;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return (int)cudaGetLastError();
}

extern "C" __attribute__((visibility("default"))) int mb_op_rate(int op, double *scratch, int iters,
                                                                 double *ops_per_s) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 8;
  auto go = [&](int it) {
    switch (op) {
      case 0: op_kernel<0><<<grid, 256>>>(scratch, it, 1e-9, 1e-3); break;
      case 1: op_kernel<1><<<grid, 256>>>(scratch, it, 0.9999999, 1e-3); break;
      case 2: op_kernel<2><<<grid, 256>>>(scratch, it, 0.9999999, 1e-3); break;
      case 3: op_kernel<3><<<grid, 256>>>(scratch, it, 0.25, 1e-3); break;
      case 4: op_kernel<4><<<grid, 256>>>(scratch, it, 0.25, 1e-3); break;
      case 5: entry2_kernel<<<grid, 256>>>(scratch, it, 1.0, 2.0, 3.0); break;
    }
  };
  go(100);
  cudaEventRecord(e0);
  go(iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  const double per = (op == 5) ? 4.0 : 8.0;
  *ops_per_s = (double)grid * 256 * iters * per / (time_ms(e0, e1) / 1e3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// latency (clock64 cycles, one thread) of the pieces of the fused assembly prologue (a1 + a2):
// out[0] Philox4x64-10 block, out[1] feat_normal (Philox + Box-Muller), out[2] feat_bias,
// out[3] prefactor_rec of a 2-term operator (C2's -Laplacian), out[4] log + sqrt alone,
// out[5] sincos alone
// ------------------------------------------------------------------------------------------
#include "../fls_feat.cuh"

// pass 0 runs cold (instruction cache misses on the SM), pass 1 warm: out[0..5] cold, out[6..11] warm
__global__ void prologue_latency_kernel(long long *out_all, double *sink, uint64_t seed, PrefArgs pa) {
  double acc = 0.0;
  long long t0, t1;
  __shared__ double w[2], rec[8];
  for (int pass = 0; pass < 2; ++pass) {
  long long *out = out_all + 6 * pass;
  uint64_t c[4] = {(uint64_t)threadIdx.x + 7, 0, 0, 0};
  t0 = clock64();
  philox4x64(c, seed, 1);
  acc += (double)(c[0] & 0xff);
  t1 = clock64();
  out[0] = t1 - t0;
  const FeatBlocks fb = {1, {1 << 20}, {5.0}};
  t0 = clock64();
  acc += feat_normal((int64_t)(acc) + 3, 2, fb, seed);
  t1 = clock64();
  out[1] = t1 - t0;
  t0 = clock64();
  acc += feat_bias((int64_t)(acc * 0) + 5, seed);
  t1 = clock64();
  out[2] = t1 - t0;
  w[0] = acc * 1e-3;
  w[1] = 1.5;
  t0 = clock64();
  prefactor_rec(pa, w, acc, rec);
  acc += rec[3];
  t1 = clock64();
  out[3] = t1 - t0;
  const double u = 0.3 + acc * 1e-12;
  t0 = clock64();
  acc += sqrt(-2.0 * log(1.0 - u));
  t1 = clock64();
  out[4] = t1 - t0;
  double sn, cs;
  t0 = clock64();
  sincos(6.283185307179586 * (u + acc * 1e-15), &sn, &cs);
  acc += sn + cs;
  t1 = clock64();
  out[5] = t1 - t0;
  }
  sink[0] = acc;
}

extern "C" __attribute__((visibility("default"))) int mb_prologue_latency(long long *out_host) {
  long long *d;
  double *sink;
  cudaMalloc(&d, 12 * sizeof(long long));
  cudaMalloc(&sink, sizeof(double));
  PrefArgs pa;
  memset(&pa, 0, sizeof pa);
  pa.D = 2;
  pa.n_terms = 2;
  pa.G = 0;
  pa.pmode = PM_SIN;
  pa.S = 4;
  pa.scale = 0.02;
  pa.terms[0].coef = -1.0;
  pa.terms[0].alpha[0] = 2;
  pa.terms[0].nfac = 2;
  pa.terms[0].fac[0] = pa.terms[0].fac[1] = 0;
  pa.terms[1].coef = -1.0;
  pa.terms[1].alpha[1] = 2;
  pa.terms[1].nfac = 2;
  pa.terms[1].fac[0] = pa.terms[1].fac[1] = 1;
  for (int rep = 0; rep < 3; ++rep) prologue_latency_kernel<<<1, 1>>>(d, sink, 0, pa);
  cudaMemcpy(out_host, d, 12 * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  cudaFree(sink);
  return (int)cudaGetLastError();
}
