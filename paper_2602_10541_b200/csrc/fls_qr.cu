// fls_qr.cu -- blocked Householder QR for the least-squares solve (Alg. 1 line 5, P:L124;
// Tikhonov form P:L156-160).  Output format = LAPACK / cuSOLVER geqrf: R in the upper
// trapezoid, the Householder vectors v_j (v_jj = 1 implicit) below the diagonal, tau_j, so
// cuSOLVER ormqr and cuBLAS trsv consume it unchanged.
//
// Why not one cusolverDnDgeqrf call: on this pool's B200 its panel factorisation costs ~30-65 us
// per column (a few launches each), so geqrf runs at 6 / 16 / 22 TFLOP/s on C3 / C4 / C5-subset
// while DGEMM runs at 34-36 TFLOP/s at the same shapes (tools/probe_dgemm.py).  Here:
//   * outer loop over panels of nb columns (compact WY: H_1..H_nb = I - V T V^T), the trailing
//     matrix updated by two DGEMMs and one DTRMM per panel;
//   * each panel factored recursively (Elmroth-Gustavson): left half, WY update of the right
//     half, right half, then T12 = -T1 (V1^T V2) T2 -- all cuBLAS DGEMM / DTRMM;
//   * the recursion's leaves (<= 32 columns, fewer when the rows are many) run in ONE
//     cooperative kernel per leaf: each CTA keeps its row slab of the leaf in shared memory,
//     and one grid-wide barrier per column separates "partial sums of ||x||^2 and x^T a_c over
//     my rows" from "finish dlarfg, update my rows", so a leaf column costs one grid sync
//     instead of several kernel launches and no global-memory pass.
// Householder vector per column (LAPACK dlarfg): beta = -sign(alpha) ||[alpha; x]||,
// tau = (beta - alpha) / beta, v = x / (alpha - beta); ||x|| = 0 gives tau = 0 (H = I).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "fls_internal.h"


namespace fls {

constexpr int kQrB = 32;    // leaf width (columns per cooperative kernel)
constexpr int kQrNT = 256;  // threads per CTA of the leaf kernel
constexpr int kQrW = kQrNT / 32;
constexpr size_t kQrSlab = 216 * 1024;  // shared-memory slab budget per CTA (one CTA per SM)
constexpr int kQrMaxGrid = 256;         // leaf CTAs at most (one per SM)
constexpr int kQrMinLeaf = 4;           // narrowest leaf; taller blocks go to cuSOLVER

struct QrLeafArgs {
  double *A;     // leaf top-left (its diagonal starts at row 0), column-major
  int64_t lda;
  int64_t m;     // rows from the leaf's top
  int64_t rc;    // rows per CTA (the shared-memory slab height)
  int32_t b;     // columns (<= kQrB)
  double *V;     // explicit V (zeros above, ones on the diagonal), same row origin as A
  int64_t ldv;
  double *tau;
  double *part;  // [2][kQrB + 1][gridDim.x] per-CTA partial sums (slot-major)
  double *rowb;  // [2][kQrB + 1] the diagonal row a_jj.. at the start of column jj
  unsigned *bar; // grid-barrier arrival counter (zeroed before the launch)
};

// grid-wide barrier of a cooperative launch (all CTAs co-resident): monotonically increasing
// arrival counter, release-add by one thread per CTA, acquire-poll until every CTA of round
// `round` has arrived
__device__ __forceinline__ void qr_grid_barrier(unsigned *bar, unsigned round) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = (round + 1) * gridDim.x;
    // release: the CTA's writes before the __syncthreads above are visible to any CTA that
    // acquires the counter value (PTX memory model: bar.sync + release is cumulative)
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// block-reduce the per-thread partial sums of column jj (slot 0: ||x||^2, slot q: x^T a_{jj+q})
// and publish them (slot-major) plus, from the owner CTA, the diagonal row a_{jj, jj..}
__device__ __forceinline__ void qr_publish(double (&acc)[kQrB], double (*red)[kQrB + 1],
                                           const double *slab, int64_t rc, int64_t r_lo, int nr,
                                           int jj, int nc, double *part, double *rowb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // 32 warp sums in 31 shuffles (recursive halving): afterwards lane l holds sum of acc[l]
#pragma unroll
  for (int sh = 16; sh >= 1; sh >>= 1) {
    const bool up = lane & sh;
#pragma unroll
    for (int t = 0; t < sh; ++t) {
      const double send = up ? acc[t] : acc[t + sh];
      const double keep = up ? acc[t + sh] : acc[t];
      acc[t] = keep + __shfl_xor_sync(0xffffffffu, send, sh);
    }
  }
  red[warp][lane] = acc[0];
  __syncthreads();  // also orders the slab updates before the row publication below
  if (threadIdx.x < nc) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kQrW; ++w) s += red[w][threadIdx.x];
    part[(int64_t)threadIdx.x * gridDim.x + blockIdx.x] = s;  // slot-major: coalesced reads
  }
  if (jj >= r_lo && jj < r_lo + nr && threadIdx.x < nc)
    rowb[threadIdx.x] = slab[(jj + threadIdx.x) * rc + (jj - r_lo)];
}

// One leaf (b <= 32 columns, m rows) of the recursive QR.  CTA k owns rows [k rc, (k+1) rc)
// and keeps them (b columns) in shared memory for the whole leaf: the global memory traffic is
// one read and one write of the leaf plus the per-column partial sums.  The update of column
// jj's reflector and the partial sums of column jj+1 share one pass over the slab.
__global__ void __launch_bounds__(kQrNT) qr_leaf_kernel(const QrLeafArgs a) {
  extern __shared__ __align__(16) double slab[];  // [b][rc], column-major
  __shared__ double red[kQrW][kQrB + 1];
  __shared__ double tot[kQrB + 1];
  __shared__ double s_tau, s_scale, s_beta;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t rc = a.rc;
  const int64_t r_lo = (int64_t)blockIdx.x * rc;
  const int nr = (int)(r_lo >= a.m ? 0 : (a.m - r_lo < rc ? a.m - r_lo : rc));
  const int b = a.b;
  // all b loads of a row in flight before the first shared-memory store (one memory round trip
  // per row instead of one per column)
  for (int r = threadIdx.x; r < nr; r += kQrNT) {
    double v[kQrB];
#pragma unroll
    for (int q = 0; q < kQrB; ++q)
      if (q < b) v[q] = a.A[(int64_t)q * a.lda + r_lo + r];
#pragma unroll
    for (int q = 0; q < kQrB; ++q)
      if (q < b) slab[q * rc + r] = v[q];
  }
  __syncthreads();
  double acc[kQrB];
  {  // partial sums of column 0 over my rows below the diagonal
#pragma unroll
    for (int q = 0; q < kQrB; ++q) acc[q] = 0.0;
    const int r0 = 1 - r_lo > 0 ? (int)(1 - r_lo) : 0;
    for (int r = r0 + threadIdx.x; r < nr; r += kQrNT) {
      const double x = slab[r];
      acc[0] = fma(x, x, acc[0]);
#pragma unroll
      for (int q = 1; q < kQrB; ++q)
        if (q < b) acc[q] = fma(x, slab[q * rc + r], acc[q]);
    }
    qr_publish(acc, red, slab, rc, r_lo, nr, 0, b, a.part, a.rowb);
  }
  for (int jj = 0; jj < b; ++jj) {
    const int nc = b - jj;
    const double *part = a.part + (size_t)(jj & 1) * gridDim.x * (kQrB + 1);
    const double *rowb = a.rowb + (jj & 1) * (kQrB + 1);
    qr_grid_barrier(a.bar, (unsigned)jj);
    // ---- every warp: totals of slot 0 and of its own slots q (same order in every CTA; all
    // loads issued before any use: one L2 round trip), then dlarfg redundantly, then
    // tot[q] = tau * v^T a_{jj+q} (v_jj = 1)
    {
      constexpr int NS = (kQrB + kQrW - 1) / kQrW;  // own slots per warp
      const int q0 = warp > 0 ? warp : kQrW;
      double v0 = 0.0, vs[NS], rq[NS];
#pragma unroll
      for (int i = 0; i < NS; ++i) vs[i] = rq[i] = 0.0;
#pragma unroll
      for (int t = 0; t < kQrMaxGrid / 32; ++t) {
        const unsigned k = lane + 32 * t;
        if (k < gridDim.x) {
          v0 += part[k];                         // the barrier's acquire invalidated L1
#pragma unroll
          for (int i = 0; i < NS; ++i) {
            const int q = q0 + kQrW * i;
            if (q < nc) vs[i] += part[(int64_t)q * gridDim.x + k];
          }
        }
      }
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        const int q = q0 + kQrW * i;
        if (q < nc) rq[i] = rowb[q];
      }
      const double alpha = rowb[0];
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
#pragma unroll
        for (int i = 0; i < NS; ++i) vs[i] += __shfl_xor_sync(0xffffffffu, vs[i], o);
      }
      double tau = 0.0, scale = 0.0, beta = alpha;
      if (v0 > 0.0) {
        // ||[alpha; x]|| without hypot's rescaling (entries here are far from over/underflow)
        // and one division for both tau = (beta - alpha) / beta and 1 / (alpha - beta)
        beta = -copysign(sqrt(fma(alpha, alpha, v0)), alpha);
        const double d = alpha - beta;
        const double inv = 1.0 / (beta * d);
        tau = -d * d * inv;
        scale = beta * inv;
      }
      if (threadIdx.x == 0) {
        s_tau = tau;
        s_scale = scale;
        s_beta = beta;
        if (blockIdx.x == 0) a.tau[jj] = tau;
      }
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        const int q = q0 + kQrW * i;
        if (q < nc && lane == 0) tot[q] = tau * fma(scale, vs[i], rq[i]);
      }
    }
    __syncthreads();
    const double tau = s_tau, scale = s_scale;
    // ---- apply H_jj to my rows of the remaining columns (v overwrites x below the diagonal)
    // and accumulate column jj+1's partial sums over rows below ITS diagonal
#pragma unroll
    for (int q = 0; q < kQrB; ++q) acc[q] = 0.0;
    double *xw = slab + jj * rc;
    const int rd = jj - r_lo >= 0 ? (int)(jj - r_lo) : -1;  // my row index of the diagonal
    for (int r = (rd > 0 ? rd : 0) + threadIdx.x; r < nr; r += kQrNT) {
      if (r > rd) {
        const double v = tau != 0.0 ? xw[r] * scale : xw[r];
        xw[r] = v;
        const bool below = r_lo + r > jj + 1;  // contributes to column jj+1's sums
        double xn = 0.0;
#pragma unroll
        for (int q = 1; q < kQrB; ++q) {
          if (q < nc) {
            const double nv = xw[q * rc + r] - v * tot[q];
            xw[q * rc + r] = nv;
            if (below) {
              if (q == 1) {
                xn = nv;
                acc[0] = fma(nv, nv, acc[0]);
              } else {
                acc[q - 1] = fma(xn, nv, acc[q - 1]);
              }
            }
          }
        }
      } else {  // r == rd: the diagonal row
        xw[r] = s_beta;
#pragma unroll
        for (int q = 1; q < kQrB; ++q)
          if (q < nc) xw[q * rc + r] -= tot[q];
      }
    }
    if (jj + 1 < b)
      qr_publish(acc, red, slab, rc, r_lo, nr, jj + 1, nc - 1,
                 a.part + (size_t)((jj + 1) & 1) * gridDim.x * (kQrB + 1),
                 a.rowb + ((jj + 1) & 1) * (kQrB + 1));
  }
  __syncthreads();
  // write back R / v and the explicit V (zeros above, ones on the diagonal)
  for (int q = 0; q < b; ++q)
    for (int r = threadIdx.x; r < nr; r += kQrNT) {
      const int64_t i = r_lo + r;
      const double x = slab[q * rc + r];
      a.A[(int64_t)q * a.lda + i] = x;
      a.V[(int64_t)q * a.ldv + i] = i > q ? x : (i == q ? 1.0 : 0.0);
    }
}

// T of a leaf from S = V^T V (b x b) and tau (LAPACK dlarft, forward, columnwise):
// T_jj = tau_j, T(0:j, j) = -tau_j T(0:j, 0:j) S(0:j, j)
__global__ void qr_larft_kernel(const double *S, int b, const double *tau, double *T, int64_t ldt) {
  __shared__ double Ts[kQrB][kQrB + 1];
  __shared__ double Ss[kQrB][kQrB + 1];
  __shared__ double tmp[kQrB], taus[kQrB];
  const int i = threadIdx.x;
  if (i < b) {
    for (int j = 0; j < b; ++j) Ss[i][j] = S[(int64_t)j * b + i];
    taus[i] = tau[i];
  }
  __syncthreads();
  for (int j = 0; j < b; ++j) {
    if (i < j) {
      double t = 0.0;
      for (int l = i; l < j; ++l) t += Ts[i][l] * Ss[l][j];
      tmp[i] = -taus[j] * t;
    }
    __syncthreads();
    if (i < b) Ts[i][j] = i < j ? tmp[i] : (i == j ? taus[j] : 0.0);
    __syncthreads();
  }
  if (i < b)
    for (int j = 0; j < b; ++j) T[(int64_t)j * ldt + i] = Ts[i][j];
}

int64_t qr_leaf_rows();

namespace {

struct QrCtx {
  cublasHandle_t h;
  cudaStream_t st;
  double *A;
  int64_t lda;
  double *V;     // panel V, ldv rows
  int64_t ldv;
  double *T;     // nb x nb
  int64_t ldt;
  double *W;     // nb x n scratch
  double *S;     // kQrB x kQrB
  double *part, *rowb;
  unsigned *bar;   // leaf grid-barrier counter
  int grid;        // CTAs of a leaf launch (one per SM)
  int bleaf;       // leaf width for the current panel (slab fits shared memory)
  const char *fail = nullptr;
  cudaError_t cerr = cudaSuccess;
  cublasStatus_t berr = CUBLAS_STATUS_SUCCESS;
};

bool ok_blas(QrCtx &q, cublasStatus_t s, const char *what) {
  if (s != CUBLAS_STATUS_SUCCESS && q.berr == CUBLAS_STATUS_SUCCESS) {
    q.berr = s;
    q.fail = what;
  }
  return s == CUBLAS_STATUS_SUCCESS;
}

bool ok_cuda(QrCtx &q, cudaError_t e, const char *what) {
  if (e != cudaSuccess && q.cerr == cudaSuccess) {
    q.cerr = e;
    q.fail = what;
  }
  return e == cudaSuccess;
}

// factor panel columns [c, c+w) (rows [c, mp) of the panel whose top-left is P), filling V and
// the diagonal block T[c:c+w, c:c+w] of the panel's T
bool rec_panel(QrCtx &q, double *P, int64_t mp, int64_t c, int64_t w, double *tau) {
  const double one = 1.0, zero = 0.0, mone = -1.0;
  double *Vc = q.V + c * q.ldv;  // V columns c.. (rows from the panel top)
  if (w <= q.bleaf) {
    if (c > 0 && !ok_cuda(q, cudaMemset2DAsync(Vc, q.ldv * sizeof(double), 0, c * sizeof(double), w, q.st),
                          "V zero"))
      return false;
    QrLeafArgs a;
    a.A = P + c * q.lda + c;
    a.lda = q.lda;
    a.m = mp - c;
    a.b = (int32_t)w;
    a.V = Vc + c;
    a.ldv = q.ldv;
    a.tau = tau + c;
    a.part = q.part;
    a.rowb = q.rowb;
    a.bar = q.bar;
    if (!ok_cuda(q, cudaMemsetAsync(q.bar, 0, sizeof(unsigned), q.st), "barrier reset")) return false;
    // fewest CTAs that hold the leaf in shared memory, but about qr_leaf_rows() rows each:
    // fewer CTAs make the per-column grid barrier and partial-sum reduction cheaper
    const int64_t slab_rows = (int64_t)kQrSlab / (w * (int64_t)sizeof(double));
    int64_t g = std::max<int64_t>((a.m + qr_leaf_rows() - 1) / qr_leaf_rows(),
                                  (a.m + slab_rows - 1) / slab_rows);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(q.grid, g));
    a.rc = (a.m + grid - 1) / grid;
    const size_t smem = (size_t)w * a.rc * sizeof(double);
    void *args[] = {&a};
    if (!ok_cuda(q, cudaLaunchCooperativeKernel((const void *)qr_leaf_kernel, dim3(grid), dim3(kQrNT),
                                                args, smem, q.st),
                 "qr_leaf_kernel"))
      return false;
    // T leaf = larft(V_leaf^T V_leaf, tau)
    if (!ok_blas(q, cublasDgemm(q.h, CUBLAS_OP_T, CUBLAS_OP_N, (int)w, (int)w, (int)(mp - c), &one,
                                Vc + c, (int)q.ldv, Vc + c, (int)q.ldv, &zero, q.S, (int)w),
                 "leaf V^T V"))
      return false;
    qr_larft_kernel<<<1, kQrB, 0, q.st>>>(q.S, (int)w, tau + c, q.T + c * q.ldt + c, q.ldt);
    return ok_cuda(q, cudaGetLastError(), "qr_larft_kernel");
  }
  const int64_t B = q.bleaf;
  int64_t w1 = ((w / 2 + B - 1) / B) * B;
  if (w1 >= w) w1 = w - B;
  const int64_t w2 = w - w1;
  if (!rec_panel(q, P, mp, c, w1, tau)) return false;
  // right half rows [c, mp): C -= V1 T1^T V1^T C
  double *C = P + (c + w1) * q.lda + c;
  const double *V1 = Vc + c;  // rows [c, mp) of columns c..c+w1
  const double *T1 = q.T + c * q.ldt + c;
  const int k1 = (int)(mp - c);
  if (!ok_blas(q, cublasDgemm(q.h, CUBLAS_OP_T, CUBLAS_OP_N, (int)w1, (int)w2, k1, &one, V1, (int)q.ldv,
                              C, (int)q.lda, &zero, q.W, (int)w1), "panel V1^T C") ||
      !ok_blas(q, cublasDtrmm(q.h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T,
                              CUBLAS_DIAG_NON_UNIT, (int)w1, (int)w2, &one, T1, (int)q.ldt, q.W,
                              (int)w1, q.W, (int)w1), "panel T1^T W") ||
      !ok_blas(q, cublasDgemm(q.h, CUBLAS_OP_N, CUBLAS_OP_N, k1, (int)w2, (int)w1, &mone, V1, (int)q.ldv,
                              q.W, (int)w1, &one, C, (int)q.lda), "panel C -= V1 W"))
    return false;
  if (!rec_panel(q, P, mp, c + w1, w2, tau)) return false;
  // T12 = -T1 (V1^T V2) T2 over rows [c + w1, mp) (V2 is zero above its diagonal)
  double *T12 = q.T + (c + w1) * q.ldt + c;
  const double *T2 = q.T + (c + w1) * q.ldt + (c + w1);
  const int k2 = (int)(mp - c - w1);
  return ok_blas(q, cublasDgemm(q.h, CUBLAS_OP_T, CUBLAS_OP_N, (int)w1, (int)w2, k2, &one,
                                Vc + c + w1, (int)q.ldv, q.V + (c + w1) * q.ldv + c + w1, (int)q.ldv,
                                &zero, T12, (int)q.ldt), "T12 gemm") &&
         ok_blas(q, cublasDtrmm(q.h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                                CUBLAS_DIAG_NON_UNIT, (int)w1, (int)w2, &mone, T1, (int)q.ldt, T12,
                                (int)q.ldt, T12, (int)q.ldt), "T12 left trmm") &&
         ok_blas(q, cublasDtrmm(q.h, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                                CUBLAS_DIAG_NON_UNIT, (int)w1, (int)w2, &one, T2, (int)q.ldt, T12,
                                (int)q.ldt, T12, (int)q.ldt), "T12 right trmm");
}

}  // namespace

int64_t qr_leaf_rows() {
  static int64_t r = 0;
  if (!r) {
    r = 256;
    if (const char *s = getenv("FLS_QR_LEAF_ROWS")) {  // tuning sweeps only
      const int64_t v = atoll(s);
      if (v >= 32) r = v;
    }
  }
  return r;
}

int64_t qr_blocked_max_rows() {
  static int64_t mx = 0;
  if (!mx) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    mx = (int64_t)std::max(1, std::min(sms, kQrMaxGrid)) * (kQrSlab / (kQrMinLeaf * sizeof(double)));
  }
  return mx;
}

// panel width for an n-column block: 128 up to 4,096 columns, 256 above (FLS_QR_NB sweep,
// profiles/r01_qr_nb_sweep.jsonl: C2 15.2 -> 14.2 ms and C3 57.5 -> 56.2 ms at 128; C4 best
// at 256, C5 flat 256-512)
int qr_panel_width(int64_t n) {
  static int forced = -1;
  if (forced < 0) {
    forced = 0;
    if (const char *s = getenv("FLS_QR_NB")) {  // tuning sweeps only
      const int v = atoi(s);
      if (v >= kQrB) forced = (v / kQrB) * kQrB;
    }
  }
  if (forced) return forced;
  return n <= 4096 ? 128 : 256;
}

static int qr_grid() {
  static int g = 0;
  if (!g) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g = std::max(1, std::min(sms, kQrMaxGrid));
  }
  return g;
}

// workspace (doubles) qr_blocked needs for an m x n block: panel V, T, W, leaf S, partials
size_t qr_blocked_ws(int64_t m, int64_t n) {
  const int64_t nb = qr_panel_width(n);
  const int64_t ldv = (m + 3) / 4 * 4;
  return (size_t)ldv * nb + (size_t)nb * nb + (size_t)nb * (n > nb ? n : nb) + (size_t)kQrB * kQrB +
         (size_t)2 * qr_grid() * (kQrB + 1) + 2 * (kQrB + 1) + 1;  // + barrier counter
}

// Row permutation of a stack of P factors into the order qr_blocked's grouped mode expects:
// block 0 first, then row group i = row i of blocks 1..P-1 followed by ridge row i (sqrt_mu at
// column i), zeros where a source is absent.  Factor r's row i, column c is S[r*bs + c*cs + i]:
// bs = kb, cs = lds for the block-row layout of fls_solve_stacked; bs = kb * n, cs = kb for the
// block-contiguous layout the multi-rank TSQR gathers into (one contiguous factor per rank).
__global__ void stack_permute_kernel(const double *S, int64_t bs, int64_t cs, int32_t P, int64_t kb,
                                     int64_t F, double sqrt_mu, int64_t gq, int64_t m_total,
                                     int64_t n, double *M, int64_t ldm) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= m_total * n) return;
  const int64_t c = idx / m_total, t = idx % m_total;
  double v = 0.0;
  if (t < kb) {
    v = S[c * cs + t];
  } else {
    const int64_t u = t - kb, i = u / gq, g = u % gq;
    if (g < P - 1) {
      if (i < kb) v = S[(g + 1) * bs + c * cs + i];
    } else if (c == i && i < F) {
      v = sqrt_mu;
    }
  }
  M[c * ldm + t] = v;
}

cudaError_t launch_stack_permute(const double *S, int64_t bs, int64_t cs, int32_t P, int64_t kb,
                                 int64_t F, double sqrt_mu, int64_t gq, int64_t m_total, int64_t n,
                                 double *M, int64_t ldm, cudaStream_t st) {
  const int64_t tot = m_total * n;
  if (tot == 0) return cudaSuccess;
  stack_permute_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(S, bs, cs, P, kb, F, sqrt_mu,
                                                                       gq, m_total, n, M, ldm);
  return cudaGetLastError();
}

// A (m x n, lda) -> R / V / tau in place, ws = qr_blocked_ws(m, n) doubles (caller-owned, so
// repeated solves do not allocate).  Returns 0 or a message (static string).
// grp_size > 0: A is a row-permuted stack of triangular factors (fls_solve_stacked): rows
// [0, grp_base) are one upper-trapezoidal block and row group i (rows grp_base + i grp_size ..
// + grp_size - 1) is zero left of column i -- so the rows of panel [j, j+w) that can be nonzero
// end at grp_base + grp_size (j + w), and the panel and its trailing update stop there.
const char *qr_blocked(cublasHandle_t h, cudaStream_t st, double *A, int64_t m, int64_t n,
                       int64_t lda, double *tau, double *ws, cudaError_t *cerr,
                       cublasStatus_t *berr, int64_t grp_base, int64_t grp_size) {
  *cerr = cudaSuccess;
  *berr = CUBLAS_STATUS_SUCCESS;
  const int64_t k = m < n ? m : n;
  if (k <= 0) return nullptr;
  const int64_t nb = qr_panel_width(n);
  QrCtx q;
  q.h = h;
  q.st = st;
  q.A = A;
  q.lda = lda;
  q.ldv = (m + 3) / 4 * 4;
  q.ldt = nb;
  q.grid = qr_grid();
  if (m > qr_blocked_max_rows()) {
    *cerr = cudaErrorInvalidValue;
    return "rows exceed the leaf slab capacity";
  }
  {  // the shared-memory opt-in is a per-device function attribute
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr[dev]) {
      cudaError_t e = cudaFuncSetAttribute(qr_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kQrSlab);
      if (e != cudaSuccess) {
        *cerr = e;
        return "qr_leaf_kernel shared-memory attribute";
      }
      if (dev >= 0 && dev < 64) attr[dev] = true;
    }
  }
  const size_t nV = (size_t)q.ldv * nb, nT = (size_t)nb * nb, nW = (size_t)nb * (n > nb ? n : nb);
  const size_t nS = (size_t)kQrB * kQrB, nP = (size_t)2 * q.grid * (kQrB + 1);
  q.V = ws;
  q.T = q.V + nV;
  q.W = q.T + nT;
  q.S = q.W + nW;
  q.part = q.S + nS;
  q.rowb = q.part + nP;
  q.bar = reinterpret_cast<unsigned *>(q.rowb + 2 * (kQrB + 1));
  const double one = 1.0, zero = 0.0, mone = -1.0;
  bool good = ok_blas(q, cublasSetStream(h, st), "cublasSetStream");
  for (int64_t j = 0; good && j < k; j += nb) {
    const int64_t w = nb < k - j ? nb : k - j;
    int64_t mp = m - j;
    if (grp_size > 0) mp = std::min<int64_t>(mp, grp_base + grp_size * (j + w) - j);
    double *P = A + j * lda + j;
    const int64_t rc = (mp + q.grid - 1) / q.grid;
    q.bleaf = (int)std::min<int64_t>(kQrB, (int64_t)kQrSlab / (rc * (int64_t)sizeof(double)));
    good = rec_panel(q, P, mp, 0, w, tau + j);
    const int64_t nt = n - j - w;
    if (good && nt > 0) {  // trailing update C -= V T^T V^T C
      double *C = P + w * lda;
      good = ok_blas(q, cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)w, (int)nt, (int)mp, &one, q.V,
                                    (int)q.ldv, C, (int)lda, &zero, q.W, (int)w), "trailing V^T C") &&
             ok_blas(q, cublasDtrmm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T,
                                    CUBLAS_DIAG_NON_UNIT, (int)w, (int)nt, &one, q.T, (int)q.ldt, q.W,
                                    (int)w, q.W, (int)w), "trailing T^T W") &&
             ok_blas(q, cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, (int)mp, (int)nt, (int)w, &mone, q.V,
                                    (int)q.ldv, q.W, (int)w, &one, C, (int)lda), "trailing C -= V W");
    }
  }
  *cerr = q.cerr;
  *berr = q.berr;
  return good ? nullptr : q.fail;
}

}  // namespace fls
