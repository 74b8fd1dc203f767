// fls_ctx.h -- host-only internals shared by the C-ABI translation units (fls_api.cu,
// fls_comm.cu): the ctx object, error helpers and the solve building blocks.
#pragma once
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <nvtx3/nvToolsExt.h>  // header-only; ranges cost nothing unless a tool is attached

#include <vector>

#include "fls_internal.h"

namespace fls {
struct Comm;  // fls_comm.cu: the communicator attached by fls_comm_init / fls_comm_init_host
}

struct fls_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  unsigned *d_err = nullptr;          // async flags: bit 0 non-finite input, bit 1 phase range
  double *d_scratch = nullptr;        // small device scratch (min diag, frob partials)
  double *ws = nullptr;               // per-feature prefactor records
  size_t ws_bytes = 0;
  double *qws = nullptr;              // blocked-QR workspace (grow-only; + tau scratch)
  size_t qws_bytes = 0;
  double *gws = nullptr;              // bandwidth-gradient partials (grow-only)
  size_t gws_bytes = 0;
  double *sws = nullptr;              // permuted stack of the TSQR root solve (grow-only)
  size_t sws_bytes = 0;
  cusolverDnHandle_t solver = nullptr;
  cublasHandle_t blas = nullptr;
  // optional per-launch timing of the assembly kernels (fls_ctx_timing)
  bool timing = false;
  std::vector<cudaEvent_t> ev;  // pairs (start, stop)
  size_t ev_used = 0;
  // host-buffer path (fls_assemble_host): copy stream, events, device staging
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t hev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t switch_ev = nullptr;  // fls_ctx_set_stream ordering
  double *hin = nullptr, *hout = nullptr;
  size_t hin_bytes = 0, hout_bytes = 0;
  fls::Comm *comm = nullptr;        // multi-rank solve (fls_comm_init*), owned
};

namespace fls {

fls_status fail(fls_status s, const char *fmt, ...);
fls_status cuda_fail(cudaError_t e, const char *where);
fls_status check_ctx(fls_ctx *ctx);

#define FLS_CUDA(call)                                         \
  do {                                                         \
    cudaError_t e_ = (call);                                   \
    if (e_ != cudaSuccess) return ::fls::cuda_fail(e_, #call); \
  } while (0)

// NVTX range for the duration of a libfls call (nsys / ncu --nvtx timelines)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// solve building blocks (fls_api.cu)
fls_status ensure_handles(fls_ctx *ctx);
fls_status geqrf_inplace(fls_ctx *ctx, double *M, int64_t m, int64_t lda, int64_t n,
                         double *tau_out = nullptr, int64_t grp_base = 0, int64_t grp_size = 0);
// sum of squares of an m x n column-major block, fixed-order (deterministic); host result
fls_status frob2_host(fls_ctx *ctx, const double *A, int64_t m, int64_t lda, int64_t n, double *out);
// single-rank least squares of [A | b] (m x (F+1)) with sqrt_mu I rows appended in place
fls_status solve_local(fls_ctx *ctx, double *Ab, int64_t n_rows, int64_t lda, int64_t F,
                       double sqrt_mu, double *beta, double *resid_norm);
// TSQR root step on a stack of P factors: factor r's row i, column c at S[r*bs + c*cs + i]
// (kb rows each); ridge rows appended when sqrt_mu > 0.  S is not modified.
fls_status solve_stacked_impl(fls_ctx *ctx, const double *S, int32_t P, int64_t kb, int64_t bs,
                              int64_t cs, int64_t F, double sqrt_mu, double *beta,
                              double *resid_norm);
// multi-rank solve when a communicator is attached (fls_comm.cu); *handled = false when the
// ctx has no communicator (or one rank and no forced TSQR) so the caller solves locally
// pending: this rank's status before the call (e.g. a pending FLS_ENONFINITE), agreed with the
// other ranks so that a local failure is returned everywhere instead of leaving peers waiting
fls_status comm_solve(fls_ctx *ctx, double *Ab, int64_t n_local, int64_t lda, int64_t F,
                      double ridge_rel, double sqrt_mu_abs, double *beta, double *resid_norm,
                      bool *handled, fls_status pending = FLS_OK);
void comm_destroy(fls_ctx *ctx);

}  // namespace fls
