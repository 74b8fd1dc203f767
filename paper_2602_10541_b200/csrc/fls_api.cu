// fls_api.cu -- the C ABI of libfls (include/fls.h): ctx, argument validation, mode selection,
// launches, and the cuSOLVER least-squares solve.
//
// Product code.  Paper = PAPER.md (arxiv 2602.10541), cited P:L<line>.
#include <cublas_v2.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "fls_ctx.h"
#include "fls_internal.h"

using namespace fls;


namespace {

thread_local std::string g_err;

fls_status ensure_ws(fls_ctx *ctx, size_t bytes) {
  if (bytes <= ctx->ws_bytes) return FLS_OK;
  if (ctx->ws) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->ws);
    ctx->ws = nullptr;
    ctx->ws_bytes = 0;
  }
  size_t nb = bytes < (1u << 20) ? (1u << 20) : bytes;
  if (cudaMalloc(&ctx->ws, nb) != cudaSuccess) {
    cudaGetLastError();
    return fail(FLS_ENOMEM, "workspace allocation of %zu bytes failed", nb);
  }
  ctx->ws_bytes = nb;
  return FLS_OK;
}

// host-side analysis of one operator: groups, parity, mode
struct OpPlan {
  int G = 0;
  int pmode = PM_SIN;
  int kmode = KM_SIN;
  int gfield[FLS_MAX_FIELDS] = {0, 0, 0, 0};
  int n_terms = 0;
  TermDev terms[FLS_MAX_TERMS];
};

fls_status plan_operator(const fls_operator *op, int32_t dim, int32_t n_fields, bool allow_fields,
                         OpPlan &pl, const char *what) {
  if (!op) return fail(FLS_EINVAL, "%s: operator is NULL", what);
  if (op->dim != dim)
    return fail(FLS_EINVAL, "%s: operator dim %d != basis dim %d", what, op->dim, dim);
  if (op->n_terms < 1 || op->n_terms > FLS_MAX_TERMS)
    return fail(FLS_EINVAL, "%s: n_terms %d not in 1..%d", what, op->n_terms, FLS_MAX_TERMS);
  if (!op->terms) return fail(FLS_EINVAL, "%s: terms is NULL", what);
  bool any_s = false, any_c = false;
  std::memset(pl.terms, 0, sizeof pl.terms);
  pl.n_terms = op->n_terms;
  pl.G = 0;
  for (int t = 0; t < op->n_terms; ++t) {
    const fls_term &T = op->terms[t];
    int order = 0;
    for (int k = 0; k < FLS_MAX_DIM; ++k) {
      if (T.alpha[k] < 0 || T.alpha[k] > 64)
        return fail(FLS_EINVAL, "%s: term %d alpha[%d] = %d out of range", what, t, k, T.alpha[k]);
      if (k >= dim && T.alpha[k] != 0)
        return fail(FLS_EINVAL, "%s: term %d alpha[%d] set beyond dim %d", what, t, k, dim);
      order += T.alpha[k];
      pl.terms[t].alpha[k] = (int8_t)T.alpha[k];
    }
    if (!std::isfinite(T.coef)) return fail(FLS_EINVAL, "%s: term %d coef not finite", what, t);
    pl.terms[t].coef = T.coef;
    int grp = 0;
    if (T.field >= 0) {
      if (!allow_fields) return fail(FLS_EINVAL, "%s: coefficient fields not allowed here", what);
      if (T.field >= n_fields)
        return fail(FLS_EINVAL, "%s: term %d field %d >= n_fields %d", what, t, T.field, n_fields);
      int g = 0;
      while (g < pl.G && pl.gfield[g] != T.field) ++g;
      if (g == pl.G) pl.gfield[pl.G++] = T.field;
      grp = g + 1;
    } else if (T.field != -1) {
      return fail(FLS_EINVAL, "%s: term %d field %d (use -1 for constant)", what, t, T.field);
    }
    pl.terms[t].group = (int8_t)grp;
    // the monomial's factors in the order the fold multiplies them (axis 0 first, alpha_0
    // times, ...): the device loop then runs |alpha| dependent multiplies and nothing else
    if (order <= kMaxFac) {
      int n = 0;
      for (int k = 0; k < dim; ++k)
        for (int e = 0; e < T.alpha[k]; ++e) pl.terms[t].fac[n++] = (int8_t)k;
      pl.terms[t].nfac = (int8_t)order;
    } else {
      pl.terms[t].nfac = -1;
    }
    if (order & 1) any_c = true; else any_s = true;
  }
  if (!any_c) { pl.pmode = PM_SIN; pl.kmode = KM_SIN; }
  else if (!any_s) { pl.pmode = PM_COSSHIFT; pl.kmode = KM_SIN; }
  else if (pl.G == 0) { pl.pmode = PM_FOLD; pl.kmode = KM_SIN; }
  else { pl.pmode = PM_SINCOS; pl.kmode = KM_SINCOS; }
  return FLS_OK;
}

}  // namespace

namespace fls {

fls_status fail(fls_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

fls_status cuda_fail(cudaError_t e, const char *where) {
  // reset the runtime's (non-sticky) last error, so that a failed call here is not reported
  // again by the next launch's cudaGetLastError() in this thread
  cudaGetLastError();
  return fail(FLS_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

fls_status check_ctx(fls_ctx *ctx) {
  if (!ctx) return fail(FLS_EINVAL, "ctx is NULL");
  return FLS_OK;
}

}  // namespace fls

extern "C" {

const char *fls_last_error(void) { return g_err.c_str(); }

const char *fls_status_string(fls_status s) {
  switch (s) {
    case FLS_OK: return "FLS_OK";
    case FLS_EINVAL: return "FLS_EINVAL";
    case FLS_ENOMEM: return "FLS_ENOMEM";
    case FLS_ECUDA: return "FLS_ECUDA";
    case FLS_ECUSOLVER: return "FLS_ECUSOLVER";
    case FLS_ENCCL: return "FLS_ENCCL";
    case FLS_ENONFINITE: return "FLS_ENONFINITE";
    case FLS_ERANK: return "FLS_ERANK";
    case FLS_EUNSUPPORTED: return "FLS_EUNSUPPORTED";
  }
  return "FLS_?";
}

int fls_api_version(void) { return FLS_API_VERSION; }

fls_status fls_ctx_create(int device, void *cuda_stream, fls_ctx **out) {
  if (!out) return fail(FLS_EINVAL, "out is NULL");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= n) return fail(FLS_EINVAL, "device %d not in [0, %d)", device, n);
  DeviceGuard g(device);
  fls_ctx *c = new fls_ctx();
  c->device = device;
  c->stream = (cudaStream_t)cuda_stream;
  if ((e = cudaMalloc(&c->d_err, sizeof(unsigned))) != cudaSuccess ||
      (e = cudaMemset(c->d_err, 0, sizeof(unsigned))) != cudaSuccess ||
      (e = cudaMalloc(&c->d_scratch, 1024 * sizeof(double))) != cudaSuccess) {
    fls_ctx_destroy(c);
    return cuda_fail(e, "fls_ctx_create");
  }
  *out = c;
  return FLS_OK;
}

fls_status fls_ctx_destroy(fls_ctx *ctx) {
  if (!ctx) return FLS_OK;
  DeviceGuard g(ctx->device);
  cudaStreamSynchronize(ctx->stream);  // kernels may still read the workspace
  comm_destroy(ctx);
  if (ctx->solver) cusolverDnDestroy(ctx->solver);
  if (ctx->blas) cublasDestroy(ctx->blas);
  for (cudaEvent_t ev : ctx->ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : ctx->hev)
    if (ev) cudaEventDestroy(ev);
  if (ctx->switch_ev) cudaEventDestroy(ctx->switch_ev);
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  cudaFree(ctx->hin);
  cudaFree(ctx->hout);
  cudaFree(ctx->ws);
  cudaFree(ctx->qws);
  cudaFree(ctx->gws);
  cudaFree(ctx->sws);
  cudaFree(ctx->d_err);
  cudaFree(ctx->d_scratch);
  delete ctx;
  return FLS_OK;
}

fls_status fls_ctx_set_stream(fls_ctx *ctx, void *cuda_stream) {
  if (fls_status s = check_ctx(ctx)) return s;
  const cudaStream_t next = (cudaStream_t)cuda_stream;
  if (next != ctx->stream) {  // the new stream waits for the old one's pending work
    DeviceGuard g(ctx->device);
    if (!ctx->switch_ev) FLS_CUDA(cudaEventCreateWithFlags(&ctx->switch_ev, cudaEventDisableTiming));
    FLS_CUDA(cudaEventRecord(ctx->switch_ev, ctx->stream));
    FLS_CUDA(cudaStreamWaitEvent(next, ctx->switch_ev, 0));
  }
  ctx->stream = next;
  if (ctx->solver) cusolverDnSetStream(ctx->solver, ctx->stream);
  if (ctx->blas) cublasSetStream(ctx->blas, ctx->stream);
  return FLS_OK;
}

fls_status fls_ctx_timing(fls_ctx *ctx, int32_t enable) {
  if (fls_status s = check_ctx(ctx)) return s;
  ctx->timing = enable != 0;
  ctx->ev_used = 0;
  return FLS_OK;
}

fls_status fls_ctx_timing_read(fls_ctx *ctx, double *ms_total, int64_t *n_launches) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (!ms_total || !n_launches) return fail(FLS_EINVAL, "NULL output");
  DeviceGuard g(ctx->device);
  FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  double tot = 0.0;
  for (size_t k = 0; k + 1 < ctx->ev_used; k += 2) {
    float ms = 0.f;
    FLS_CUDA(cudaEventElapsedTime(&ms, ctx->ev[k], ctx->ev[k + 1]));
    tot += ms;
  }
  *ms_total = tot;
  *n_launches = (int64_t)(ctx->ev_used / 2);
  ctx->ev_used = 0;
  return FLS_OK;
}

fls_status fls_sync(fls_ctx *ctx) {
  if (fls_status s = check_ctx(ctx)) return s;
  DeviceGuard g(ctx->device);
  FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  unsigned h = 0;
  FLS_CUDA(cudaMemcpyAsync(&h, ctx->d_err, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (h) {
    FLS_CUDA(cudaMemsetAsync(ctx->d_err, 0, sizeof(unsigned), ctx->stream));
    FLS_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h & 1u)
      return fail(FLS_ENONFINITE, "non-finite value in an input (W, b, X, values or fields)");
    return fail(FLS_EUNSUPPORTED, "a phase |W_j . x_i + b_j| exceeds FLS_MAX_PHASE = %g (the "
                "half-turn range reduction loses accuracy as ulp(|z|); entries unspecified)",
                (double)FLS_MAX_PHASE);
  }
  return FLS_OK;
}

// ---------------------------------------------------------------------------------------------
fls_status fls_features(fls_ctx *ctx, int32_t dim, int64_t n_features, double sigma,
                        uint64_t seed, double *W, double *b) {
  return fls_features_blocks(ctx, dim, 1, &n_features, &sigma, seed, W, b);
}

fls_status fls_features_blocks(fls_ctx *ctx, int32_t dim, int32_t n_blocks,
                               const int64_t *block_features, const double *sigmas, uint64_t seed,
                               double *W, double *b) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (dim < 1 || dim > FLS_MAX_DIM) return fail(FLS_EINVAL, "dim %d not in 1..%d", dim, FLS_MAX_DIM);
  if (n_blocks < 1 || n_blocks > FLS_MAX_FEAT_BLOCKS)
    return fail(FLS_EINVAL, "n_blocks %d not in 1..%d", n_blocks, FLS_MAX_FEAT_BLOCKS);
  if (!block_features || !sigmas) return fail(FLS_EINVAL, "block_features or sigmas is NULL");
  FeatBlocks fb;
  std::memset(&fb, 0, sizeof fb);
  fb.n = n_blocks;
  int64_t F = 0;
  for (int q = 0; q < n_blocks; ++q) {
    if (block_features[q] < 1)
      return fail(FLS_EINVAL, "block %d: n_features %lld < 1", q, (long long)block_features[q]);
    if (!(sigmas[q] > 0.0) || !std::isfinite(sigmas[q]))
      return fail(FLS_EINVAL, "block %d: sigma must be > 0 and finite", q);
    F += block_features[q];
    fb.ends[q] = F;
    fb.sigma[q] = sigmas[q];
  }
  if (!W || !b) return fail(FLS_EINVAL, "W or b is NULL");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_features(dim, F, fb, seed, W, b, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "features_kernel");
  return FLS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// assembly: validation shared by the device and host entry points
namespace {

struct AsmPlan {
  int32_t n_blocks = 0;
  int64_t total = 0;
  OpPlan plans[64];
};

fls_status validate_assemble(int32_t dim, int64_t n_features, const double *W, const double *b,
                             const fls_block *blocks, int32_t n_blocks, int64_t row_begin,
                             int64_t row_end, const double *A, int64_t lda, int32_t layout,
                             AsmPlan &ap) {
  if (dim < 1 || dim > FLS_MAX_DIM) return fail(FLS_EINVAL, "dim %d not in 1..%d", dim, FLS_MAX_DIM);
  if (n_features < 1) return fail(FLS_EINVAL, "n_features %lld < 1", (long long)n_features);
  if (!W || !b) return fail(FLS_EINVAL, "W or b is NULL");
  if (!blocks || n_blocks < 1) return fail(FLS_EINVAL, "need n_blocks >= 1 block descriptors");
  if (n_blocks > 64) return fail(FLS_EUNSUPPORTED, "more than 64 blocks");
  if (layout != FLS_COL_MAJOR && layout != FLS_ROW_MAJOR)
    return fail(FLS_EINVAL, "layout %d unknown", layout);
  ap.n_blocks = n_blocks;
  ap.total = 0;
  for (int q = 0; q < n_blocks; ++q) {
    const fls_block &B = blocks[q];
    if (B.n_points < 0) return fail(FLS_EINVAL, "block %d: n_points < 0", q);
    if (B.n_fields < 0 || B.n_fields > FLS_MAX_FIELDS)
      return fail(FLS_EINVAL, "block %d: n_fields %d not in 0..%d", q, B.n_fields, FLS_MAX_FIELDS);
    if (B.n_points > 0 && !B.X) return fail(FLS_EINVAL, "block %d: X is NULL", q);
    if (B.n_points > 0 && B.n_fields > 0 && !B.coef_fields)
      return fail(FLS_EINVAL, "block %d: coef_fields is NULL with n_fields %d", q, B.n_fields);
    if (!std::isfinite(B.weight)) return fail(FLS_EINVAL, "block %d: weight not finite", q);
    char what[32];
    snprintf(what, sizeof what, "block %d", q);
    if (fls_status s = plan_operator(B.op, dim, B.n_fields, true, ap.plans[q], what)) return s;
    ap.total += B.n_points;
  }
  if (row_begin < 0 || row_end < row_begin || row_end > ap.total)
    return fail(FLS_EINVAL, "row range [%lld, %lld) not within [0, %lld]", (long long)row_begin,
                (long long)row_end, (long long)ap.total);
  const int64_t n_local = row_end - row_begin;
  if (n_local == 0) return FLS_OK;
  if (!A) return fail(FLS_EINVAL, "A is NULL");
  if (layout == FLS_COL_MAJOR && lda < n_local)
    return fail(FLS_EINVAL, "lda %lld < local rows %lld", (long long)lda, (long long)n_local);
  if (layout == FLS_ROW_MAJOR && lda < n_features)
    return fail(FLS_EINVAL, "lda %lld < n_features %lld", (long long)lda, (long long)n_features);
  return FLS_OK;
}

constexpr int kSmax = pf_stride(FLS_MAX_DIM, FLS_MAX_FIELDS, KM_SINCOS);

// fold arguments of block q (its record array at ctx->ws + q F kSmax)
void make_pref(fls_ctx *ctx, PrefArgs &pa, const OpPlan &pl, const fls_block &B, int q,
               const double *W, const double *b, int32_t dim, int64_t F, double s_norm) {
  std::memset(&pa, 0, sizeof pa);
  pa.W = W;
  pa.b = b;
  pa.F = F;
  pa.D = dim;
  pa.n_terms = pl.n_terms;
  pa.G = pl.G;
  pa.pmode = pl.pmode;
  pa.S = pf_stride(dim, pl.G, pl.kmode);
  pa.scale = s_norm * B.weight;
  pa.pf = ctx->ws + (size_t)q * F * kSmax;
  pa.err = ctx->d_err;
  std::memcpy(pa.terms, pl.terms, sizeof pl.terms);
}

// a2: prefactor records of every block that has rows in [row_begin, row_end), up to
// kMaxBatch blocks per launch
fls_status launch_prefactors(fls_ctx *ctx, const AsmPlan &ap, const double *W, const double *b,
                             int32_t dim, int64_t F, int32_t normalize, const fls_block *blocks,
                             int64_t row_begin, int64_t row_end, cudaStream_t st) {
  if (fls_status s = ensure_ws(ctx, (size_t)ap.n_blocks * F * kSmax * sizeof(double))) return s;
  const double s_norm = normalize ? 1.0 / std::sqrt((double)F) : 1.0;
  static thread_local PrefBatch pb;
  pb.n = 0;
  int64_t g0 = 0;
  for (int q = 0; q < ap.n_blocks; ++q) {
    const fls_block &B = blocks[q];
    const int64_t lo = std::max(g0, row_begin), hi = std::min(g0 + B.n_points, row_end);
    g0 += B.n_points;
    if (hi <= lo) continue;
    make_pref(ctx, pb.blk[pb.n++], ap.plans[q], B, q, W, b, dim, F, s_norm);
    if (pb.n == kMaxBatch) {
      cudaError_t e = launch_prefactor_batch(pb, F, st);
      if (e != cudaSuccess) return cuda_fail(e, "prefactor_batch_kernel");
      pb.n = 0;
    }
  }
  if (pb.n > 0) {
    cudaError_t e = launch_prefactor_batch(pb, F, st);
    if (e != cudaSuccess) return cuda_fail(e, "prefactor_batch_kernel");
  }
  return FLS_OK;
}

// largest assembly launch that gets PDL: C3 (1e8 entries) 147.8 -> 144.9 us per graph step,
// unfused C2 27.5 -> 24.6 us; none for C4 / C5
constexpr int64_t kPdlMaxEntries = int64_t(1) << 28;

// a3-a8: assembly launches for global rows [row_begin, row_end) into local rows of A / rhs.
// blocks[q]'s X / fields / values pointers refer to point index pt_base[q] (0 for the caller's
// own arrays; the slice start for staged copies).  Column-major: consecutive blocks that share
// the kernel variant (same field-group count and sin / sin+cos family) go into one launch.
fls_status assemble_range(fls_ctx *ctx, const AsmPlan &ap, int32_t dim, int64_t F,
                          const fls_block *blocks, const int64_t *pt_base, int64_t row_begin,
                          int64_t row_end, double *A, int64_t lda, int32_t layout, double *rhs,
                          cudaStream_t st, bool pdl, const FusedBatch *fz_proto = nullptr,
                          double s_norm = 1.0) {
  // vector stores need every column segment aligned: 16 B (row pairs) or 32 B (kQuad rows);
  // the row-major kernel always stores feature pairs (16 B)
  const bool quad = kQuad && layout == FLS_COL_MAJOR;
  const bool vec = quad ? ((reinterpret_cast<uintptr_t>(A) & 31) == 0) && (lda % 4 == 0)
                        : ((reinterpret_cast<uintptr_t>(A) & 15) == 0) && (lda % 2 == 0);
  AsmArgs batch[kMaxBatch];
  int bq[kMaxBatch];  // block index of each batch entry
  int nb = 0, bG = 0, bK = 0;
  bool first_launch = true;
  static thread_local FusedBatch fz;
  auto flush = [&]() -> fls_status {
    if (nb == 0) return FLS_OK;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->timing) {
      if (ctx->ev_used + 2 > ctx->ev.size()) {
        for (int k = 0; k < 2; ++k) {
          cudaEvent_t ev;
          FLS_CUDA(cudaEventCreate(&ev));
          ctx->ev.push_back(ev);
        }
      }
      e0 = ctx->ev[ctx->ev_used++];
      e1 = ctx->ev[ctx->ev_used++];
      FLS_CUDA(cudaEventRecord(e0, st));
    }
    cudaError_t e = cudaSuccess;
    if (layout == FLS_COL_MAJOR) {
      // PDL only between kernels (a timing event recorded in between would sit in the way),
      // and only for launches short enough that the saved launch latency shows: on C5
      // (1.7e10 entries) it cost 0.6% (early-dispatched CTAs skew its two long waves)
      int64_t entries = 0;
      for (int i = 0; i < nb; ++i) entries += (batch[i].lr1 - batch[i].lr0) * F;
      if (fz_proto) {  // single launch: the CTAs draw and fold their features' records
        fz = *fz_proto;
        fz.write_wb = first_launch ? 1 : 0;
        for (int i = 0; i < nb; ++i)
          make_pref(ctx, fz.pre[i], ap.plans[bq[i]], blocks[bq[i]], bq[i], fz.W, fz.b, dim, F, s_norm);
        // PDL behind whatever precedes: the first chunk's draws and folds overlap it (the
        // kernel touches no global memory before its griddepcontrol.wait)
        e = launch_assemble_cm_fused(dim, bG, batch, nb, fz, st,
                                     pdl && !ctx->timing && entries <= kPdlMaxEntries);
      } else {
        e = launch_assemble_cm(dim, bG, bK, batch, nb, st,
                               pdl && !ctx->timing && entries <= kPdlMaxEntries);
      }
      first_launch = false;
    } else {
      for (int i = 0; i < nb && e == cudaSuccess; ++i) e = launch_assemble_rm(dim, bG, bK, batch[i], st);
    }
    if (e != cudaSuccess) return cuda_fail(e, "assemble kernel");
    if (ctx->timing) FLS_CUDA(cudaEventRecord(e1, st));
    nb = 0;
    return FLS_OK;
  };
  int64_t g0 = 0;  // first global row of block q
  for (int q = 0; q < ap.n_blocks; ++q) {
    const fls_block &B = blocks[q];
    const int64_t lo = std::max(g0, row_begin), hi = std::min(g0 + B.n_points, row_end);
    const int64_t blk_start = g0;
    g0 += B.n_points;
    if (hi <= lo) continue;
    const OpPlan &pl = ap.plans[q];
    if (nb > 0 && (pl.G != bG || pl.kmode != bK || nb == kMaxBatch))
      if (fls_status s = flush()) return s;
    bG = pl.G;
    bK = pl.kmode;
    bq[nb] = q;
    AsmArgs &aa = batch[nb++];
    std::memset(&aa, 0, sizeof aa);
    aa.pf = ctx->ws + (size_t)q * F * kSmax;
    aa.F = F;
    aa.X = B.X;
    aa.fields = B.coef_fields;
    aa.values = B.values;
    aa.weight = B.weight;
    aa.pt0 = (lo - blk_start) - (pt_base ? pt_base[q] : 0);
    aa.lr0 = lo - row_begin;
    aa.lr1 = hi - row_begin;
    aa.A = A;
    aa.lda = lda;
    aa.rhs = rhs;
    aa.err = ctx->d_err;
    aa.nf = B.n_fields;
    aa.vec = vec ? 1 : 0;
    for (int i = 0; i < FLS_MAX_FIELDS; ++i) aa.gfield[i] = pl.gfield[i];
  }
  return flush();
}

// largest fls_features_assemble call (local entries) that runs as ONE fused launch; read per
// call so tuning sweeps / tests can switch it (FLS_FUSE_MAX_ENTRIES=0 turns the fusion off)
int64_t fuse_max_entries() {
  const char *v = getenv("FLS_FUSE_MAX_ENTRIES");
  // default 2^22: C1 (5e5 entries: 10-step-graph step 7.1 -> 6.1 us fused); C2 (9.6e6) is
  // slower fused (19.8 vs 18.4 us: each CTA's Box-Muller + fold chain sits on its critical
  // path, tools/small_step_probe.py)
  return v && *v ? (int64_t)atoll(v) : (int64_t(1) << 22);
}

// programmatic dependent launch of the assembly after its prefactor launch (FLS_PDL=0: off)
bool pdl_enabled() {
  static const bool on = [] {
    const char *v = getenv("FLS_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

fls_status ensure_dev(double *&p, size_t &cap, size_t bytes, cudaStream_t st) {
  if (bytes <= cap) return FLS_OK;
  if (p) {
    cudaStreamSynchronize(st);
    cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(FLS_ENOMEM, "staging allocation of %zu bytes failed", bytes);
  }
  cap = bytes;
  return FLS_OK;
}

}  // namespace

extern "C" {

fls_status fls_features_assemble(fls_ctx *ctx, int32_t dim, int64_t n_features, double sigma,
                                 uint64_t seed, double *W, double *b, int32_t normalize,
                                 const fls_block *blocks, int32_t n_blocks, int64_t row_begin,
                                 int64_t row_end, double *A, int64_t lda, int32_t layout,
                                 double *rhs) {
  NvtxRange nvtx_("fls_features_assemble");
  if (fls_status s = check_ctx(ctx)) return s;
  if (!(sigma > 0.0) || !std::isfinite(sigma)) return fail(FLS_EINVAL, "sigma must be > 0 and finite");
  static thread_local AsmPlan ap;
  if (fls_status s = validate_assemble(dim, n_features, W, b, blocks, n_blocks, row_begin, row_end,
                                       A, lda, layout, ap))
    return s;
  const int64_t F = n_features;
  DeviceGuard g(ctx->device);
  if (fls_status s = ensure_ws(ctx, (size_t)ap.n_blocks * F * kSmax * sizeof(double))) return s;
  FeatBlocks fb;
  std::memset(&fb, 0, sizeof fb);
  fb.n = 1;
  fb.ends[0] = F;
  fb.sigma[0] = sigma;
  // records of the blocks that have rows in range (kMaxBatch fit in the fused launch)
  static thread_local PrefBatch pb;
  pb.n = 0;
  const double s_norm = normalize ? 1.0 / std::sqrt((double)F) : 1.0;
  int64_t g0 = 0;
  bool overflow = false;
  for (int q = 0; q < ap.n_blocks; ++q) {
    const fls_block &B = blocks[q];
    const int64_t lo = std::max(g0, row_begin), hi = std::min(g0 + B.n_points, row_end);
    g0 += B.n_points;
    if (hi <= lo) continue;
    if (pb.n == kMaxBatch) {
      overflow = true;
      break;
    }
    make_pref(ctx, pb.blk[pb.n++], ap.plans[q], B, q, W, b, dim, F, s_norm);
  }
  // small problems (launch-latency bound): ONE launch -- each assembly CTA draws
  // W_j, b_j of its own features and folds their records in its prologue (bit-identical to the
  // two-launch path); needs every block in range on a fused variant, column-major
  const int64_t n_local = row_end - row_begin;
  if (layout == FLS_COL_MAJOR && n_local > 0 && n_local * F <= fuse_max_entries()) {
    bool ok = true;
    g0 = 0;
    for (int q = 0; q < ap.n_blocks; ++q) {
      const int64_t lo = std::max(g0, row_begin), hi = std::min(g0 + blocks[q].n_points, row_end);
      g0 += blocks[q].n_points;
      if (hi > lo && !fused_variant(dim, ap.plans[q].G, ap.plans[q].kmode)) ok = false;
    }
    if (ok) {
      static thread_local FusedBatch proto;
      std::memset(&proto, 0, sizeof proto);
      proto.fb = fb;
      proto.seed = seed;
      proto.W = W;
      proto.b = b;
      return assemble_range(ctx, ap, dim, F, blocks, nullptr, row_begin, row_end, A, lda, layout,
                            rhs, ctx->stream, pdl_enabled(), &proto, s_norm);
    }
  }
  if (overflow) pb.n = 0;  // many blocks: fused features only, prefactors in batches below
  // PDL behind whatever precedes on the stream (typically the previous step's assembly): the
  // draws and folds overlap its tail, the writes wait for it (features_prefactor_kernel)
  const bool pdl_fp = pdl_enabled() && !ctx->timing && n_local * F <= kPdlMaxEntries;
  cudaError_t e = launch_features_prefactor(dim, F, fb, seed, W, b, pb, ctx->stream, pdl_fp);
  if (e != cudaSuccess) return cuda_fail(e, "features_prefactor_kernel");
  if (overflow) {
    if (fls_status s = launch_prefactors(ctx, ap, W, b, dim, F, normalize, blocks, row_begin,
                                         row_end, ctx->stream))
      return s;
  }
  if (row_end == row_begin) return FLS_OK;
  return assemble_range(ctx, ap, dim, F, blocks, nullptr, row_begin, row_end, A, lda, layout, rhs,
                        ctx->stream, pdl_enabled());
}

fls_status fls_assemble(fls_ctx *ctx, const double *W, const double *b, int32_t dim,
                        int64_t n_features, int32_t normalize, const fls_block *blocks,
                        int32_t n_blocks, int64_t row_begin, int64_t row_end, double *A,
                        int64_t lda, int32_t layout, double *rhs) {
  NvtxRange nvtx_("fls_assemble");
  if (fls_status s = check_ctx(ctx)) return s;
  static thread_local AsmPlan ap;
  if (fls_status s = validate_assemble(dim, n_features, W, b, blocks, n_blocks, row_begin, row_end,
                                       A, lda, layout, ap))
    return s;
  if (row_end == row_begin) return FLS_OK;
  DeviceGuard g(ctx->device);
  if (fls_status s = launch_prefactors(ctx, ap, W, b, dim, n_features, normalize, blocks,
                                       row_begin, row_end, ctx->stream))
    return s;
  return assemble_range(ctx, ap, dim, n_features, blocks, nullptr, row_begin, row_end, A, lda,
                        layout, rhs, ctx->stream, pdl_enabled());
}

fls_status fls_assemble_host(fls_ctx *ctx, const double *W, const double *b, int32_t dim,
                             int64_t n_features, int32_t normalize, const fls_block *blocks,
                             int32_t n_blocks, int64_t row_begin, int64_t row_end, double *A,
                             int64_t lda, double *rhs, int64_t chunk_rows) {
  NvtxRange nvtx_("fls_assemble_host");
  if (fls_status s = check_ctx(ctx)) return s;
  static thread_local AsmPlan ap;
  if (fls_status s = validate_assemble(dim, n_features, W, b, blocks, n_blocks, row_begin, row_end,
                                       A, lda, FLS_COL_MAJOR, ap))
    return s;
  if (row_end == row_begin) return FLS_OK;
  if (chunk_rows < 0) return fail(FLS_EINVAL, "chunk_rows < 0");
  const int64_t F = n_features;
  if (chunk_rows == 0) {  // ~2 GiB per staging buffer
    chunk_rows = ((int64_t)1 << 31) / (8 * (F + 1));
    chunk_rows = std::max<int64_t>(1024, chunk_rows / 1024 * 1024);
  }
  const int64_t n_local = row_end - row_begin;
  chunk_rows = std::min(chunk_rows, n_local);
  const int64_t ldc = (chunk_rows + 3) / 4 * 4;
  DeviceGuard g(ctx->device);
  cudaStream_t cs = ctx->stream;
  if (!ctx->copy_stream) FLS_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  cudaStream_t xs = ctx->copy_stream;
  for (int k = 0; k < 4; ++k)
    if (!ctx->hev[k]) FLS_CUDA(cudaEventCreateWithFlags(&ctx->hev[k], cudaEventDisableTiming));

  // 1. stage inputs: W, b and each block's slice of points / fields / values for the range
  size_t in_doubles = (size_t)F * dim + F;
  int64_t g0 = 0;
  int64_t lo_pt[64], n_pt[64];
  for (int q = 0; q < ap.n_blocks; ++q) {
    const fls_block &B = blocks[q];
    const int64_t lo = std::max(g0, row_begin), hi = std::min(g0 + B.n_points, row_end);
    lo_pt[q] = std::max<int64_t>(0, lo - g0);
    n_pt[q] = std::max<int64_t>(0, hi - lo);
    g0 += B.n_points;
    in_doubles += (size_t)n_pt[q] * (dim + B.n_fields + (B.values ? 1 : 0));
  }
  if (fls_status s = ensure_dev(ctx->hin, ctx->hin_bytes, in_doubles * sizeof(double), cs)) return s;
  if (fls_status s = ensure_dev(ctx->hout, ctx->hout_bytes, 2 * (size_t)ldc * (F + 1) * sizeof(double), cs))
    return s;
  double *Wd = ctx->hin, *bd = Wd + F * dim, *cur = bd + F;
  FLS_CUDA(cudaMemcpyAsync(Wd, W, sizeof(double) * F * dim, cudaMemcpyHostToDevice, cs));
  FLS_CUDA(cudaMemcpyAsync(bd, b, sizeof(double) * F, cudaMemcpyHostToDevice, cs));
  fls_block dblk[64];
  int64_t base[64];
  for (int q = 0; q < ap.n_blocks; ++q) {
    const fls_block &B = blocks[q];
    dblk[q] = B;
    base[q] = lo_pt[q];
    if (n_pt[q] == 0) continue;
    dblk[q].X = cur;
    FLS_CUDA(cudaMemcpyAsync(cur, B.X + lo_pt[q] * dim, sizeof(double) * n_pt[q] * dim,
                             cudaMemcpyHostToDevice, cs));
    cur += n_pt[q] * dim;
    if (B.n_fields > 0) {
      dblk[q].coef_fields = cur;
      FLS_CUDA(cudaMemcpyAsync(cur, B.coef_fields + lo_pt[q] * B.n_fields,
                               sizeof(double) * n_pt[q] * B.n_fields, cudaMemcpyHostToDevice, cs));
      cur += n_pt[q] * B.n_fields;
    }
    if (B.values) {
      dblk[q].values = cur;
      FLS_CUDA(cudaMemcpyAsync(cur, B.values + lo_pt[q], sizeof(double) * n_pt[q],
                               cudaMemcpyHostToDevice, cs));
      cur += n_pt[q];
    }
  }
  // 2. prefactors once, then chunks: compute on cs into buffer k%2, copy out on xs
  if (fls_status s = launch_prefactors(ctx, ap, Wd, bd, dim, F, normalize, dblk, row_begin,
                                       row_end, cs))
    return s;
  const int64_t n_chunks = (n_local + chunk_rows - 1) / chunk_rows;
  for (int64_t c = 0; c < n_chunks; ++c) {
    const int slot = (int)(c & 1);
    double *buf = ctx->hout + (size_t)slot * ldc * (F + 1);
    const int64_t r0 = row_begin + c * chunk_rows, r1 = std::min(row_end, r0 + chunk_rows);
    if (c >= 2) FLS_CUDA(cudaStreamWaitEvent(cs, ctx->hev[2 + slot], 0));  // buffer drained
    if (fls_status s = assemble_range(ctx, ap, dim, F, dblk, base, r0, r1, buf, ldc, FLS_COL_MAJOR,
                                      rhs ? buf + F * ldc : nullptr, cs, false))
      return s;
    FLS_CUDA(cudaEventRecord(ctx->hev[slot], cs));
    FLS_CUDA(cudaStreamWaitEvent(xs, ctx->hev[slot], 0));
    const int64_t nr = r1 - r0, off = r0 - row_begin;
    FLS_CUDA(cudaMemcpy2DAsync(A + off, sizeof(double) * lda, buf, sizeof(double) * ldc,
                               sizeof(double) * nr, F, cudaMemcpyDeviceToHost, xs));
    if (rhs)
      FLS_CUDA(cudaMemcpyAsync(rhs + off, buf + F * ldc, sizeof(double) * nr,
                               cudaMemcpyDeviceToHost, xs));
    FLS_CUDA(cudaEventRecord(ctx->hev[2 + slot], xs));
  }
  FLS_CUDA(cudaStreamSynchronize(xs));
  FLS_CUDA(cudaStreamSynchronize(cs));
  return FLS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// least squares (Alg. 1 line 5; Tikhonov form P:L156-160)
// ---------------------------------------------------------------------------------------------
namespace fls {

fls_status ensure_handles(fls_ctx *ctx) {
  if (!ctx->solver) {
    if (cusolverDnCreate(&ctx->solver) != CUSOLVER_STATUS_SUCCESS)
      return fail(FLS_ECUSOLVER, "cusolverDnCreate failed");
  }
  if (!ctx->blas) {
    if (cublasCreate(&ctx->blas) != CUBLAS_STATUS_SUCCESS)
      return fail(FLS_ECUSOLVER, "cublasCreate failed");
  }
  cusolverDnSetStream(ctx->solver, ctx->stream);
  cublasSetStream(ctx->blas, ctx->stream);
  return FLS_OK;
}

// Householder QR of an m x n column-major block in place (R in the upper trapezoid, reflectors
// below, geqrf format).  Default: libfls's blocked QR (fls_qr.cu) for n >= 1000 columns, one
// cusolverDnDgeqrf call below that (profiles/r01_qr_small.log: cuSOLVER 2.6 / 4.8 ms vs 3.2 /
// 5.2 ms at 1,002 x 501 / 2,000 x 801; blocked 6.8 vs 9.1 ms at 4,000 x 1,001).
// tau_out (k = min(m, n) doubles) may be NULL.
constexpr int64_t kQrBlockedMinCols = 1000;

// per-context solver scratch (grow-only): repeated solves (Newton, AdamW, RHS sweeps) never
// allocate -- per-call stream-ordered allocations stalled the host sporadically
static fls_status ensure_qws(fls_ctx *ctx, size_t bytes) {
  if (bytes <= ctx->qws_bytes) return FLS_OK;
  cudaStreamSynchronize(ctx->stream);
  cudaFree(ctx->qws);
  ctx->qws = nullptr;
  ctx->qws_bytes = 0;
  if (cudaMalloc((void **)&ctx->qws, bytes) != cudaSuccess) {
    cudaGetLastError();
    return fail(FLS_ENOMEM, "solver workspace of %zu bytes", bytes);
  }
  ctx->qws_bytes = bytes;
  return FLS_OK;
}

// FLS_QR: "cusolver" / "blocked" force a method (A/B timing, tests); unset = by size.  Read
// per call so a test can switch it.
static int qr_method() {
  const char *s = getenv("FLS_QR");
  if (s && std::strcmp(s, "cusolver") == 0) return 1;
  if (s && std::strcmp(s, "blocked") == 0) return 2;
  return 0;
}

fls_status geqrf_inplace(fls_ctx *ctx, double *M, int64_t m, int64_t lda, int64_t n,
                         double *tau_out, int64_t grp_base, int64_t grp_size) {
  if (m > INT32_MAX || n > INT32_MAX || lda > INT32_MAX)
    return fail(FLS_EUNSUPPORTED, "geqrf: dimensions exceed int32 (m=%lld n=%lld lda=%lld)",
                (long long)m, (long long)n, (long long)lda);
  const int64_t k = m < n ? m : n;
  // small problems (C1: 1,002 x 501) are launch-latency bound: one cuSOLVER call is faster
  const int method = qr_method();
  if (method != 1 && m <= qr_blocked_max_rows() && (method == 2 || n >= kQrBlockedMinCols)) {
    const size_t need = (qr_blocked_ws(m, n) + (size_t)(k > 0 ? k : 1)) * sizeof(double);
    if (fls_status s = ensure_qws(ctx, need)) return s;
    double *tau = tau_out ? tau_out : ctx->qws + qr_blocked_ws(m, n);
    cudaError_t ce;
    cublasStatus_t be;
    const char *msg = qr_blocked(ctx->blas, ctx->stream, M, m, n, lda, tau, ctx->qws, &ce, &be,
                                 grp_base, grp_size);
    cudaError_t e = cudaStreamSynchronize(ctx->stream);
    if (msg) {
      if (ce == cudaErrorMemoryAllocation) return fail(FLS_ENOMEM, "blocked QR: %s", msg);
      if (ce != cudaSuccess) return cuda_fail(ce, msg);
      return fail(FLS_ECUSOLVER, "blocked QR: %s (cublas status %d)", msg, (int)be);
    }
    if (e != cudaSuccess) return cuda_fail(e, "blocked QR");
    return FLS_OK;
  }
  int lwork = 0;
  if (cusolverDnDgeqrf_bufferSize(ctx->solver, (int)m, (int)n, M, (int)lda, &lwork) !=
      CUSOLVER_STATUS_SUCCESS)
    return fail(FLS_ECUSOLVER, "cusolverDnDgeqrf_bufferSize failed");
  size_t bytes = ((size_t)lwork + (size_t)k + 2) * sizeof(double);
  if (fls_status s = ensure_qws(ctx, bytes)) return s;
  double *work = ctx->qws;
  double *tau = tau_out ? tau_out : work + lwork;
  int *info = reinterpret_cast<int *>(work + lwork + k);
  cusolverStatus_t st = cusolverDnDgeqrf(ctx->solver, (int)m, (int)n, M, (int)lda, tau, work,
                                         lwork, info);
  int h_info = 0;
  cudaMemcpyAsync(&h_info, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "geqrf");
  if (st != CUSOLVER_STATUS_SUCCESS || h_info != 0)
    return fail(FLS_ECUSOLVER, "cusolverDnDgeqrf status %d info %d", (int)st, h_info);
  return FLS_OK;
}

// [A | b] (m x (F+1), lda; ridge rows already in place) -> beta = R^-1 (Q^T b)[0:F], |R(F,F)|
static fls_status qr_trsv(fls_ctx *ctx, double *Ab, int64_t m, int64_t lda, int64_t n_features,
                          double *beta, double *resid_norm, int64_t grp_base, int64_t grp_size) {
  const int64_t n = n_features + 1;
  if (fls_status s = geqrf_inplace(ctx, Ab, m, lda, n, nullptr, grp_base, grp_size)) return s;
  // zero diagonal?
  cudaError_t e = launch_min_abs_diag(Ab, lda, n_features, ctx->d_scratch, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "min_abs_diag");
  double dmin = 0.0, rnn = 0.0;
  FLS_CUDA(cudaMemcpyAsync(&dmin, ctx->d_scratch, sizeof dmin, cudaMemcpyDeviceToHost, ctx->stream));
  if (m > n_features)
    FLS_CUDA(cudaMemcpyAsync(&rnn, Ab + n_features * lda + n_features, sizeof rnn,
                             cudaMemcpyDeviceToHost, ctx->stream));
  FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (dmin == 0.0) return fail(FLS_ERANK, "R has an exactly zero diagonal entry (rank deficient)");
  // beta = R^{-1} (Q^T b)[0:n]
  FLS_CUDA(cudaMemcpyAsync(beta, Ab + n_features * lda, n_features * sizeof(double),
                           cudaMemcpyDeviceToDevice, ctx->stream));
  if (n_features > INT32_MAX) return fail(FLS_EUNSUPPORTED, "n_features exceeds int32");
  if (cublasDtrsv(ctx->blas, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT,
                  (int)n_features, Ab, (int)lda, beta, 1) != CUBLAS_STATUS_SUCCESS)
    return fail(FLS_ECUSOLVER, "cublasDtrsv failed");
  FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (resid_norm) *resid_norm = std::fabs(rnn);
  return FLS_OK;
}

fls_status frob2_host(fls_ctx *ctx, const double *A, int64_t m, int64_t lda, int64_t n,
                      double *out) {
  DeviceGuard g(ctx->device);
  const int nblk = 592;  // 4 x 148 SMs, fixed -> deterministic summation order
  cudaError_t e = launch_frob2(A, lda, m, n, ctx->d_scratch + 8, nblk, ctx->d_scratch, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "frob2");
  FLS_CUDA(cudaMemcpyAsync(out, ctx->d_scratch, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  return FLS_OK;
}

fls_status solve_local(fls_ctx *ctx, double *Ab, int64_t n_rows, int64_t lda, int64_t F,
                       double sqrt_mu, double *beta, double *resid_norm) {
  const int64_t m = n_rows + (sqrt_mu > 0.0 ? F : 0);
  if (n_rows < 0 || lda < m)
    return fail(FLS_EINVAL, "lda %lld < rows %lld (ridge rows included)", (long long)lda,
                (long long)m);
  if (m < F)
    return fail(FLS_EINVAL, "underdetermined: %lld rows < %lld features without ridge",
                (long long)m, (long long)F);
  DeviceGuard g(ctx->device);
  if (fls_status s = ensure_handles(ctx)) return s;
  if (sqrt_mu > 0.0) {
    cudaError_t e = launch_ridge_fill(Ab, lda, n_rows, F, F + 1, sqrt_mu, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(e, "ridge_fill");
  }
  // the ridge rows [sqrt_mu I | 0] below row n_rows: ridge row i is zero left of column i, so
  // the blocked QR can stop each panel where the ridge rows still are (grouped mode, G = 1)
  return qr_trsv(ctx, Ab, m, lda, F, beta, resid_norm, sqrt_mu > 0.0 ? n_rows : 0,
                 sqrt_mu > 0.0 ? 1 : 0);
}

fls_status solve_stacked_impl(fls_ctx *ctx, const double *S, int32_t P, int64_t kb, int64_t bs,
                              int64_t cs, int64_t F, double sqrt_mu, double *beta,
                              double *resid_norm) {
  const int64_t n = F + 1;
  const int64_t gq = (P - 1) + (sqrt_mu > 0.0 ? 1 : 0);
  const int64_t groups = gq > 0 ? std::max<int64_t>(kb, sqrt_mu > 0.0 ? F : 0) : 0;
  const int64_t m = kb + groups * gq;
  if (m < F) return fail(FLS_EINVAL, "underdetermined: %lld rows < %lld features", (long long)m,
                         (long long)F);
  const int64_t ldm = (m + 3) / 4 * 4;
  DeviceGuard g(ctx->device);
  if (fls_status s = ensure_handles(ctx)) return s;
  const size_t need = sizeof(double) * (size_t)ldm * n;
  if (need > ctx->sws_bytes) {  // grow-only scratch for the permuted stack
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->sws);
    ctx->sws = nullptr;
    ctx->sws_bytes = 0;
    if (cudaMalloc((void **)&ctx->sws, need) != cudaSuccess) {
      cudaGetLastError();
      return fail(FLS_ENOMEM, "stacked-solve workspace of %zu bytes", need);
    }
    ctx->sws_bytes = need;
  }
  cudaError_t e = launch_stack_permute(S, bs, cs, P, kb, F, sqrt_mu, gq > 0 ? gq : 1, m, n,
                                       ctx->sws, ldm, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "stack_permute");
  return qr_trsv(ctx, ctx->sws, m, ldm, F, beta, resid_norm, kb, gq);
}

}  // namespace fls

extern "C" {

fls_status fls_solve(fls_ctx *ctx, double *Ab, int64_t n_rows, int64_t lda, int64_t n_features,
                     double ridge_rel, double *beta, double *resid_norm) {
  NvtxRange nvtx_("fls_solve");
  if (fls_status s = check_ctx(ctx)) return s;
  if (!Ab || !beta) return fail(FLS_EINVAL, "Ab or beta is NULL");
  if (n_features < 1) return fail(FLS_EINVAL, "n_features < 1");
  if (n_rows < 0) return fail(FLS_EINVAL, "n_rows < 0");
  if (!(ridge_rel >= 0.0) || !std::isfinite(ridge_rel))
    return fail(FLS_EINVAL, "ridge_rel must be >= 0 and finite");
  DeviceGuard g(ctx->device);
  // surface pending async errors first -- with a communicator the status is agreed with the
  // other ranks inside comm_solve (returning here alone would leave them waiting)
  const fls_status pending = fls_sync(ctx);
  bool handled = false;
  fls_status cs = comm_solve(ctx, Ab, n_rows, lda, n_features, ridge_rel, -1.0, beta, resid_norm,
                             &handled, pending);
  if (handled) return cs;
  if (pending) return pending;
  double sqrt_mu = 0.0;
  if (ridge_rel > 0.0) {  // reading A16: sqrt(mu) = tau ||A||_F (A without the rhs column)
    if (lda < n_rows) return fail(FLS_EINVAL, "lda < n_rows");
    double fro2 = 0.0;
    if (fls_status s = frob2_host(ctx, Ab, n_rows, lda, n_features, &fro2)) return s;
    sqrt_mu = ridge_rel * std::sqrt(fro2);
  }
  return solve_local(ctx, Ab, n_rows, lda, n_features, sqrt_mu, beta, resid_norm);
}

fls_status fls_solve_mu(fls_ctx *ctx, double *Ab, int64_t n_rows, int64_t lda, int64_t n_features,
                        double sqrt_mu, double *beta, double *resid_norm) {
  NvtxRange nvtx_("fls_solve_mu");
  if (fls_status s = check_ctx(ctx)) return s;
  if (!Ab || !beta) return fail(FLS_EINVAL, "Ab or beta is NULL");
  if (n_features < 1) return fail(FLS_EINVAL, "n_features < 1");
  if (n_rows < 0) return fail(FLS_EINVAL, "n_rows < 0");
  if (!(sqrt_mu >= 0.0) || !std::isfinite(sqrt_mu)) return fail(FLS_EINVAL, "sqrt_mu must be >= 0");
  DeviceGuard g(ctx->device);
  const fls_status pending = fls_sync(ctx);
  bool handled = false;
  fls_status cs = comm_solve(ctx, Ab, n_rows, lda, n_features, 0.0, sqrt_mu, beta, resid_norm,
                             &handled, pending);
  if (handled) return cs;
  if (pending) return pending;
  return solve_local(ctx, Ab, n_rows, lda, n_features, sqrt_mu, beta, resid_norm);
}

fls_status fls_solve_stacked(fls_ctx *ctx, const double *S, int32_t n_blocks, int64_t kb,
                             int64_t lds, int64_t n_features, double sqrt_mu, double *beta,
                             double *resid_norm) {
  NvtxRange nvtx_("fls_solve_stacked");
  if (fls_status s = check_ctx(ctx)) return s;
  if (!S || !beta) return fail(FLS_EINVAL, "S or beta is NULL");
  if (n_features < 1 || n_blocks < 1 || kb < 1) return fail(FLS_EINVAL, "bad sizes");
  if (lds < (int64_t)n_blocks * kb)
    return fail(FLS_EINVAL, "lds %lld < n_blocks * kb = %lld", (long long)lds,
                (long long)n_blocks * kb);
  if (!(sqrt_mu >= 0.0) || !std::isfinite(sqrt_mu)) return fail(FLS_EINVAL, "sqrt_mu must be >= 0");
  DeviceGuard g(ctx->device);
  if (fls_status s = fls_sync(ctx)) return s;
  return solve_stacked_impl(ctx, S, n_blocks, kb, kb, lds, n_features, sqrt_mu, beta, resid_norm);
}

}  // extern "C"

struct fls_qr {
  int device = 0;
  int64_t m = 0, n = 0, ld = 0, m_rows = 0;  // m = factored rows (incl. ridge), m_rows = data rows
  double *M = nullptr;                        // Householder vectors + R, column-major
  double *tau = nullptr;
};

extern "C" {

fls_status fls_qr_factor(fls_ctx *ctx, const double *A, int64_t n_rows, int64_t lda,
                         int64_t n_features, double sqrt_mu, fls_qr **out) {
  NvtxRange nvtx_("fls_qr_factor");
  if (fls_status s = check_ctx(ctx)) return s;
  if (!A || !out) return fail(FLS_EINVAL, "A or out is NULL");
  *out = nullptr;
  if (n_features < 1 || n_rows < 0 || lda < n_rows) return fail(FLS_EINVAL, "bad sizes");
  if (!(sqrt_mu >= 0.0) || !std::isfinite(sqrt_mu)) return fail(FLS_EINVAL, "sqrt_mu must be >= 0");
  const int64_t m = n_rows + (sqrt_mu > 0.0 ? n_features : 0);
  if (m < n_features) return fail(FLS_EINVAL, "underdetermined without ridge");
  DeviceGuard g(ctx->device);
  if (fls_status s = fls_sync(ctx)) return s;
  if (fls_status s = ensure_handles(ctx)) return s;
  fls_qr *q = new fls_qr();
  q->device = ctx->device;
  q->m = m;
  q->m_rows = n_rows;
  q->n = n_features;
  q->ld = (m + 3) / 4 * 4;
  if (cudaMalloc(&q->M, sizeof(double) * q->ld * n_features) != cudaSuccess ||
      cudaMalloc(&q->tau, sizeof(double) * n_features) != cudaSuccess) {
    cudaGetLastError();
    fls_qr_destroy(q);
    return fail(FLS_ENOMEM, "fls_qr_factor: %lld x %lld storage", (long long)q->ld, (long long)n_features);
  }
  cudaError_t e = cudaMemcpy2DAsync(q->M, sizeof(double) * q->ld, A, sizeof(double) * lda,
                                    sizeof(double) * n_rows, n_features, cudaMemcpyDeviceToDevice,
                                    ctx->stream);
  if (e == cudaSuccess && sqrt_mu > 0.0)
    e = launch_ridge_fill(q->M, q->ld, n_rows, n_features, n_features, sqrt_mu, ctx->stream);
  if (e != cudaSuccess) {
    fls_qr_destroy(q);
    return cuda_fail(e, "fls_qr_factor copy");
  }
  // grouped mode for the ridge rows (zero left of their column); the stored reflectors are
  // zero wherever a panel stopped, so ormqr applies them unchanged
  if (fls_status s = geqrf_inplace(ctx, q->M, m, q->ld, n_features, q->tau,
                                   sqrt_mu > 0.0 ? n_rows : 0, sqrt_mu > 0.0 ? 1 : 0)) {
    fls_qr_destroy(q);
    return s;
  }
  double dmin = 0.0;
  launch_min_abs_diag(q->M, q->ld, n_features, ctx->d_scratch, ctx->stream);
  cudaMemcpyAsync(&dmin, ctx->d_scratch, sizeof dmin, cudaMemcpyDeviceToHost, ctx->stream);
  e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    fls_qr_destroy(q);
    return cuda_fail(e, "fls_qr_factor");
  }
  if (dmin == 0.0) {
    fls_qr_destroy(q);
    return fail(FLS_ERANK, "R has an exactly zero diagonal entry (rank deficient)");
  }
  *out = q;
  return FLS_OK;
}

fls_status fls_qr_solve(fls_ctx *ctx, const fls_qr *q, const double *B, int64_t ldb, int64_t nrhs,
                        double *Beta, int64_t ldbeta) {
  NvtxRange nvtx_("fls_qr_solve");
  if (fls_status s = check_ctx(ctx)) return s;
  if (!q || !B || !Beta) return fail(FLS_EINVAL, "qr, B or Beta is NULL");
  if (nrhs < 1 || ldb < q->m_rows || ldbeta < q->n) return fail(FLS_EINVAL, "bad sizes");
  if (q->device != ctx->device) return fail(FLS_EINVAL, "qr factored on device %d", q->device);
  DeviceGuard g(ctx->device);
  if (fls_status s = ensure_handles(ctx)) return s;
  double *C = nullptr;
  const int64_t ldc = q->ld;
  int lwork = 0;
  if (cusolverDnDormqr_bufferSize(ctx->solver, CUBLAS_SIDE_LEFT, CUBLAS_OP_T, (int)q->m, (int)nrhs,
                                  (int)q->n, q->M, (int)q->ld, q->tau, C, (int)ldc, &lwork) !=
      CUSOLVER_STATUS_SUCCESS)
    return fail(FLS_ECUSOLVER, "ormqr_bufferSize");
  const size_t cbytes = sizeof(double) * ldc * nrhs;
  if (fls_status s = ensure_qws(ctx, cbytes + sizeof(double) * (lwork + 2))) return s;
  C = ctx->qws;
  double *work = C + ldc * nrhs;
  int *info = reinterpret_cast<int *>(work + lwork);
  FLS_CUDA(cudaMemsetAsync(C, 0, cbytes, ctx->stream));
  FLS_CUDA(cudaMemcpy2DAsync(C, sizeof(double) * ldc, B, sizeof(double) * ldb,
                             sizeof(double) * q->m_rows, nrhs, cudaMemcpyDeviceToDevice, ctx->stream));
  cusolverStatus_t st = cusolverDnDormqr(ctx->solver, CUBLAS_SIDE_LEFT, CUBLAS_OP_T, (int)q->m,
                                         (int)nrhs, (int)q->n, q->M, (int)q->ld, q->tau, C,
                                         (int)ldc, work, lwork, info);
  const double one = 1.0;
  cublasStatus_t bs = cublasDtrsm(ctx->blas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                                  CUBLAS_DIAG_NON_UNIT, (int)q->n, (int)nrhs, &one, q->M,
                                  (int)q->ld, C, (int)ldc);
  cudaMemcpy2DAsync(Beta, sizeof(double) * ldbeta, C, sizeof(double) * ldc, sizeof(double) * q->n,
                    nrhs, cudaMemcpyDeviceToDevice, ctx->stream);
  FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (st != CUSOLVER_STATUS_SUCCESS) return fail(FLS_ECUSOLVER, "ormqr status %d", (int)st);
  if (bs != CUBLAS_STATUS_SUCCESS) return fail(FLS_ECUSOLVER, "trsm status %d", (int)bs);
  return FLS_OK;
}

fls_status fls_qr_destroy(fls_qr *q) {
  if (!q) return FLS_OK;
  DeviceGuard g(q->device);
  cudaFree(q->M);
  cudaFree(q->tau);
  delete q;
  return FLS_OK;
}

fls_status fls_geqrf(fls_ctx *ctx, double *M, int64_t n_rows, int64_t lda, int64_t n_cols,
                     double *tau) {
  NvtxRange nvtx_("fls_geqrf");
  if (fls_status s = check_ctx(ctx)) return s;
  if (!M || !tau) return fail(FLS_EINVAL, "M or tau is NULL");
  if (n_rows < 1 || n_cols < 1 || lda < n_rows)
    return fail(FLS_EINVAL, "bad sizes n_rows %lld n_cols %lld lda %lld", (long long)n_rows,
                (long long)n_cols, (long long)lda);
  DeviceGuard g(ctx->device);
  if (fls_status s = fls_sync(ctx)) return s;
  if (fls_status s = ensure_handles(ctx)) return s;
  return geqrf_inplace(ctx, M, n_rows, lda, n_cols, tau);
}

fls_status fls_ipc_handle(fls_ctx *ctx, void *dev_ptr, void *handle, int64_t *offset) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (!dev_ptr || !handle || !offset) return fail(FLS_EINVAL, "dev_ptr, handle or offset is NULL");
  static_assert(sizeof(cudaIpcMemHandle_t) <= FLS_IPC_HANDLE_BYTES, "IPC handle size");
  DeviceGuard g(ctx->device);
  // allocation base through the driver entry point (no link-time libcuda dependency)
  typedef CUresult (*range_fn)(CUdeviceptr *, size_t *, CUdeviceptr);
  static range_fn get_range = nullptr;
  if (!get_range) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(FLS_ECUDA, "cuMemGetAddressRange entry point unavailable");
    get_range = reinterpret_cast<range_fn>(fn);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return fail(FLS_EINVAL, "dev_ptr is not device memory");
  *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  cudaIpcMemHandle_t h;
  FLS_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base)));
  std::memset(handle, 0, FLS_IPC_HANDLE_BYTES);
  std::memcpy(handle, &h, sizeof h);
  return FLS_OK;
}

fls_status fls_ipc_open(fls_ctx *ctx, const void *handle, void **dev_ptr) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (!handle || !dev_ptr) return fail(FLS_EINVAL, "handle or dev_ptr is NULL");
  DeviceGuard g(ctx->device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  *dev_ptr = nullptr;
  FLS_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return FLS_OK;
}

fls_status fls_ipc_close(fls_ctx *ctx, void *dev_ptr) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (!dev_ptr) return fail(FLS_EINVAL, "dev_ptr is NULL");
  DeviceGuard g(ctx->device);
  FLS_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return FLS_OK;
}

fls_status fls_qr_r(fls_ctx *ctx, double *M, int64_t n_rows, int64_t lda, int64_t n_cols,
                    double *R, int64_t ldr) {
  NvtxRange nvtx_("fls_qr_r");
  if (fls_status s = check_ctx(ctx)) return s;
  if (!M || !R) return fail(FLS_EINVAL, "M or R is NULL");
  if (n_rows < 1 || n_cols < 1 || lda < n_rows)
    return fail(FLS_EINVAL, "bad sizes n_rows %lld n_cols %lld lda %lld", (long long)n_rows,
                (long long)n_cols, (long long)lda);
  const int64_t k = n_rows < n_cols ? n_rows : n_cols;
  if (ldr < k) return fail(FLS_EINVAL, "ldr %lld < %lld", (long long)ldr, (long long)k);
  DeviceGuard g(ctx->device);
  if (fls_status s = fls_sync(ctx)) return s;
  if (fls_status s = ensure_handles(ctx)) return s;
  if (fls_status s = geqrf_inplace(ctx, M, n_rows, lda, n_cols)) return s;
  cudaError_t e = launch_copy_upper(M, lda, k, n_cols, R, ldr, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "copy_upper");
  FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  return FLS_OK;
}

static fls_status sample_common(fls_ctx *ctx, int32_t dim, const double *lo, const double *hi,
                                SampleArgs &sa) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (dim < 1 || dim > FLS_MAX_DIM) return fail(FLS_EINVAL, "dim %d not in 1..%d", dim, FLS_MAX_DIM);
  if (!lo || !hi) return fail(FLS_EINVAL, "lo or hi is NULL");
  sa.D = dim;
  for (int k = 0; k < dim; ++k) {
    if (!(lo[k] < hi[k]) || !std::isfinite(lo[k]) || !std::isfinite(hi[k]))
      return fail(FLS_EINVAL, "need finite lo[%d] < hi[%d]", k, k);
    sa.lo[k] = lo[k];
    sa.hi[k] = hi[k];
  }
  return FLS_OK;
}

fls_status fls_sample_box(fls_ctx *ctx, int32_t dim, int64_t n, const double *lo, const double *hi,
                          uint64_t seed, uint64_t stream, double *X) {
  SampleArgs sa;
  std::memset(&sa, 0, sizeof sa);
  if (fls_status s = sample_common(ctx, dim, lo, hi, sa)) return s;
  if (n < 0) return fail(FLS_EINVAL, "n < 0");
  if (n > 0 && !X) return fail(FLS_EINVAL, "X is NULL");
  sa.rows = n;
  sa.seed = seed;
  sa.stream = stream;
  sa.X = X;
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_sample(sa, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "sample_kernel");
  return FLS_OK;
}

fls_status fls_sample_faces(fls_ctx *ctx, int32_t dim, int64_t per_face, uint32_t axes_mask,
                            const double *lo, const double *hi, uint64_t seed, uint64_t stream,
                            double *X) {
  SampleArgs sa;
  std::memset(&sa, 0, sizeof sa);
  if (fls_status s = sample_common(ctx, dim, lo, hi, sa)) return s;
  if (per_face < 0) return fail(FLS_EINVAL, "per_face < 0");
  if (axes_mask >> dim) return fail(FLS_EINVAL, "axes_mask has bits beyond dim %d", dim);
  int nax = 0;
  for (int k = 0; k < dim; ++k)
    if (axes_mask & (1u << k)) sa.face_axis[nax++] = k;
  sa.rows = 2 * per_face * nax;
  if (sa.rows > 0 && !X) return fail(FLS_EINVAL, "X is NULL");
  sa.per_face = per_face;
  sa.seed = seed;
  sa.stream = stream;
  sa.X = X;
  if (sa.rows == 0) return FLS_OK;
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_sample(sa, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "sample_kernel");
  return FLS_OK;
}

fls_status fls_features_transform(fls_ctx *ctx, int32_t dim, int64_t n_features, const double *L,
                                  const double *W_hat, double *W) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (dim < 1 || dim > FLS_MAX_DIM) return fail(FLS_EINVAL, "dim %d not in 1..%d", dim, FLS_MAX_DIM);
  if (n_features < 1) return fail(FLS_EINVAL, "n_features < 1");
  if (!L || !W_hat || !W) return fail(FLS_EINVAL, "NULL pointer");
  TransformArgs t;
  std::memset(&t, 0, sizeof t);
  for (int i = 0; i < dim * dim; ++i) {
    if (!std::isfinite(L[i])) return fail(FLS_EINVAL, "L[%d] not finite", i);
    t.L[i] = L[i];
  }
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_transform(dim, n_features, t, W_hat, W, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "transform_kernel");
  return FLS_OK;
}

fls_status fls_bandwidth_grad(fls_ctx *ctx, const double *W, const double *W_hat, const double *b,
                              int32_t dim, int64_t n_features, int32_t normalize,
                              const fls_block *blocks, int32_t n_blocks, const double *beta,
                              double *G) {
  NvtxRange nvtx_("fls_bandwidth_grad");
  if (fls_status s = check_ctx(ctx)) return s;
  if (!W_hat || !beta || !G) return fail(FLS_EINVAL, "W_hat, beta or G is NULL");
  static thread_local AsmPlan ap;
  int64_t total = 0;
  for (int q = 0; blocks && q < n_blocks; ++q) total += blocks[q].n_points;
  // same block / operator validation as the assembly (no output matrix: pass W as a dummy A
  // with a row-major lda that always passes)
  if (fls_status s = validate_assemble(dim, n_features, W, b, blocks, n_blocks, 0, total, W,
                                       n_features, FLS_ROW_MAJOR, ap))
    return s;
  for (int q = 0; q < n_blocks; ++q) {
    if (blocks[q].n_points > 0 && !blocks[q].values)
      return fail(FLS_EINVAL, "block %d: values (the residual rows) is NULL", q);
  }
  const int64_t F = n_features;
  DeviceGuard g(ctx->device);
  // records: kGradRec doubles per feature per block; partial slots: <= 16 per block
  if (fls_status s = ensure_ws(ctx, (size_t)n_blocks * F * kGradRec * sizeof(double))) return s;
  int nslots = 0;
  int slots_q[64];
  for (int q = 0; q < n_blocks; ++q) {
    const int64_t n = blocks[q].n_points;
    slots_q[q] = n == 0 ? 0 : (int)std::min<int64_t>(16, (n + 255) / 256);
    nslots += slots_q[q];
  }
  // partial sums: grow-only per-context buffer (repeated calls in the AdamW loop)
  const size_t pbytes = sizeof(double) * ((size_t)std::max(nslots, 1) * F * dim + (size_t)dim * dim);
  if (pbytes > ctx->gws_bytes) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->gws);
    ctx->gws = nullptr;
    ctx->gws_bytes = 0;
    if (cudaMalloc((void **)&ctx->gws, pbytes) != cudaSuccess) {
      cudaGetLastError();
      return fail(FLS_ENOMEM, "bandwidth_grad workspace");
    }
    ctx->gws_bytes = pbytes;
  }
  double *partials = ctx->gws;
  double *Gd = partials + (size_t)std::max(nslots, 1) * F * dim;
  const double s_norm = normalize ? 1.0 / std::sqrt((double)F) : 1.0;
  int slot0 = 0;
  cudaError_t e = cudaSuccess;
  for (int q = 0; q < n_blocks && e == cudaSuccess; ++q) {
    if (slots_q[q] == 0) continue;
    const fls_block &B = blocks[q];
    PrefArgs pa;
    std::memset(&pa, 0, sizeof pa);
    pa.W = W;
    pa.b = b;
    pa.F = F;
    pa.D = dim;
    pa.n_terms = ap.plans[q].n_terms;
    pa.G = ap.plans[q].G;
    pa.S = grad_stride(dim, pa.G);
    pa.scale = s_norm * B.weight;
    pa.pf = ctx->ws + (size_t)q * F * kGradRec;
    pa.err = ctx->d_err;
    std::memcpy(pa.terms, ap.plans[q].terms, sizeof pa.terms);
    e = launch_grad_prefactor(pa, ctx->stream);
    if (e != cudaSuccess) break;
    GradArgs ga;
    std::memset(&ga, 0, sizeof ga);
    ga.pf = pa.pf;
    ga.S = pa.S;
    ga.fields = B.coef_fields;
    ga.nf = B.n_fields;
    for (int g2 = 0; g2 < pa.G; ++g2) ga.gfield[g2] = ap.plans[q].gfield[g2];
    ga.F = F;
    ga.X = B.X;
    ga.r = B.values;
    ga.row0 = 0;
    ga.row1 = B.n_points;
    ga.rows_per_slot = (B.n_points + slots_q[q] - 1) / slots_q[q];
    ga.slot0 = slot0;
    ga.partials = partials;
    ga.err = ctx->d_err;
    e = launch_grad_reduce(dim, pa.G, ga, slots_q[q], ctx->stream);
    slot0 += slots_q[q];
  }
  if (e == cudaSuccess) {
    if (nslots == 0) e = cudaMemsetAsync(Gd, 0, sizeof(double) * dim * dim, ctx->stream);
    else e = launch_grad_final(dim, F, nslots, partials, beta, W_hat, Gd, ctx->stream);
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(G, Gd, sizeof(double) * dim * dim, cudaMemcpyDeviceToHost, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "bandwidth_grad");
  FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  return FLS_OK;
}

fls_status fls_nl_residual(fls_ctx *ctx, const fls_nonlinearity *nl, int64_t n, const double *Lu,
                           const double *u, const double *u_prev, const double *f,
                           double *neg_res, double *dN, double *stats) {
  return fls_nl_residual2(ctx, nl, n, Lu, u, nullptr, u_prev, f, neg_res, dN, nullptr, stats);
}

fls_status fls_nl_residual2(fls_ctx *ctx, const fls_nonlinearity *nl, int64_t n, const double *Lu,
                            const double *u, const double *Du, const double *u_prev,
                            const double *f, double *neg_res, double *dN, double *dN_dDu,
                            double *stats) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (!nl) return fail(FLS_EINVAL, "nl is NULL");
  if (nl->kind != FLS_NL_POLY && nl->kind != FLS_NL_EXP && nl->kind != FLS_NL_UDU)
    return fail(FLS_EINVAL, "nonlinearity kind %d unknown", nl->kind);
  if (nl->kind == FLS_NL_UDU && n > 0 && !Du)
    return fail(FLS_EINVAL, "FLS_NL_UDU needs the derivative vector Du");
  if (nl->kind == FLS_NL_POLY && (nl->degree < 0 || nl->degree > 7))
    return fail(FLS_EINVAL, "polynomial degree %d not in 0..7", nl->degree);
  for (int k = 0; k < 8; ++k)
    if (!std::isfinite(nl->a[k])) return fail(FLS_EINVAL, "nonlinearity coefficient %d not finite", k);
  if (n < 0) return fail(FLS_EINVAL, "n < 0");
  if (n > 0 && (!Lu || !u || !f || !neg_res)) return fail(FLS_EINVAL, "NULL vector");
  DeviceGuard g(ctx->device);
  NlArgs a;
  std::memset(&a, 0, sizeof a);
  a.kind = nl->kind;
  a.degree = nl->kind == FLS_NL_POLY ? nl->degree : 1;
  for (int k = 0; k < 8; ++k) a.c[k] = nl->a[k];
  a.n = n;
  a.Lu = Lu;
  a.u = u;
  a.u_prev = u_prev;
  a.f = f;
  a.neg_res = neg_res;
  a.dN = dN;
  a.Du = Du;
  a.dN2 = dN_dDu;
  a.partials = ctx->d_scratch + 8;
  a.err = ctx->d_err;
  const int nblk = 296;  // 2 x 148 SMs, fixed -> deterministic sums
  cudaError_t e = launch_nl_residual(a, nblk, ctx->d_scratch, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "nl_residual");
  if (stats) {
    FLS_CUDA(cudaMemcpyAsync(stats, ctx->d_scratch, 3 * sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    FLS_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  return FLS_OK;
}

fls_status fls_axpy(fls_ctx *ctx, int64_t n, double alpha, const double *x, const double *y,
                    double *out) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (n < 0 || !std::isfinite(alpha)) return fail(FLS_EINVAL, "bad n or alpha");
  if (n > 0 && (!x || !y || !out)) return fail(FLS_EINVAL, "NULL vector");
  DeviceGuard g(ctx->device);
  cudaError_t e = launch_axpy(n, alpha, x, y, out, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "axpy");
  return FLS_OK;
}

fls_status fls_frob2(fls_ctx *ctx, const double *A, int64_t n_rows, int64_t lda, int64_t n_cols,
                     double *out) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (!A || !out) return fail(FLS_EINVAL, "A or out is NULL");
  if (n_rows < 0 || n_cols < 0 || lda < n_rows) return fail(FLS_EINVAL, "bad sizes");
  return frob2_host(ctx, A, n_rows, lda, n_cols, out);
}

// ---------------------------------------------------------------------------------------------
static fls_status eval_common(fls_ctx *ctx, const double *W, const double *b, int32_t dim,
                              int64_t n_features, int32_t normalize, const double *beta,
                              const fls_operator *op, const double *X, int64_t n_points,
                              const double *fields, int32_t n_fields, double weight, double *out,
                              bool allow_fields) {
  if (fls_status s = check_ctx(ctx)) return s;
  if (dim < 1 || dim > FLS_MAX_DIM) return fail(FLS_EINVAL, "dim %d not in 1..%d", dim, FLS_MAX_DIM);
  if (n_features < 1) return fail(FLS_EINVAL, "n_features < 1");
  if (!W || !b || !beta) return fail(FLS_EINVAL, "W, b or beta is NULL");
  if (n_points < 0) return fail(FLS_EINVAL, "n_points < 0");
  if (n_points > 0 && (!X || !out)) return fail(FLS_EINVAL, "X or out is NULL");
  if (!std::isfinite(weight)) return fail(FLS_EINVAL, "weight not finite");
  fls_term ident;
  std::memset(&ident, 0, sizeof ident);
  ident.coef = 1.0;
  ident.field = -1;
  fls_operator idop{dim, 1, &ident};
  OpPlan pl;
  if (fls_status s = plan_operator(op ? op : &idop, dim, n_fields, allow_fields, pl, "eval operator"))
    return s;
  if (pl.G > 0 && n_points > 0 && !fields)
    return fail(FLS_EINVAL, "eval operator uses coefficient fields but coef_fields is NULL");
  if (n_points == 0) return FLS_OK;
  DeviceGuard g(ctx->device);
  const int S = pf_stride(dim, pl.G, KM_SINCOS);
  const int Smax = pf_stride(FLS_MAX_DIM, FLS_MAX_FIELDS, KM_SINCOS);
  if (fls_status s = ensure_ws(ctx, (size_t)n_features * Smax * sizeof(double))) return s;
  PrefArgs pa;
  std::memset(&pa, 0, sizeof pa);
  pa.W = W;
  pa.b = b;
  pa.F = n_features;
  pa.D = dim;
  pa.n_terms = pl.n_terms;
  pa.G = pl.G;
  pa.pmode = PM_SINCOS;
  pa.S = S;
  pa.scale = (normalize ? 1.0 / std::sqrt((double)n_features) : 1.0) * weight;
  pa.pf = ctx->ws;
  pa.err = ctx->d_err;
  std::memcpy(pa.terms, pl.terms, sizeof pl.terms);
  cudaError_t e = launch_prefactor(pa, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "prefactor_kernel");
  EvalArgs ea;
  std::memset(&ea, 0, sizeof ea);
  ea.pf = pa.pf;
  ea.S = S;
  ea.F = n_features;
  ea.beta = beta;
  ea.X = X;
  ea.n = n_points;
  ea.out = out;
  ea.err = ctx->d_err;
  ea.fields = fields;
  ea.nf = n_fields;
  ea.G = pl.G;
  for (int q = 0; q < pl.G; ++q) ea.gfield[q] = pl.gfield[q];
  ea.sin_only = pl.pmode == PM_SIN ? 1 : 0;   // all orders even (e.g. u_N itself)
  e = launch_eval(dim, ea, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "eval_kernel");
  return FLS_OK;
}

fls_status fls_eval(fls_ctx *ctx, const double *W, const double *b, int32_t dim,
                    int64_t n_features, int32_t normalize, const double *beta,
                    const fls_operator *op, const double *X, int64_t n_points, double *out) {
  NvtxRange nvtx_("fls_eval");
  return eval_common(ctx, W, b, dim, n_features, normalize, beta, op, X, n_points, nullptr, 0, 1.0,
                     out, false);
}

fls_status fls_eval_block(fls_ctx *ctx, const double *W, const double *b, int32_t dim,
                          int64_t n_features, int32_t normalize, const double *beta,
                          const fls_block *block, double *out) {
  NvtxRange nvtx_("fls_eval_block");
  if (!block) return fail(FLS_EINVAL, "block is NULL");
  if (!block->op) return fail(FLS_EINVAL, "block operator is NULL");
  if (block->n_fields < 0 || block->n_fields > 64) return fail(FLS_EINVAL, "n_fields out of range");
  return eval_common(ctx, W, b, dim, n_features, normalize, beta, block->op, block->X,
                     block->n_points, block->coef_fields, block->n_fields, block->weight, out, true);
}

}  // extern "C"
