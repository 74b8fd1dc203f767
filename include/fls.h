/*
 * fls.h -- C ABI of the B200-native Fast-LSQ assembly library (libfls.so).
 *
 * Fast-LSQ (arxiv 2602.10541) solves a linear PDE  L[u] = f in Omega,  B[u] = g on dOmega
 * with the sinusoidal random-feature ansatz (Eq. 1)
 *
 *     u_N(x) = s * sum_j beta_j sin(W_j . x + b_j),   s = 1/sqrt(N),
 *     W_j ~ N(0, sigma^2 I_d),  b_j ~ U(0, 2 pi)  frozen,
 *
 * by one least-squares solve of the augmented system (Eq. 3)
 *
 *     [ A_pde ; lambda A_bc ] beta = [ f ; lambda g ],   A_ij = L[phi_j](x_i),
 *
 * where every entry is the closed form of the cyclic derivative (Eq. 2)
 *
 *     D^alpha sin(W_j . x + b_j) = (prod_k W_jk^alpha_k) Phi_{|alpha| mod 4}(W_j . x + b_j),
 *     Phi_0 = sin, Phi_1 = cos, Phi_2 = -sin, Phi_3 = -cos.
 *
 * This library implements Algorithm 1 on one B200 per process:
 *     fls_features  -- line 1, sample W and b
 *     fls_assemble  -- lines 3-5 (first half): A_pde, lambda A_bc, (lambda A_ic), rhs
 *     fls_solve     -- line 5 (second half): beta = argmin ||A beta - b||^2 (+ mu ||beta||^2),
 *                      TSQR over the ranks when a communicator is attached (fls_comm_init)
 *     fls_eval      -- line 6: u_N (or L[u_N]) at arbitrary points
 * Notation in this header: n_features = N of the paper (BASELINE.json calls it M),
 * n_points = collocation rows (the paper's M_1, M_2).
 *
 * Conventions (all entry points)
 *   - Every floating-point quantity is fp64.  Pointers are DEVICE pointers (cudaMalloc'd or
 *     torch CUDA tensors on the ctx's device) unless the comment says "host".
 *   - Ownership: the caller owns every buffer passed in; the library never frees caller
 *     memory and never retains a caller pointer after a call returns (the enqueued kernels
 *     read / write it later on the ctx's stream, so the caller must keep it alive until the
 *     stream reaches that point).  The ctx owns a small internal workspace (per-feature
 *     prefactors, O(n_blocks * n_features * (dim + 6)) doubles), grown on demand.
 *   - Streams: work is enqueued on the stream borrowed at fls_ctx_create (0 = legacy default
 *     stream).  fls_features / fls_assemble / fls_eval are ASYNCHRONOUS; fls_solve and
 *     fls_sync are blocking.  A ctx is not thread-safe: use one ctx per host thread (or
 *     serialise calls); several ctx may share a device and a stream.
 *   - Errors: every call returns fls_status.  Argument errors (FLS_EINVAL) are detected on
 *     the host before anything is enqueued.  Non-finite inputs (W, b, X, values, coefficient
 *     fields) are detected by the kernels themselves and reported asynchronously: the next
 *     fls_sync / fls_solve on the ctx returns FLS_ENONFINITE (the affected output is then
 *     unspecified).  fls_last_error() returns a thread-local message for the last failure.
 *   - Determinism: for fixed inputs every assembled entry is bit-identical regardless of the
 *     row range [row_begin, row_end) a call produces (row sharding), the layout, lda, and the
 *     launch configuration.
 */
#ifndef FLS_H_
#define FLS_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define FLS_API __attribute__((visibility("default")))
#else
#define FLS_API
#endif

#define FLS_API_VERSION 3  /* 3: fls_comm_* (multi-rank TSQR inside fls_solve), fls_solve takes ridge_rel, fls_solve_mu; 2: fls_features_assemble, fls_geqrf, fls_eval_block, fls_ipc_*, fls_solve_stacked */
#define FLS_MAX_DIM 8      /* spatial / space-time dimension d <= 8 */
#define FLS_MAX_TERMS 64   /* terms per operator */
#define FLS_MAX_FIELDS 4   /* coefficient fields per block */
#define FLS_MAX_FEAT_BLOCKS 16 /* bandwidth blocks of a multi-block basis */
/* Phase range: every phase z_ij = W_j . x_i + b_j the assembly / eval kernels evaluate (b_j
 * including the amplitude/phase fold's shift, |psi| <= pi) must satisfy |z_ij| <= FLS_MAX_PHASE.
 * The kernels reduce z in half turns (z / pi - rint(z / pi)) exactly, but z itself carries the
 * rounding of W_j . x_i + b_j, so an entry's error grows like pi ulp(|z| / pi): <= ~4e-14 of its
 * term-magnitude scale at |z| <= 60 (the BASELINE configs), ~1e-12 at |z| ~ 2e3, ~5e-12 at the
 * limit.  Beyond it the call still completes but the next fls_sync (or fls_solve) returns
 * FLS_EUNSUPPORTED and the affected entries are unspecified.  The check is exact (|z| itself,
 * not a bound) and costs nothing on the entry path: a per-CTA bound ||W_j||_1 ||x_i||_inf +
 * |b_j| selects the rows that are re-checked. */
#define FLS_MAX_PHASE 1.0e4

typedef enum {
    FLS_OK = 0,
    FLS_EINVAL = 1,        /* bad argument (null pointer, size, dim / alpha mismatch, lda) */
    FLS_ENOMEM = 2,        /* device allocation failed */
    FLS_ECUDA = 3,         /* CUDA runtime error */
    FLS_ECUSOLVER = 4,     /* cuSOLVER / cuBLAS error */
    FLS_ENCCL = 5,         /* collective layer: NCCL unavailable / failed, host callback failed */
    FLS_ENONFINITE = 6,    /* NaN / Inf in an input (reported by fls_sync / fls_solve) */
    FLS_ERANK = 7,         /* exactly zero diagonal in R with no ridge */
    FLS_EUNSUPPORTED = 8   /* valid request this build does not implement */
} fls_status;

/* thread-local message describing the last non-FLS_OK return of this thread */
FLS_API const char *fls_last_error(void);
FLS_API const char *fls_status_string(fls_status s);
FLS_API int fls_api_version(void);

/* ---------------------------------------------------------------------------------------- */
/* context                                                                                  */
/* ---------------------------------------------------------------------------------------- */
typedef struct fls_ctx fls_ctx;

/* device: CUDA ordinal; cuda_stream: a cudaStream_t (borrowed, not destroyed), or NULL for
 * the legacy default stream.  *out receives the ctx.  Errors: FLS_EINVAL (out NULL, bad
 * device), FLS_ECUDA. */
FLS_API fls_status fls_ctx_create(int device, void *cuda_stream, fls_ctx **out);
/* frees the ctx workspace and library handles; NULL is a no-op. */
FLS_API fls_status fls_ctx_destroy(fls_ctx *ctx);
/* re-point the ctx at another stream (borrowed).  Work already enqueued on the old stream is
 * ordered before anything later enqueued on the new one (an event wait, no host sync), so the
 * ctx's workspace is never used by both streams at once.  Errors: FLS_EINVAL, FLS_ECUDA. */
FLS_API fls_status fls_ctx_set_stream(fls_ctx *ctx, void *cuda_stream);
/* block until the ctx stream is idle; returns FLS_ENONFINITE (and clears the flag) if a
 * kernel saw a non-finite input since the last check, FLS_EUNSUPPORTED if a phase exceeded
 * FLS_MAX_PHASE, FLS_ECUDA on an asynchronous fault. */
FLS_API fls_status fls_sync(fls_ctx *ctx);
/* measurement hook: with enable != 0 every assembly-kernel launch of fls_assemble is bracketed
 * by CUDA events on the ctx stream (the prefactor kernel is not included).  timing_read
 * synchronises the stream, returns the summed kernel milliseconds and the launch count since
 * the last enable / read (host outputs), and restarts the count. */
FLS_API fls_status fls_ctx_timing(fls_ctx *ctx, int32_t enable);
FLS_API fls_status fls_ctx_timing_read(fls_ctx *ctx, double *ms_total, int64_t *n_launches);

/* ---------------------------------------------------------------------------------------- */
/* operators as data: L = sum_t c_t(x) D^{alpha_t}   (P:L92 multi-index; "linear    */
/* PDE L[u] = f"; P:L402-403 variable coefficients)                                         */
/* ---------------------------------------------------------------------------------------- */
typedef struct {
    int32_t alpha[FLS_MAX_DIM];  /* derivative orders per axis; entries >= dim must be 0 */
    double coef;                 /* constant coefficient c_t */
    int32_t field;               /* -1: constant; g in [0, n_fields): c_t(x_i) = coef *
                                    coef_fields[i * n_fields + g] */
} fls_term;

typedef struct {
    int32_t dim;                 /* must equal the basis dim */
    int32_t n_terms;             /* 1 .. FLS_MAX_TERMS */
    const fls_term *terms;       /* host array of n_terms */
} fls_operator;

/* one row block of Eq. 3: its rows are  weight * L_blk[phi_j](x_i),  rhs  weight * values_i.
 * Dirichlet BC / IC blocks use the identity operator (one term, alpha = 0, coef = 1). */
typedef struct {
    const double *X;             /* device, n_points x dim, row-major */
    int64_t n_points;            /* >= 0; 0 = empty block */
    const fls_operator *op;      /* host */
    const double *coef_fields;   /* device, n_points x n_fields row-major, or NULL if n_fields=0 */
    int32_t n_fields;            /* 0 .. FLS_MAX_FIELDS */
    double weight;               /* 1 for PDE rows, lambda for BC / IC rows */
    const double *values;        /* device, n_points (f, g or h), or NULL: rhs rows = 0 */
} fls_block;

/* ---------------------------------------------------------------------------------------- */
/* Alg. 1 line 1: W_j ~ N(0, sigma^2 I_dim), b_j ~ U[0, 2 pi).              */
/* Counter-based and bit-reproducible: Philox4x64-10 keyed (seed, stream), raw output n is  */
/* word n%4 of the block at counter (n/4 + 1, 0, 0, 0); stream 1 feeds W through Box-Muller */
/* on uniform pairs (u = (raw >> 11) 2^-53; r = sqrt(-2 log(1-u1)), th = 2 pi u2; normal   */
/* 2m = r cos th, 2m+1 = r sin th; W[j][k] = sigma * normal[j*dim + k]); stream 2 feeds    */
/* b_j = 2 pi u_j.  (DESIGN.md §3 R1 -- the paper names no generator.)                     */
/*   W: device, n_features x dim row-major (written).  b: device, n_features (written).    */
/*   Errors: FLS_EINVAL for dim not in 1..FLS_MAX_DIM, n_features < 1, sigma <= 0 or not   */
/*   finite, NULL outputs.                                                                  */
/* ---------------------------------------------------------------------------------------- */
FLS_API fls_status fls_features(fls_ctx *ctx, int32_t dim, int64_t n_features, double sigma,
                        uint64_t seed, double *W, double *b);

/* Multi-block basis ("B blocks at potentially different bandwidths sigma_b,
 * concatenating all features"): block q holds block_features[q] consecutive features drawn
 * with sigmas[q]; the same Philox streams as fls_features, with W[j][k] =
 * sigma_{block(j)} * normal[j*dim + k] (n_blocks = 1 is exactly fls_features).
 *   block_features, sigmas: host arrays of n_blocks (1..FLS_MAX_FEAT_BLOCKS), each >= 1 / > 0.
 *   W: device, (sum block_features) x dim.  b: device, sum block_features. */
FLS_API fls_status fls_features_blocks(fls_ctx *ctx, int32_t dim, int32_t n_blocks,
                                       const int64_t *block_features, const double *sigmas,
                                       uint64_t seed, double *W, double *b);

/* Alg. 1 line 2 ("Sample collocation points"): seeded points in a box domain, same
 * Philox4x64-10 generator and uniform map as fls_features (u = (raw >> 11) 2^-53), stream
 * `stream` (convention: 3 interior, 4 boundary, 5 initial, 6 held-out test).
 *   fls_sample_box:   X[i][k] = lo_k + (hi_k - lo_k) * u(i*dim + k),  i < n.
 *   fls_sample_faces: for each axis k with bit k of axes_mask set, in increasing k, per_face
 *                     points on the face x_k = lo_k then per_face on x_k = hi_k, the other
 *                     coordinates as in fls_sample_box (point index = running output row).
 * lo, hi: host arrays of dim with lo_k < hi_k.  X: device, rows x dim (rows = n, or
 * 2 * per_face * popcount(axes_mask)).  Asynchronous.  Errors: FLS_EINVAL. */
FLS_API fls_status fls_sample_box(fls_ctx *ctx, int32_t dim, int64_t n, const double *lo,
                                  const double *hi, uint64_t seed, uint64_t stream, double *X);
FLS_API fls_status fls_sample_faces(fls_ctx *ctx, int32_t dim, int64_t per_face,
                                    uint32_t axes_mask, const double *lo, const double *hi,
                                    uint64_t seed, uint64_t stream, double *X);

#define FLS_COL_MAJOR 0   /* A[j * lda + i]: rows contiguous (what fls_solve consumes) */
#define FLS_ROW_MAJOR 1   /* A[i * lda + j]: features contiguous */

/* ---------------------------------------------------------------------------------------- */
/* Alg. 1 lines 3-5, Eq. 3 with Eq. 2:                    */
/*   A_ij = w_blk * s * sum_t c_t(x_i) (prod_k W_jk^alpha_tk) Phi_{|alpha_t| mod 4}(z_ij),   */
/*   z_ij = W_j . x_i + b_j,   s = 1/sqrt(n_features) if normalize else 1,                  */
/*   rhs_i = w_blk * values_i.                                                               */
/* The blocks are stacked in order (global row g runs over block 0's points, then block 1's */
/* ...).  This call writes the global rows [row_begin, row_end) -- one rank's shard -- to    */
/* local row (g - row_begin) of A, and of rhs if rhs != NULL.                               */
/*   W, b: device (fls_features layout).  dim: 1..FLS_MAX_DIM.  n_features >= 1.             */
/*   blocks: host array of n_blocks (>= 1) descriptors.                                      */
/*   0 <= row_begin <= row_end <= total rows.  row_begin == row_end is a no-op (FLS_OK).     */
/*   A: device; FLS_COL_MAJOR needs lda >= row_end - row_begin, FLS_ROW_MAJOR lda >=         */
/*   n_features.  Fastest when A is 16-byte aligned and lda is even (vector stores).        */
/*   rhs: device, row_end - row_begin doubles, or NULL.  For the solver's [A | b] layout pass */
/*   rhs = A + n_features * lda (column-major).                                              */
/*   Errors (host, before any launch): FLS_EINVAL for NULL pointers, sizes, layout, lda,     */
/*   op->dim != dim, alpha entries < 0 or set beyond dim, field >= n_fields, too many terms. */
/*   Non-finite inputs: FLS_ENONFINITE at the next fls_sync.                                 */
/* ---------------------------------------------------------------------------------------- */
FLS_API fls_status fls_assemble(fls_ctx *ctx, const double *W, const double *b, int32_t dim,
                        int64_t n_features, int32_t normalize, const fls_block *blocks,
                        int32_t n_blocks, int64_t row_begin, int64_t row_end, double *A,
                        int64_t lda, int32_t layout, double *rhs);

/* Alg. 1 lines 1 + 3-5 in one call: fls_features(ctx, dim, n_features, sigma, seed, W, b)
 * followed by fls_assemble(ctx, W, b, ...), with the feature draw and the per-block prefactor
 * fold fused into one kernel ahead of the assembly -- or, for column-major calls of at most
 * FLS_FUSE_MAX_ENTRIES local entries (environment, default 2^22), into the assembly kernel
 * itself (ONE launch: each CTA draws and folds its own features).  Consecutive calls on a
 * stream overlap (programmatic dependent launch: the next call's draws run while this call's
 * assembly finishes; every write still lands in stream order).  W and b are written
 * (bit-identical to fls_features) and must be device buffers of n_features x dim and
 * n_features.  Other arguments, errors and asynchrony as fls_assemble. */
FLS_API fls_status fls_features_assemble(fls_ctx *ctx, int32_t dim, int64_t n_features,
                                         double sigma, uint64_t seed, double *W, double *b,
                                         int32_t normalize, const fls_block *blocks,
                                         int32_t n_blocks, int64_t row_begin, int64_t row_end,
                                         double *A, int64_t lda, int32_t layout, double *rhs);

/* ---------------------------------------------------------------------------------------- */
/* fls_assemble with HOST buffers (the end-to-end path of a caller whose data lives in host  */
/* memory).  Same arguments and semantics as fls_assemble with FLS_COL_MAJOR, except that    */
/* W, b, every block's X / coef_fields / values, A and rhs are HOST pointers (pinned memory   */
/* gives full PCIe bandwidth; pageable works, slower).  The call copies W, b and the points   */
/* of [row_begin, row_end) to ctx-owned device staging, assembles in row chunks of at most    */
/* chunk_rows rows (0 = about 2 GiB per chunk) into two device buffers, and copies each chunk */
/* into A / rhs (cudaMemcpy2DAsync on a second stream) while the next chunk computes.        */
/* Blocking: on return A and rhs hold the result.  The ctx keeps the staging for reuse.       */
/*   Errors: as fls_assemble; FLS_ENOMEM if the staging does not fit.                        */
/* ---------------------------------------------------------------------------------------- */
FLS_API fls_status fls_assemble_host(fls_ctx *ctx, const double *W, const double *b, int32_t dim,
                                     int64_t n_features, int32_t normalize,
                                     const fls_block *blocks, int32_t n_blocks,
                                     int64_t row_begin, int64_t row_end, double *A, int64_t lda,
                                     double *rhs, int64_t chunk_rows);

/* ---------------------------------------------------------------------------------------- */
/* Alg. 1 line 5 ("beta* = argmin ||A beta - b||^2 via QR"), with the Tikhonov term  */
/* of P:L156-160:  beta = argmin ||A beta - b||^2 + mu ||beta||^2,  sqrt(mu) = ridge_rel *     */
/* ||A||_F (reading A16: ridge_rel = tau = 0 for C1-C4, 1e-10 for C5; ||A||_F over  */
/* the n_features columns of A, not b, and over ALL ranks' rows when a communicator is        */
/* attached).  Householder QR of the column-major [A | b] (n_rows x (n_features + 1), b as    */
/* column n_features), then R beta = (Q^T b)[0:n].                                            */
/*   Without a communicator (or one rank): a single QR; when sqrt(mu) > 0 the rows            */
/*   [sqrt(mu) I | 0] are written at rows n_rows .. n_rows + n_features - 1 of the same       */
/*   buffer, so lda >= n_rows + n_features is then required.                                  */
/*   With a communicator of P ranks (fls_comm_init / fls_comm_init_host): Ab holds THIS rank's */
/*   rows (n_rows may differ per rank, may be 0; lda >= n_rows), every rank calls fls_solve    */
/*   with the same n_features and ridge_rel, and the call runs TSQR: local QR, the R factors   */
/*   to rank 0 (peer-memory stores or NCCL, fls_comm_config), the root's structured QR of the  */
/*   stacked factors plus the ridge rows, trsv, and beta + the residual broadcast -- on return */
/*   beta and *resid_norm are identical on every rank.  A failure on any rank is returned on   */
/*   every rank (no rank is left waiting).                                                    */
/*   Ab: device, destroyed.  beta: device, n_features (written).                              */
/*   resid_norm: host, optional: ||A beta - b||_2 (+ ridge part) = |R[n, n]|.                 */
/*   Blocking.  Errors: FLS_EINVAL, FLS_ENOMEM, FLS_ECUSOLVER, FLS_ERANK (exact zero on the   */
/*   diagonal of R with mu = 0), FLS_ENONFINITE (pending from an earlier kernel), FLS_ENCCL,  */
/*   FLS_EUNSUPPORTED (forced P2P transport unavailable).                                     */
/* fls_solve_mu: the same with an ABSOLUTE sqrt(mu) >= 0 (the Newton step's mu = 1e-10,       */
/*   P:L158, L189).                                                                           */
/* ---------------------------------------------------------------------------------------- */
FLS_API fls_status fls_solve(fls_ctx *ctx, double *Ab, int64_t n_rows, int64_t lda, int64_t n_features,
                     double ridge_rel, double *beta, double *resid_norm);
FLS_API fls_status fls_solve_mu(fls_ctx *ctx, double *Ab, int64_t n_rows, int64_t lda,
                                int64_t n_features, double sqrt_mu, double *beta, double *resid_norm);

/* ---------------------------------------------------------------------------------------- */
/* Communicator for the multi-rank solve (row-sharded assembly needs no     */
/* collective; the least-squares solve of Alg. 1 line 5, has one exchange step,     */
/* TSQR).  One ctx per rank, one rank per GPU.  The communicator belongs to the ctx (freed by */
/* fls_comm_destroy or fls_ctx_destroy).                                                       */
/* fls_comm_unique_id: an NCCL unique id (host, FLS_COMM_ID_BYTES) -- rank 0 creates it and   */
/*   the caller distributes it to every rank by its own means (torch.distributed, MPI, file). */
/* fls_comm_init: NCCL communicator of nranks ranks on the ctx's device and stream; blocks    */
/*   until all ranks have called it.  NCCL is loaded at run time ("libnccl.so.2", or the path  */
/*   in FLS_NCCL_LIB): FLS_ENCCL when it cannot be loaded or the init fails.                   */
/* fls_comm_init_host: the control plane through caller callbacks instead of NCCL (the R      */
/*   factors then move only by peer memory, so the ranks' GPUs -- or ONE shared GPU, e.g. in  */
/*   tests -- must support CUDA IPC).  allgather(user, send, recv, bytes) must gather `bytes`  */
/*   host bytes from every rank into recv (nranks * bytes, rank r at offset r * bytes) and    */
/*   return 0; it is called from inside fls_solve on the calling thread.  *coll is copied;   */
/*   user must stay valid until the communicator is destroyed.                                 */
/* fls_comm_config: transport of the R factors -- FLS_TSQR_AUTO (peer memory if every rank    */
/*   can map the root's buffer, else NCCL), FLS_TSQR_P2P (peer memory only), FLS_TSQR_NCCL;   */
/*   force_tsqr != 0 runs the TSQR path even with one rank (tests).                            */
/* fls_comm_info: nranks / rank (0 / 0 without a communicator) and the transport the last     */
/*   solve used (0 none, FLS_TSQR_P2P, FLS_TSQR_NCCL).                                         */
/*   Errors: FLS_EINVAL (NULL, rank not in [0, nranks), ctx already has a communicator),      */
/*   FLS_ENCCL.                                                                                */
/* ---------------------------------------------------------------------------------------- */
#define FLS_COMM_ID_BYTES 128
#define FLS_TSQR_AUTO 0
#define FLS_TSQR_P2P 1
#define FLS_TSQR_NCCL 2
typedef struct {
    void *user;
    int32_t (*allgather)(void *user, const void *send, void *recv, int64_t bytes);
} fls_host_coll;
FLS_API fls_status fls_comm_unique_id(void *id);
FLS_API fls_status fls_comm_init(fls_ctx *ctx, const void *nccl_unique_id, int32_t nranks,
                                 int32_t rank);
FLS_API fls_status fls_comm_init_host(fls_ctx *ctx, int32_t nranks, int32_t rank,
                                      const fls_host_coll *coll);
FLS_API fls_status fls_comm_destroy(fls_ctx *ctx);
FLS_API fls_status fls_comm_config(fls_ctx *ctx, int32_t transport, int32_t force_tsqr);
FLS_API fls_status fls_comm_info(fls_ctx *ctx, int32_t *nranks, int32_t *rank,
                                 int32_t *last_transport);

/* ---------------------------------------------------------------------------------------- */
/* Learnable bandwidth (App. E): W_j = L W^_j with frozen W^_j ~ N(0, I) and a    */
/* learnable d x d factor L (scalar sigma: L = sigma I; anisotropic: lower-triangular        */
/* Cholesky factor).  The outer loss is  Lout = ||A(L) beta* - b||^2, beta* the     */
/* least-squares optimum; by optimality of beta* its gradient needs no differentiation of   */
/* the solve:  dLout/dL_kl = 2 sum_i r_i sum_j beta_j dA_ij/dW_jk W^_jl,  r = A beta* - b,    */
/* with dA_ij/dW_jk = w s sum_t c_t(x_i) [alpha_tk prod W^(alpha_t - e_k) Phi_p(z_ij)         */
/*                                   + prod W^alpha_t x_ik Phi_{p+1}(z_ij)]  (Eq. 2 + chain), */
/* c_t(x_i) = coef_t, times the block's coefficient field for field terms.                   */
/* fls_features_transform: W (F x dim) = rows L W^_j (L host, dim x dim row-major).          */
/* fls_bandwidth_grad: blocks as for fls_assemble (coefficient fields allowed) but values =  */
/*   the block's rows of r (device); G (host, dim x dim row-major) receives dLout/dL;        */
/*   deterministic; blocking.                                                                */
/* ---------------------------------------------------------------------------------------- */
FLS_API fls_status fls_features_transform(fls_ctx *ctx, int32_t dim, int64_t n_features,
                                          const double *L, const double *W_hat, double *W);
FLS_API fls_status fls_bandwidth_grad(fls_ctx *ctx, const double *W, const double *W_hat,
                                      const double *b, int32_t dim, int64_t n_features,
                                      int32_t normalize, const fls_block *blocks,
                                      int32_t n_blocks, const double *beta, double *G);

/* ---------------------------------------------------------------------------------------- */
/* Newton-Raphson support (Eq. 4-5): nonlinear PDE  L[u] + N(u) = f  with a      */
/* pointwise nonlinearity N.  The Jacobian  J_ij = L[phi_j](x_i) + N'(u(x_i)) s phi_j(x_i)  */
/* is fls_assemble with one extra identity term whose coefficient field is          */
/* dN = N'(u); this call produces that field and the Newton right-hand side.                 */
/*   kind FLS_NL_POLY: N(u) = sum_{k=0}^{degree} a[k] u^k  (u^3, Allen-Cahn, ...)             */
/*   kind FLS_NL_EXP:  N(u) = a[0] exp(a[1] u)            (Bratu: a = {lambda, 1})            */
/* For i < n:  neg_res_i = f_i - Lu_i - N(u_i)   (= -R_i, the rhs of J delta = -R),           */
/*             dN_i = N'(u_i)  (dN may be NULL).                                               */
/* stats (host, optional, blocking when given): {sum neg_res^2, sum u^2, sum (u - u_prev)^2}  */
/* (u_prev may be NULL -> third entry 0), a fixed-order deterministic reduction.              */
/* All arrays are device vectors of n doubles.                                                 */
/* ---------------------------------------------------------------------------------------- */
#define FLS_NL_POLY 1
#define FLS_NL_EXP 2
typedef struct {
    int32_t kind;     /* FLS_NL_POLY | FLS_NL_EXP */
    int32_t degree;   /* POLY: 0..7 */
    double a[8];
} fls_nonlinearity;
FLS_API fls_status fls_nl_residual(fls_ctx *ctx, const fls_nonlinearity *nl, int64_t n,
                                   const double *Lu, const double *u, const double *u_prev,
                                   const double *f, double *neg_res, double *dN, double *stats);
/* Quasi-linear nonlinearities that also depend on one derivative Du = D^e u of the solution
 * (steady Burgers u u_x): kind FLS_NL_UDU, N(u, Du) = a[0] u Du.  For i < n:
 *   neg_res_i = f_i - Lu_i - N(u_i, Du_i),  dN_du_i = dN/du,  dN_dDu_i = dN/dDu
 * (the Jacobian gets dN_du on the identity term and dN_dDu on the D^e term).
 * Du may be NULL for the pointwise kinds (then dN_dDu is not written).  stats as for
 * fls_nl_residual.  fls_nl_residual(...) == fls_nl_residual2(..., Du = NULL, dN_dDu = NULL). */
#define FLS_NL_UDU 3
FLS_API fls_status fls_nl_residual2(fls_ctx *ctx, const fls_nonlinearity *nl, int64_t n,
                                    const double *Lu, const double *u, const double *Du,
                                    const double *u_prev, const double *f, double *neg_res,
                                    double *dN_du, double *dN_dDu, double *stats);
/* out_i = y_i + alpha * x_i for i < n (the Newton update beta + alpha delta, Eq. 4).
 * Device vectors; out may alias y or x.  Asynchronous. */
FLS_API fls_status fls_axpy(fls_ctx *ctx, int64_t n, double alpha, const double *x,
                            const double *y, double *out);

/* ---------------------------------------------------------------------------------------- */
/* Cached / prefactored solves (App. I "Matrix caching": factor A once, then     */
/* every new right-hand side costs a cached apply; inverse problems P:L395-397).             */
/* fls_qr_factor copies the column-major A (n_rows x n_features, lda) into ctx-independent   */
/* device storage owned by the returned handle, appends [sqrt_mu I] rows when sqrt_mu > 0,   */
/* and runs Householder QR (fls_geqrf).  fls_qr_solve then computes, for each of nrhs columns of  */
/* B (n_rows x nrhs, ldb; the ridge rows' rhs are 0), beta = R^-1 (Q^T [b; 0])[0:n_features] */
/* (ormqr + trsm) into Beta (n_features x nrhs, ldbeta).  All device pointers; blocking.      */
/* The handle is immutable after factoring and may be used from any ctx on the same device.  */
/*   Errors: FLS_EINVAL (sizes, NULL), FLS_ENOMEM, FLS_ECUSOLVER, FLS_ERANK (zero diagonal,   */
/*   sqrt_mu = 0; reported by fls_qr_factor).                                                 */
/* ---------------------------------------------------------------------------------------- */
typedef struct fls_qr fls_qr;
FLS_API fls_status fls_qr_factor(fls_ctx *ctx, const double *A, int64_t n_rows, int64_t lda,
                                 int64_t n_features, double sqrt_mu, fls_qr **out);
FLS_API fls_status fls_qr_solve(fls_ctx *ctx, const fls_qr *qr, const double *B, int64_t ldb,
                                int64_t nrhs, double *Beta, int64_t ldbeta);
FLS_API fls_status fls_qr_destroy(fls_qr *qr);

/* TSQR root step (P:L124 solve of the stacked factors): S holds n_blocks upper-triangular or
 * -trapezoidal factors [R_r | c_r] in block order -- block r = rows [r kb, (r+1) kb) of the
 * column-major S (lds >= n_blocks kb, n_features + 1 columns), zero-padded to kb rows -- and
 * the solve appends [sqrt_mu I | 0] rows when sqrt_mu > 0, then returns beta (device,
 * n_features) and |R(F, F)| (host, may be NULL) exactly as fls_solve on the stacked matrix.
 * The triangular structure is exploited: the rows are permuted (block 0, then row i of every
 * other block and of the ridge, for i = 0, 1, ...) so that for the columns [j, j + w) only the
 * first kb + G (j + w) rows can be nonzero, and the blocked QR stops each panel there (about
 * half the flops of a dense QR of the stack at P = 8).  S is not modified.  Blocking.
 *   Errors: FLS_EINVAL (sizes, NULL, underdetermined), FLS_ENOMEM, FLS_ECUSOLVER, FLS_ERANK. */
FLS_API fls_status fls_solve_stacked(fls_ctx *ctx, const double *S, int32_t n_blocks, int64_t kb,
                                     int64_t lds, int64_t n_features, double sqrt_mu, double *beta,
                                     double *resid_norm);

/* TSQR building block:Householder QR of the local column-major block M (n_rows x n_cols,
 * destroyed) and copy of its upper-trapezoidal R (min(n_rows, n_cols) x n_cols, zeros below
 * the diagonal) into R (device, column-major, ldr >= min(n_rows, n_cols)).  Blocking. */
FLS_API fls_status fls_qr_r(fls_ctx *ctx, double *M, int64_t n_rows, int64_t lda, int64_t n_cols,
                    double *R, int64_t ldr);

/* Householder QR of the column-major block M (n_rows x n_cols, lda) in place, in LAPACK /
 * cuSOLVER geqrf format: R in the upper trapezoid, the Householder vectors v_j (v_jj = 1
 * implicit) below the diagonal, tau (device, min(n_rows, n_cols) doubles), H_j = I - tau_j
 * v_j v_j^T, Q = H_1 ... H_k.  This is the factorisation fls_solve / fls_qr_factor / fls_qr_r
 * run (Alg. 1 line 5): libfls's blocked QR (nb-column compact-WY panels factored
 * recursively on cuBLAS DGEMM, <= 32-column leaves in one cooperative kernel per leaf) for
 * n_cols >= 1024, a single cusolverDnDgeqrf call for narrower blocks; the environment
 * variable FLS_QR=blocked / FLS_QR=cusolver forces one of the two (read at every call).
 *   Errors: FLS_EINVAL (sizes, NULL), FLS_EUNSUPPORTED (a dimension > INT32_MAX), FLS_ENOMEM,
 *   FLS_ECUSOLVER (cuBLAS failure).  Blocking. */
FLS_API fls_status fls_geqrf(fls_ctx *ctx, double *M, int64_t n_rows, int64_t lda, int64_t n_cols,
                             double *tau);

/* CUDA IPC building blocks (fls_solve with a communicator runs its own exchange internally;    */
/* these serve callers that orchestrate one themselves).  Peer memory (NVLink / NVSwitch): the root exports its
 * stacking buffer, every rank maps it and fls_qr_r writes its R factor straight into the
 * root's memory (the R-extraction kernel's stores ARE the transfer; no staging, no NCCL
 * gather).  fls_ipc_handle: handle (host, FLS_IPC_HANDLE_BYTES) of the allocation that
 * CONTAINS dev_ptr, and *offset = dev_ptr - that allocation's base (caching allocators
 * sub-allocate).  fls_ipc_open maps a handle exported by ANOTHER process (same or peer
 * device) and returns the allocation's base in this process (add the offset);
 * fls_ipc_close unmaps it.  Errors: FLS_EINVAL (NULL), FLS_ECUDA (CUDA IPC failure, e.g.
 * no peer access). */
#define FLS_IPC_HANDLE_BYTES 64
FLS_API fls_status fls_ipc_handle(fls_ctx *ctx, void *dev_ptr, void *handle, int64_t *offset);
FLS_API fls_status fls_ipc_open(fls_ctx *ctx, const void *handle, void **dev_ptr);
FLS_API fls_status fls_ipc_close(fls_ctx *ctx, void *dev_ptr);

/* sum of squares of the n_rows x n_cols column-major block (for ||A||_F^2).  out: host.
 * Blocking. */
FLS_API fls_status fls_frob2(fls_ctx *ctx, const double *A, int64_t n_rows, int64_t lda, int64_t n_cols,
                     double *out);

/* ---------------------------------------------------------------------------------------- */
/* Alg. 1 line 6, Eq. 1:  out_i = s * sum_j beta_j sin(W_j . x_i + b_j),    */
/* or with op != NULL,  out_i = L[u_N](x_i) = sum_j beta_j A_ij  (the PDE residual check of   */
/* P:L191).  A is never materialised.  op may not use coefficient fields (FLS_EINVAL).        */
/*   X: device, n_points x dim.  out: device, n_points.  Asynchronous.                       */
/* ---------------------------------------------------------------------------------------- */
FLS_API fls_status fls_eval(fls_ctx *ctx, const double *W, const double *b, int32_t dim,
                    int64_t n_features, int32_t normalize, const double *beta,
                    const fls_operator *op, const double *X, int64_t n_points, double *out);

/* out_i = sum_j A_ij beta_j for the rows of one row block, with A_ij exactly as fls_assemble
 * defines them (s, the block weight, its operator including coefficient fields, Eq. 2 / Eq. 3,
 * P:L95-121) -- i.e. A_block beta without materialising A (PDE residuals of variable-
 * coefficient operators such as C5's, Newton residuals).  block->values is ignored.
 *   block: host descriptor of device arrays (X n_points x dim, coef_fields n_points x
 *   n_fields).  out: device, n_points.  Errors as fls_eval (FLS_EINVAL also for a field id
 *   >= n_fields or fields used with coef_fields NULL).  Asynchronous. */
FLS_API fls_status fls_eval_block(fls_ctx *ctx, const double *W, const double *b, int32_t dim,
                                  int64_t n_features, int32_t normalize, const double *beta,
                                  const fls_block *block, double *out);

#ifdef __cplusplus
}
#endif
#endif /* FLS_H_ */
