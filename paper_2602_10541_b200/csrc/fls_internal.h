// fls_internal.h -- host-side internals of libfls (ctx, errors, kernel launch interfaces).
#pragma once
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fls.h"

namespace fls {

// per-feature parameter layouts produced by the prefactor kernel
enum PrefMode : int32_t {
  PM_SIN = 0,      // A = (P_0 + sum_g c_g P_g) sin z
  PM_COSSHIFT = 1, // all terms odd: cos z = sin(z + pi/2) -> b' += 1/2, P_g = Pc_g
  PM_FOLD = 2,     // constant coefficients, mixed parity: Ps sin z + Pc cos z = rho sin(z + psi)
  PM_SINCOS = 3    // general: (Ps_0 + sum c_g Ps_g) sin z + (Pc_0 + sum c_g Pc_g) cos z
};

// kernel families
enum KMode : int32_t { KM_SIN = 0, KM_SINCOS = 1 };

// column-major assembly tiling (compile-time; -D overrides are for tuning sweeps only)
#ifndef FLS_PAIRS
#define FLS_PAIRS 2
#endif
#ifndef FLS_FUNROLL
#define FLS_FUNROLL 2
#endif
#ifndef FLS_NT
#define FLS_NT 256
#endif
#ifndef FLS_QUAD
#define FLS_QUAD 0  // 1: 4 consecutive rows per thread, one 32-byte store per feature
#endif
constexpr bool kQuad = FLS_QUAD != 0 && FLS_PAIRS == 2;
constexpr int kRowAlign = kQuad ? 4 : 2;    // rows per thread-contiguous store
constexpr int kNT = FLS_NT;                 // threads per CTA
constexpr int kPairs = FLS_PAIRS;           // 16-byte row pairs per thread
constexpr int kFUnroll = FLS_FUNROLL;       // features per loop iteration
constexpr int kRowsCTA = 2 * kPairs * kNT;  // rows per CTA tile
constexpr int kFC = 128;                    // features per shared-memory chunk

constexpr int kMaxFac = 22;  // factor list length kept per term (orders up to 22)
struct TermDev {
  double coef;
  int8_t alpha[FLS_MAX_DIM];
  int8_t group;  // 0 = constant coefficient, 1..G = compacted field groups
  int8_t nfac;   // |alpha| if <= kMaxFac, else -1
  int8_t fac[kMaxFac];  // alpha expanded in axis order: the axis of each factor of prod W^alpha
};
static_assert(sizeof(TermDev) == 40, "TermDev layout");

struct PrefArgs {
  const double *W;
  const double *b;
  int64_t F;
  int32_t D;
  int32_t n_terms;
  int32_t G;      // number of field groups
  int32_t pmode;  // PrefMode
  int32_t S;      // doubles per feature in pf
  double scale;   // s * weight
  double *pf;
  unsigned *err;
  TermDev terms[FLS_MAX_TERMS];
};

struct AsmArgs {
  const double *pf;
  int64_t F;
  const double *X;
  const double *fields;
  const double *values;
  double weight;
  int64_t pt0;  // point index of local row lr0
  int64_t lr0, lr1;
  double *A;
  int64_t lda;
  double *rhs;
  unsigned *err;
  int32_t nf;                    // n_fields of the block (row stride of fields)
  int32_t vec;                   // 16-byte vector stores allowed
  int64_t fpc;                   // features per CTA (set by the launcher)
  int64_t batch_span;            // rows of all blocks in this launch (set by the launcher)
  int32_t gfield[FLS_MAX_FIELDS];// field id of group g+1
  int64_t f_begin, f_end;        // feature range of this launch segment (set by the launcher)
  int32_t pre_idx;               // the segment's row block within the launch (fused fold args)
};

struct EvalArgs {
  const double *pf;  // PM_SINCOS layout: [W'_0..W'_{D-1}, b', Ps_0, Pc_0, .., Ps_G, Pc_G] (+pad)
  int32_t S;
  int64_t F;
  const double *beta;
  const double *X;
  int64_t n;
  double *out;
  unsigned *err;
  const double *fields;           // n x nf coefficient fields (G > 0), row-major
  int32_t nf;
  int32_t G;                      // field groups (0: constant coefficients)
  int32_t gfield[FLS_MAX_FIELDS]; // field id of group g+1
  int32_t sin_only;               // every term of even order: Pc = 0, skip the cos polynomial
};

// layout helper shared by host and kernels
__host__ __device__ constexpr int pf_stride(int D, int G, int kmode) {
  return (D + 1 + (G + 1) * (kmode == KM_SINCOS ? 2 : 1) + 1) & ~1;
}

// launchers (fls_kernels.cu / fls_assemble_*.cu)
struct FeatBlocks {  // multi-block bandwidths; n = 1 is the plain basis
  int32_t n;
  int64_t ends[FLS_MAX_FEAT_BLOCKS];
  double sigma[FLS_MAX_FEAT_BLOCKS];
};
cudaError_t launch_features(int32_t dim, int64_t F, const FeatBlocks &fb, uint64_t seed, double *W,
                            double *b, cudaStream_t st);
struct SampleArgs {
  int32_t D;
  int64_t rows;
  double lo[FLS_MAX_DIM], hi[FLS_MAX_DIM];
  uint64_t seed, stream;
  int64_t per_face;                  // 0: box interior
  int32_t face_axis[FLS_MAX_DIM];    // axis of face pair f/2
  double *X;
};
cudaError_t launch_sample(const SampleArgs &a, cudaStream_t st);
// several row blocks sharing a kernel variant in one launch
constexpr int kMaxBatch = 4;
// a launch's segments: each row block's feature range split into a main part and a tail of
// narrower CTAs dispatched last (asm_plan)
constexpr int kMaxSeg = 2 * kMaxBatch;
struct AsmBatch {
  int32_t n;
  int64_t cta_end[kMaxSeg];  // prefix sums of the segments' CTA counts
  int64_t rt[kMaxSeg];       // row tiles per segment
  AsmArgs blk[kMaxSeg];
};
struct PrefBatch {
  int32_t n;
  PrefArgs blk[kMaxBatch];
};

// single-launch a1 + a2-a8 (fls_features_assemble on small problems): every assembly CTA
// draws W_j, b_j of its own features and folds their records in its prologue (bit-identical to
// features_prefactor_kernel); the CTAs of row tile 0 of the first block also write W and b
struct FusedBatch {
  FeatBlocks fb;
  uint64_t seed;
  double *W, *b;
  int32_t write_wb;             // this launch writes W, b (the first launch of the call)
  PrefArgs pre[kMaxBatch];      // fold arguments of each block of the batch
};
// variants with a fused instantiation (launch_assemble_cm_fused returns cudaErrorNotSupported
// for the others)
inline bool fused_variant(int D, int G, int kmode) { return kmode == KM_SIN && G <= 1 && D >= 1 && D <= FLS_MAX_DIM; }
cudaError_t launch_assemble_cm_fused(int D, int G, AsmArgs *blks, int n, const FusedBatch &fz,
                                     cudaStream_t st, bool pdl);

cudaError_t launch_prefactor(const PrefArgs &a, cudaStream_t st);
cudaError_t launch_prefactor_batch(const PrefBatch &b, int64_t F, cudaStream_t st);
// pdl: launch behind the previous kernel with programmatic dependent launch (the kernel writes
// nothing before griddepcontrol.wait, so it may overlap whatever precedes it on the stream)
cudaError_t launch_features_prefactor(int32_t dim, int64_t F, const FeatBlocks &fb, uint64_t seed,
                                      double *W, double *b, const PrefBatch &pb, cudaStream_t st,
                                      bool pdl);
// blks: n (<= kMaxBatch) blocks of one variant; fpc is set per block by the launcher
// pdl: launch with programmatic dependent launch (only right after this call's prefactor launch)
cudaError_t launch_assemble_cm(int D, int G, int kmode, AsmArgs *blks, int n, cudaStream_t st,
                               bool pdl);
cudaError_t launch_assemble_rm(int D, int G, int kmode, const AsmArgs &a, cudaStream_t st);
cudaError_t launch_eval(int D, const EvalArgs &a, cudaStream_t st);
cudaError_t launch_ridge_fill(double *Ab, int64_t lda, int64_t row0, int64_t F, int64_t ncols,
                              double sqrt_mu,
                              cudaStream_t st);
// R (rows_out x n, ldr) = upper trapezoid of M's first k rows, zeros below (rows_out >= k);
// upper_only: store only the trapezoid (R pre-zeroed, e.g. a peer's buffer: half the traffic)
cudaError_t launch_copy_upper(const double *M, int64_t lda, int64_t k, int64_t n, double *R,
                              int64_t ldr, cudaStream_t st, int64_t rows_out = -1,
                              bool upper_only = false);
cudaError_t launch_min_abs_diag(const double *M, int64_t lda, int64_t n, double *out,
                                cudaStream_t st);
struct NlArgs {
  int32_t kind, degree;
  double c[8];
  int64_t n;
  const double *Lu, *u, *u_prev, *f;
  double *neg_res, *dN, *partials;
  unsigned *err;
  const double *Du;  // FLS_NL_UDU: the derivative D^e u
  double *dN2;       // FLS_NL_UDU: dN/dDu
};
cudaError_t launch_nl_residual(const NlArgs &a, int nblk, double *stats, cudaStream_t st);

// learnable bandwidth (fls_bandwidth.cu)
struct TransformArgs {
  double L[FLS_MAX_DIM * FLS_MAX_DIM];
};
// gradient record per feature: [W/pi (D), b/pi, then per field group g = 0..G: Ps (D), Pc (D),
// Qs, Qc]; stride bound for D = FLS_MAX_DIM, G = FLS_MAX_FIELDS
__host__ __device__ constexpr int grad_stride(int D, int G) { return D + 1 + (G + 1) * (2 * D + 2); }
constexpr int kGradRec = grad_stride(FLS_MAX_DIM, FLS_MAX_FIELDS);
struct GradArgs {
  const double *pf;
  int32_t S;
  int64_t F;
  const double *X;
  const double *r;
  const double *fields;            // n x nf coefficient fields (G > 0)
  int32_t nf;
  int32_t gfield[FLS_MAX_FIELDS];  // field id of group g+1
  int64_t row0, row1, rows_per_slot;
  int32_t slot0;
  double *partials;
  unsigned *err;
};
cudaError_t launch_transform(int32_t D, int64_t F, const TransformArgs &t, const double *Wh,
                             double *W, cudaStream_t st);
cudaError_t launch_grad_prefactor(const PrefArgs &a, cudaStream_t st);
cudaError_t launch_grad_reduce(int D, int G, const GradArgs &a, int slots, cudaStream_t st);
cudaError_t launch_grad_final(int D, int64_t F, int nslots, const double *partials,
                              const double *beta, const double *Wh, double *G, cudaStream_t st);
cudaError_t launch_axpy(int64_t n, double alpha, const double *x, const double *y, double *out,
                        cudaStream_t st);
cudaError_t launch_frob2(const double *A, int64_t lda, int64_t m, int64_t n, double *partials,
                         int nblk, double *out, cudaStream_t st);

// blocked Householder QR (fls_qr.cu), geqrf output format; nullptr or a failure message
const char *qr_blocked(cublasHandle_t h, cudaStream_t st, double *A, int64_t m, int64_t n,
                       int64_t lda, double *tau, double *ws, cudaError_t *cerr,
                       cublasStatus_t *berr, int64_t grp_base = 0, int64_t grp_size = 0);
cudaError_t launch_stack_permute(const double *S, int64_t bs, int64_t cs, int32_t P, int64_t kb,
                                 int64_t F, double sqrt_mu, int64_t gq, int64_t m_total, int64_t n,
                                 double *M, int64_t ldm, cudaStream_t st);
size_t qr_blocked_ws(int64_t m, int64_t n);  // doubles of ws (incl. nothing for tau)
int qr_panel_width(int64_t n);
int64_t qr_blocked_max_rows();  // taller blocks use cusolverDnDgeqrf

}  // namespace fls
