/*
 * oracle.c -- CPU ORACLE for the Fast-LSQ operator-assembly hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2602_10541_b200/csrc/); neither side includes or links the other.
 *
 * Everything here is the plain definition written out, in fp64, slow on
 * purpose.  Built with  gcc -O2 -ffp-contract=off -fopenmp  (no contraction,
 * no intrinsics); OpenMP only splits independent rows / columns.
 *
 * Paper = /root/reference/PAPER.md (arxiv 2602.10541), cited "P:L<line>".
 *
 *   orc_philox4x64      Philox4x64-10 block (counter-based RNG, DESIGN.md §3 R1)
 *   orc_features        W_j ~ N(0, sigma^2 I), b_j ~ U[0, 2pi)      P:L82, Alg.1 l.1
 *   orc_diff            symbolic D^alpha of sin(W.x+b), one derivative
 *                       at a time: chain rule + the cycle
 *                       sin -> cos -> -sin -> -cos                  P:L93-97 (Eq.2), P:L706-718 (App.F)
 *   orc_assemble        A_ij = L[phi_j](x_i), term by term, then the
 *                       weighted row blocks [A_pde; lam A_bc; ...]
 *                       and rhs [f; lam g; ...]                     P:L118-124 (Eq.3), Alg.1 l.3-5
 *   orc_assemble_truth  the same definition in long double (tiny inputs: the
 *                       near-exact reference both fp64 paths are measured against)
 *   orc_lstsq           argmin ||A beta - b||^2 + mu ||beta||^2 by
 *                       unblocked Householder QR of [A | b] with
 *                       sqrt(mu) I rows appended (GVL Alg. 5.2.1),
 *                       then back substitution                     P:L124 ("via QR"), P:L156-160 (Tikhonov)
 *   orc_eval            u_N(x) = (1/sqrt N) sum_j beta_j sin(W_j.x+b_j)
 *                       (or L[u_N](x) through orc_assemble rows)   P:L77-82 (Eq.1), Alg.1 l.6
 *   orc_features_blocks multi-block bandwidths
 *   orc_sample_box/faces seeded collocation points                 Alg.1 l.2
 *   orc_lstsq_mu        the Tikhonov solve with an absolute sqrt(mu) P:L158 (Newton step)
 * Newton (oracle/newton.py) and learnable bandwidth (oracle/learnable.py) are Python on top.
 *
 * Parity pins for every function: tests/test_oracle_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAX_DIM 8

/* ------------------------------------------------------------------------- */
/* Philox4x64-10 (Salmon et al., SC'11).  raw(n) of stream (seed, stream_id)  */
/* is word n%4 of the block computed at counter (n/4 + 1, 0, 0, 0) with key   */
/* (seed, stream_id) -- the convention of numpy.random.Philox, which pins it. */
/* ------------------------------------------------------------------------- */
static void mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
    unsigned __int128 p = (unsigned __int128)a * (unsigned __int128)b;
    *hi = (uint64_t)(p >> 64);
    *lo = (uint64_t)p;
}

void orc_philox4x64(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
    uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint64_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo64(0xD2E7470EE14C6C93ULL, c0, &hi0, &lo0);
        mulhilo64(0xCA5A826395121157ULL, c2, &hi1, &lo1);
        uint64_t n0 = hi1 ^ c1 ^ k0;
        uint64_t n1 = lo1;
        uint64_t n2 = hi0 ^ c3 ^ k1;
        uint64_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B97F4A7C15ULL;
        k1 += 0xBB67AE8584CAA73BULL;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static uint64_t raw64(uint64_t seed, uint64_t stream, uint64_t n) {
    uint64_t ctr[4] = {n / 4 + 1, 0, 0, 0};
    uint64_t key[2] = {seed, stream};
    uint64_t out[4];
    orc_philox4x64(ctr, key, out);
    return out[n % 4];
}

/* u = (raw >> 11) * 2^-53 in [0, 1) */
static double uniform01(uint64_t seed, uint64_t stream, uint64_t n) {
    return (double)(raw64(seed, stream, n) >> 11) * (1.0 / 9007199254740992.0);
}

void orc_raw_stream(uint64_t seed, uint64_t stream, uint64_t n0, int64_t count, uint64_t *out) {
    for (int64_t i = 0; i < count; ++i) out[i] = raw64(seed, stream, n0 + (uint64_t)i);
}

/*
 * Alg. 1 line 1: "Sample frozen weights W_j ~ N(0, sigma^2 I_d), b_j ~ U(0, 2 pi)".
 * Stream 1 -> W (Box-Muller on consecutive uniform pairs, normal index j*dim + k),
 * stream 2 -> b.  DESIGN.md §3 R1 states this recipe; the paper names no RNG.
 */
int orc_features(int dim, int64_t n_features, double sigma, uint64_t seed, double *W, double *b) {
    const double two_pi = 6.283185307179586476925286766559;
    int64_t n_norm = n_features * (int64_t)dim;
    for (int64_t m = 0; 2 * m < n_norm; ++m) {
        double u1 = uniform01(seed, 1, (uint64_t)(2 * m));
        double u2 = uniform01(seed, 1, (uint64_t)(2 * m + 1));
        double rad = sqrt(-2.0 * log(1.0 - u1));
        double th = two_pi * u2;
        double g0 = rad * cos(th);
        double g1 = rad * sin(th);
        W[2 * m] = sigma * g0;
        if (2 * m + 1 < n_norm) W[2 * m + 1] = sigma * g1;
    }
    for (int64_t j = 0; j < n_features; ++j) b[j] = two_pi * uniform01(seed, 2, (uint64_t)j);
    return 0;
}

/*
 * Multi-block basis ("B blocks at potentially different bandwidths sigma_b,
 * concatenating all features"): the same streams as orc_features; feature j of block q
 * (counts[0] + ... + counts[q-1] <= j < ... + counts[q]) gets W_j = sigmas[q] * normals.
 */
int orc_features_blocks(int dim, int n_blocks, const int64_t *counts, const double *sigmas,
                        uint64_t seed, double *W, double *b) {
    const double two_pi = 6.283185307179586476925286766559;
    int64_t F = 0;
    for (int q = 0; q < n_blocks; ++q) F += counts[q];
    int64_t n_norm = F * (int64_t)dim;
    for (int64_t m = 0; m < n_norm; ++m) {
        int64_t pair = m / 2;
        double u1 = uniform01(seed, 1, (uint64_t)(2 * pair));
        double u2 = uniform01(seed, 1, (uint64_t)(2 * pair + 1));
        double rad = sqrt(-2.0 * log(1.0 - u1));
        double th = two_pi * u2;
        double g = (m % 2 == 0) ? rad * cos(th) : rad * sin(th);
        int64_t j = m / dim, end = 0;
        int q = 0;
        for (q = 0; q < n_blocks; ++q) {
            end += counts[q];
            if (j < end) break;
        }
        W[m] = sigmas[q] * g;
    }
    for (int64_t j = 0; j < F; ++j) b[j] = two_pi * uniform01(seed, 2, (uint64_t)j);
    return 0;
}

/*
 * Alg. 1 line 2: seeded collocation points in a box (R1 streams).
 * Coordinate n of the row-major output uses raw word n of the stream: x = lo + (hi - lo) u.
 * Faces: for each axis k in axes_mask (increasing), per_face points on x_k = lo_k, then
 * per_face on x_k = hi_k; the face coordinate replaces the drawn one.
 */
int orc_sample_box(int dim, int64_t n, const double *lo, const double *hi, uint64_t seed,
                   uint64_t stream, double *X) {
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < dim; ++k) {
            double u = uniform01(seed, stream, (uint64_t)(i * dim + k));
            X[i * dim + k] = lo[k] + (hi[k] - lo[k]) * u;
        }
    return 0;
}

int orc_sample_faces(int dim, int64_t per_face, uint32_t axes_mask, const double *lo,
                     const double *hi, uint64_t seed, uint64_t stream, double *X) {
    int64_t row = 0;
    for (int k = 0; k < dim; ++k) {
        if (!(axes_mask & (1u << k))) continue;
        for (int side = 0; side < 2; ++side)
            for (int64_t p = 0; p < per_face; ++p, ++row)
                for (int l = 0; l < dim; ++l) {
                    double u = uniform01(seed, stream, (uint64_t)(row * dim + l));
                    double v = lo[l] + (hi[l] - lo[l]) * u;
                    if (l == k) v = side ? hi[k] : lo[k];
                    X[row * dim + l] = v;
                }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Symbolic differentiation of  c * Phi_p(W.x + b) * prod_k W_k^{e_k}.        */
/* State (e, p); Phi_0 = sin, Phi_1 = cos, Phi_2 = -sin, Phi_3 = -cos.        */
/* d/dx_k: chain rule pulls out W_k (e_k += 1) and the derivative moves one  */
/* step along the cycle (p += 1 mod 4).  P:L95-97.                */
/* Applied one derivative at a time (never the |alpha| mod 4 shortcut).      */
/* ------------------------------------------------------------------------- */
void orc_diff(int dim, const int32_t *alpha, int32_t *e_out, int32_t *p_out) {
    int32_t e[ORC_MAX_DIM];
    int32_t p = 0;                       /* start: sin(z) = Phi_0 */
    for (int k = 0; k < dim; ++k) e[k] = 0;
    for (int k = 0; k < dim; ++k) {
        for (int32_t n = 0; n < alpha[k]; ++n) {
            e[k] += 1;                   /* chain rule: d z / d x_k = W_k */
            p = (p + 1) % 4;             /* d/dz Phi_p = Phi_{p+1} */
        }
    }
    for (int k = 0; k < dim; ++k) e_out[k] = e[k];
    *p_out = p;
}

/* Phi_p(z): the four-element cycle */
static double Phi(int32_t p, double z) {
    switch (p) {
        case 0: return sin(z);
        case 1: return cos(z);
        case 2: return -sin(z);
        default: return -cos(z);
    }
}

typedef struct {
    int32_t alpha[ORC_MAX_DIM];
    double coef;
    int32_t field;          /* -1: constant coefficient; g >= 0: coef * coef_fields[i*n_fields + g] */
} orc_term;

typedef struct {
    const double *X;        /* n_points x dim, row-major */
    int64_t n_points;
    const orc_term *terms;
    int32_t n_terms;
    const double *coef_fields;  /* n_points x n_fields or NULL */
    int32_t n_fields;
    double weight;          /* 1 for PDE rows, lambda for BC / IC rows */
    const double *values;   /* f / g / h at the points, or NULL (rhs row = 0) */
} orc_block;

/*
 * A[r][j] for the global stacked row ids rows[r] (blocks in order: pde, bc, ic, ...),
 *   A_ij = w_blk * s * sum_t c_t(x_i) * (prod_k W_jk^{e_tk}) * Phi_{p_t}(z_ij),
 *   z_ij = sum_k W_jk x_ik + b_j,  s = 1/sqrt(F) if normalize else 1  (Eq.1).
 * rhs[r] = w_blk * values_i.  scale[r][j] (optional) is the sum of absolute term
 * magnitudes  w_blk * s * sum_t |c_t(x_i)| |prod_k W_jk^{e_tk}|  used by the A14 parity metric.
 * Returns 0, or -1 on a bad row id, -2 on |z| >= 1e5 (reading A15).
 */
int orc_assemble(int dim, int64_t n_features, const double *W, const double *b, int normalize,
                 const orc_block *blocks, int n_blocks, const int64_t *rows, int64_t n_rows,
                 double *A, double *rhs, double *scale) {
    const double s = normalize ? 1.0 / sqrt((double)n_features) : 1.0;
    int64_t total = 0;
    for (int q = 0; q < n_blocks; ++q) total += blocks[q].n_points;
    int status = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(min : status)
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t g = rows[r];
        if (g < 0 || g >= total) { status = -1; continue; }
        int q = 0;
        int64_t i = g;
        while (i >= blocks[q].n_points) { i -= blocks[q].n_points; ++q; }
        const orc_block *B = &blocks[q];
        const double *x = B->X + i * dim;
        if (rhs) rhs[r] = B->values ? B->weight * B->values[i] : 0.0;
        for (int64_t j = 0; j < n_features; ++j) {
            const double *w = W + j * dim;
            double z = 0.0;
            for (int k = 0; k < dim; ++k) z = z + w[k] * x[k];
            z = z + b[j];
            if (!(fabs(z) < 1e5) && status > -2) status = -2;
            double acc = 0.0, mag = 0.0;
            for (int t = 0; t < B->n_terms; ++t) {
                const orc_term *T = &B->terms[t];
                int32_t e[ORC_MAX_DIM], p;
                orc_diff(dim, T->alpha, e, &p);
                double mono = 1.0;
                for (int k = 0; k < dim; ++k)
                    for (int32_t n = 0; n < e[k]; ++n) mono = mono * w[k];
                double c = T->coef;
                if (T->field >= 0) c = c * B->coef_fields[i * B->n_fields + T->field];
                acc = acc + c * mono * Phi(p, z);
                mag = mag + fabs(c) * fabs(mono);
            }
            A[r * n_features + j] = B->weight * (s * acc);
            if (scale) scale[r * n_features + j] = fabs(B->weight) * (s * mag);
        }
    }
    return status;
}

/*
 * "Truth" mode for tiny inputs: orc_assemble's definition, same term-by-term
 * order, carried out in long double (x87 80-bit: 64-bit significand, unit roundoff 5.4e-20) with
 * sinl / cosl, rounded to double only at the end.  Measures how far the fp64 oracle AND the GPU
 * path sit from near-exact values (tests/test_oracle_pins.py, tests/test_gpu_parity.py); pinned
 * itself to mpmath's numerical derivatives of sin(W.x + b) at 40 digits.
 */
static long double Phi_l(int32_t p, long double z) {
    switch (p) {
        case 0: return sinl(z);
        case 1: return cosl(z);
        case 2: return -sinl(z);
        default: return -cosl(z);
    }
}

int orc_assemble_truth(int dim, int64_t n_features, const double *W, const double *b, int normalize,
                       const orc_block *blocks, int n_blocks, const int64_t *rows, int64_t n_rows,
                       double *A) {
    const long double s = normalize ? 1.0L / sqrtl((long double)n_features) : 1.0L;
    int64_t total = 0;
    for (int q = 0; q < n_blocks; ++q) total += blocks[q].n_points;
    for (int64_t r = 0; r < n_rows; ++r) {
        int64_t g = rows[r];
        if (g < 0 || g >= total) return -1;
        int q = 0;
        int64_t i = g;
        while (i >= blocks[q].n_points) { i -= blocks[q].n_points; ++q; }
        const orc_block *B = &blocks[q];
        const double *x = B->X + i * dim;
        for (int64_t j = 0; j < n_features; ++j) {
            const double *w = W + j * dim;
            long double z = 0.0L;
            for (int k = 0; k < dim; ++k) z = z + (long double)w[k] * (long double)x[k];
            z = z + (long double)b[j];
            long double acc = 0.0L;
            for (int t = 0; t < B->n_terms; ++t) {
                const orc_term *T = &B->terms[t];
                int32_t e[ORC_MAX_DIM], p;
                orc_diff(dim, T->alpha, e, &p);
                long double mono = 1.0L;
                for (int k = 0; k < dim; ++k)
                    for (int32_t n = 0; n < e[k]; ++n) mono = mono * (long double)w[k];
                long double c = T->coef;
                if (T->field >= 0) c = c * (long double)B->coef_fields[i * B->n_fields + T->field];
                acc = acc + c * mono * Phi_l(p, z);
            }
            A[r * n_features + j] = (double)((long double)B->weight * (s * acc));
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Least squares.  Golub & Van Loan, Matrix Computations (4th ed.):          */
/*   Alg. 5.1.1 (house) and Alg. 5.2.1 (Householder QR), unblocked.          */
/* The system is [A; sqrt(mu) I] beta ~ [b; 0] with sqrt(mu) = ridge_rel *   */
/* ||A||_F (reading A16; Tikhonov form P:L158).  Column-major      */
/* working copy M = [A_aug | b_aug], m_aug x (n+1).                          */
/* ------------------------------------------------------------------------- */

/* house(x): v with v[0] = 1 and beta such that (I - beta v v^T) x = ||x|| e_1 (GVL 5.1.1) */
static void house(const double *x, int64_t len, double *v, double *beta_out, double *mu_out) {
    double sigma = 0.0;
    for (int64_t i = 1; i < len; ++i) sigma = sigma + x[i] * x[i];
    v[0] = 1.0;
    for (int64_t i = 1; i < len; ++i) v[i] = x[i];
    double x0 = x[0];
    if (sigma == 0.0) {
        if (x0 >= 0.0) { *beta_out = 0.0; *mu_out = x0; }
        else { *beta_out = 2.0; *mu_out = -x0; }
        return;
    }
    double mu = sqrt(x0 * x0 + sigma);
    double v0 = (x0 <= 0.0) ? x0 - mu : -sigma / (x0 + mu);
    double beta = 2.0 * v0 * v0 / (sigma + v0 * v0);
    for (int64_t i = 1; i < len; ++i) v[i] = v[i] / v0;
    *beta_out = beta;
    *mu_out = mu;
}

/*
 * A: m x n row-major (as orc_assemble writes it), bvec: m.  beta_out: n.
 * resid_out (optional): ||A_aug beta - b_aug||_2 = norm of the trailing part of Q^T b_aug.
 * R_diag_out (optional): the n diagonal entries of R.
 * Returns 0, -1 on a zero diagonal of R (rank deficiency with mu = 0), -3 on allocation failure.
 */
static int lstsq_core(const double *A, int64_t m, int64_t n, const double *bvec, double sqmu,
                      double *beta_out, double *resid_out, double *R_diag_out);

int orc_lstsq(const double *A, int64_t m, int64_t n, const double *bvec, double ridge_rel,
              double *beta_out, double *resid_out, double *R_diag_out) {
    double fro = 0.0;
    for (int64_t i = 0; i < m * n; ++i) fro = fro + A[i] * A[i];
    fro = sqrt(fro);
    return lstsq_core(A, m, n, bvec, ridge_rel * fro, beta_out, resid_out, R_diag_out);
}

/* the same with an absolute sqrt(mu) (the Newton-step Tikhonov term, mu = 1e-10 P:L189) */
int orc_lstsq_mu(const double *A, int64_t m, int64_t n, const double *bvec, double sqrt_mu,
                 double *beta_out, double *resid_out, double *R_diag_out) {
    return lstsq_core(A, m, n, bvec, sqrt_mu, beta_out, resid_out, R_diag_out);
}

static int lstsq_core(const double *A, int64_t m, int64_t n, const double *bvec, double sqmu,
                      double *beta_out, double *resid_out, double *R_diag_out) {
    int64_t ma = m + ((sqmu > 0.0) ? n : 0);
    int64_t nc = n + 1;
    double *M = (double *)calloc((size_t)(ma * nc), sizeof(double));
    double *v = (double *)malloc((size_t)ma * sizeof(double));
    if (!M || !v) { free(M); free(v); return -3; }
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) M[j * ma + i] = A[i * n + j];
    for (int64_t i = 0; i < m; ++i) M[n * ma + i] = bvec[i];
    if (ma > m)
        for (int64_t j = 0; j < n; ++j) M[j * ma + m + j] = sqmu;

    int64_t steps = (n < ma) ? n : ma;
    for (int64_t k = 0; k < steps; ++k) {
        double bet, mu;
        house(&M[k * ma + k], ma - k, v, &bet, &mu);
        /* apply H_k = I - bet v v^T to columns k+1 .. n (including the rhs column) */
#pragma omp parallel for schedule(static)
        for (int64_t j = k + 1; j < nc; ++j) {
            double *col = &M[j * ma + k];
            double dot = 0.0;
            for (int64_t i = 0; i < ma - k; ++i) dot = dot + v[i] * col[i];
            double f = bet * dot;
            for (int64_t i = 0; i < ma - k; ++i) col[i] = col[i] - f * v[i];
        }
        M[k * ma + k] = mu;
        for (int64_t i = k + 1; i < ma; ++i) M[k * ma + i] = 0.0;
    }
    /* back substitution R beta = (Q^T b)[0:n]  (upper triangular R = M[0:n, 0:n]) */
    int status = 0;
    for (int64_t i = n - 1; i >= 0; --i) {
        double acc = (i < ma) ? M[n * ma + i] : 0.0;
        for (int64_t j = i + 1; j < n; ++j) acc = acc - M[j * ma + i] * beta_out[j];
        double rii = (i < ma) ? M[i * ma + i] : 0.0;
        if (rii == 0.0) { status = -1; beta_out[i] = 0.0; continue; }
        beta_out[i] = acc / rii;
    }
    if (R_diag_out)
        for (int64_t i = 0; i < n; ++i) R_diag_out[i] = (i < ma) ? M[i * ma + i] : 0.0;
    if (resid_out) {
        double r2 = 0.0;
        for (int64_t i = n; i < ma; ++i) r2 = r2 + M[n * ma + i] * M[n * ma + i];
        *resid_out = sqrt(r2);
    }
    free(M);
    free(v);
    return status;
}

/*
 * u_N(x_i) = s * sum_j beta_j sin(W_j . x_i + b_j)   (Eq. 1; Alg. 1 line 6 P:L141).
 */
int orc_eval(int dim, int64_t n_features, const double *W, const double *b, int normalize,
             const double *beta, const double *X, int64_t n_points, double *out) {
    const double s = normalize ? 1.0 / sqrt((double)n_features) : 1.0;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_points; ++i) {
        const double *x = X + i * dim;
        double acc = 0.0;
        for (int64_t j = 0; j < n_features; ++j) {
            double z = 0.0;
            for (int k = 0; k < dim; ++k) z = z + W[j * dim + k] * x[k];
            z = z + b[j];
            acc = acc + beta[j] * sin(z);
        }
        out[i] = s * acc;
    }
    return 0;
}

/* thread count of the OpenMP loops (cpu_baseline reports 1 thread and all host threads) */
void orc_set_threads(int n) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_max_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
