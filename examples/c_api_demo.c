/*
 * c_api_demo.c -- Algorithm 1 through the plain C ABI of libfls, no
 * Python: features -> collocation points -> assembly of [A | b] -> Householder QR solve ->
 * u_N at test points, for -u'' = pi^2 sin(pi x) on [0, 1], u(0) = u(1) = 0 (exact u = sin(pi x)).
 * Then the same solve through the multi-rank path: an NCCL communicator (here one rank; a
 * launcher would hand every rank the same id), TSQR forced, the relative Tikhonov ridge
 * sqrt(mu) = ridge_rel ||A||_F computed inside libfls.
 *
 *   gcc -O2 -I include examples/c_api_demo.c -L paper_2602_10541_b200 -lfls \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2602_10541_b200 -lm -o c_api_demo
 *   ./c_api_demo        (prints the relative L2 error of u_N; exit 0 if < 1e-6)
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "fls.h"

#define CHECK(x)                                                                   \
  do {                                                                             \
    fls_status s_ = (x);                                                           \
    if (s_ != FLS_OK) {                                                            \
      fprintf(stderr, "%s -> %s: %s\n", #x, fls_status_string(s_), fls_last_error()); \
      return 2;                                                                    \
    }                                                                              \
  } while (0)

int main(void) {
  const double PI = 3.14159265358979323846;
  const int d = 1;
  const int64_t F = 200, n_int = 1000, n_test = 2000;
  fls_ctx *ctx = NULL;
  CHECK(fls_ctx_create(0, NULL, &ctx));

  double *W, *b, *Xi, *Xb, *f, *g, *Ab, *beta, *Xt, *ut;
  const int64_t R = n_int + 2, lda = (R + 3) / 4 * 4;
  cudaMalloc((void **)&W, sizeof(double) * F * d);
  cudaMalloc((void **)&b, sizeof(double) * F);
  cudaMalloc((void **)&Xi, sizeof(double) * n_int);
  cudaMalloc((void **)&Xb, sizeof(double) * 2);
  cudaMalloc((void **)&f, sizeof(double) * n_int);
  cudaMalloc((void **)&g, sizeof(double) * 2);
  cudaMalloc((void **)&Ab, sizeof(double) * lda * (F + 1));
  cudaMalloc((void **)&beta, sizeof(double) * F);
  cudaMalloc((void **)&Xt, sizeof(double) * n_test);
  cudaMalloc((void **)&ut, sizeof(double) * n_test);

  /* line 1: W ~ N(0, 3^2), b ~ U[0, 2 pi) */
  CHECK(fls_features(ctx, d, F, 3.0, 0, W, b));
  /* line 2: interior points and the two boundary points */
  const double lo = 0.0, hi = 1.0;
  CHECK(fls_sample_box(ctx, d, n_int, &lo, &hi, 0, 3, Xi));
  CHECK(fls_sample_faces(ctx, d, 1, 1u, &lo, &hi, 0, 4, Xb));
  CHECK(fls_sample_box(ctx, d, n_test, &lo, &hi, 0, 6, Xt));
  CHECK(fls_sync(ctx));
  double *h = (double *)malloc(sizeof(double) * n_test);
  cudaMemcpy(h, Xi, sizeof(double) * n_int, cudaMemcpyDeviceToHost);
  for (int64_t i = 0; i < n_int; ++i) h[i] = PI * PI * sin(PI * h[i]);   /* f = pi^2 sin(pi x) */
  cudaMemcpy(f, h, sizeof(double) * n_int, cudaMemcpyHostToDevice);
  cudaMemset(g, 0, sizeof(double) * 2);                                    /* g = 0 */

  /* lines 3-5: [ -u'' rows ; 100 u rows ] and rhs [f ; 100 g] as column F of [A | b] */
  fls_term lap = {{2}, -1.0, -1}, ident = {{0}, 1.0, -1};
  fls_operator op_pde = {d, 1, &lap}, op_bc = {d, 1, &ident};
  fls_block blocks[2] = {{Xi, n_int, &op_pde, NULL, 0, 1.0, f}, {Xb, 2, &op_bc, NULL, 0, 100.0, g}};
  CHECK(fls_assemble(ctx, W, b, d, F, 1, blocks, 2, 0, R, Ab, lda, FLS_COL_MAJOR, Ab + F * lda));
  double resid = 0.0;
  CHECK(fls_solve(ctx, Ab, R, lda, F, 0.0, beta, &resid));
  /* line 6: u_N at the test points */
  CHECK(fls_eval(ctx, W, b, d, F, 1, beta, NULL, Xt, n_test, ut));
  CHECK(fls_sync(ctx));

  double *hx = (double *)malloc(sizeof(double) * n_test);
  cudaMemcpy(hx, Xt, sizeof(double) * n_test, cudaMemcpyDeviceToHost);
  double rel[2];
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      /* the multi-rank solve: communicator, TSQR, relative ridge inside libfls */
      unsigned char id[FLS_COMM_ID_BYTES];
      CHECK(fls_comm_unique_id(id));
      CHECK(fls_comm_init(ctx, id, 1, 0));
      CHECK(fls_comm_config(ctx, FLS_TSQR_AUTO, 1));
      CHECK(fls_assemble(ctx, W, b, d, F, 1, blocks, 2, 0, R, Ab, lda, FLS_COL_MAJOR, Ab + F * lda));
      CHECK(fls_solve(ctx, Ab, R, lda, F, 1e-12, beta, &resid));
      CHECK(fls_eval(ctx, W, b, d, F, 1, beta, NULL, Xt, n_test, ut));
      CHECK(fls_sync(ctx));
    }
    cudaMemcpy(h, ut, sizeof(double) * n_test, cudaMemcpyDeviceToHost);
    double e2 = 0.0, n2 = 0.0;
    for (int64_t i = 0; i < n_test; ++i) {
      const double ex = sin(PI * hx[i]);
      e2 += (h[i] - ex) * (h[i] - ex);
      n2 += ex * ex;
    }
    rel[pass] = sqrt(e2 / n2);
  }
  int32_t nr = 0, rk = 0, tr = 0;
  CHECK(fls_comm_info(ctx, &nr, &rk, &tr));
  printf("c_api_demo: residual %.3e, relative L2 error of u_N %.3e (single QR), %.3e "
         "(communicator of %d rank(s), TSQR transport %s, ridge_rel 1e-12)\n", resid, rel[0], rel[1],
         nr, tr == FLS_TSQR_P2P ? "p2p" : tr == FLS_TSQR_NCCL ? "nccl" : "none");
  fls_ctx_destroy(ctx);
  return (rel[0] < 1e-6 && rel[1] < 1e-6 && tr != 0) ? 0 : 1;
}
