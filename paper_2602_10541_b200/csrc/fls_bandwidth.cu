// fls_bandwidth.cu -- learnable-bandwidth support (App. E).
//
//   W_j = L W^_j,   Lout(L) = ||A(L) beta* - b||^2,
//   dLout/dL_kl = 2 sum_j beta_j W^_jl V_jk,   V_jk = sum_i r_i dA_ij/dW_jk,
//   dA_ij/dW_jk = w s sum_t c_t(x_i) [alpha_tk prod W^(alpha_t - e_k) Phi_p(z) + prod W^alpha_t x_ik Phi_{p+1}(z)].
//
// Per feature and coefficient-field group g the bracket folds to  Ps_k sin z + Pc_k cos z +
// x_ik (Qs sin z + Qc cos z)  (the same cyclic-derivative bookkeeping as the assembly
// prefactors); a row combines the groups with its coefficients c_g(x_i) (c_0 = 1), so each
// (row, feature) pair costs one half-turn sin/cos pair plus (G + 1)(2d + 2) + 2d FMAs.  All
// reductions run in a fixed order.
#include <math.h>

#include "fls_device.cuh"
#include "fls_internal.h"

namespace fls {

__global__ void transform_kernel(int32_t D, int64_t F, const TransformArgs t, const double *Wh,
                                 double *W) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= F) return;
  double w[FLS_MAX_DIM];
  for (int l = 0; l < D; ++l) w[l] = Wh[j * D + l];
  for (int k = 0; k < D; ++k) {
    double acc = 0.0;
    for (int l = 0; l < D; ++l) acc = fma(t.L[k * D + l], w[l], acc);
    W[j * D + k] = acc;
  }
}

cudaError_t launch_transform(int32_t D, int64_t F, const TransformArgs &t, const double *Wh,
                             double *W, cudaStream_t st) {
  transform_kernel<<<(unsigned)((F + 255) / 256), 256, 0, st>>>(D, F, t, Wh, W);
  return cudaGetLastError();
}

// record per feature (stride a.S = grad_stride(D, G)): [W_k/pi (D), b/pi, then for each field
// group g = 0..G (0 = constant coefficients): Ps_k (D), Pc_k (D), Qs, Qc]
__global__ void grad_prefactor_kernel(const PrefArgs a) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.F) return;
  const int D = a.D;
  double w[FLS_MAX_DIM];
  bool ok = true;
  for (int k = 0; k < D; ++k) {
    w[k] = a.W[j * D + k];
    ok &= finite(w[k]);
  }
  const double bj = a.b[j];
  ok &= finite(bj);
  if (!ok) atomicOr(a.err, 1u);
  double *out = a.pf + j * a.S;
  for (int k = 0; k < D; ++k) out[k] = w[k] * kInvPi;
  out[D] = bj * kInvPi;
  for (int g = 0; g <= a.G; ++g) {
    double Ps[FLS_MAX_DIM], Pc[FLS_MAX_DIM], Qs = 0.0, Qc = 0.0;
    for (int k = 0; k < D; ++k) Ps[k] = Pc[k] = 0.0;
    for (int t = 0; t < a.n_terms; ++t) {
      const TermDev &T = a.terms[t];
      if (T.group != g) continue;
      int order = 0;
      for (int k = 0; k < D; ++k) order += T.alpha[k];
      const int p = order & 3;
      // phase-derivative part: c prod W^alpha Phi_{p+1}
      double m = T.coef;
      for (int k = 0; k < D; ++k)
        for (int e = 0; e < T.alpha[k]; ++e) m *= w[k];
      const int q = (p + 1) & 3;
      const double mq = (q & 2) ? -m : m;
      if (q & 1) Qc += mq; else Qs += mq;
      // monomial-derivative part: c alpha_k prod W^(alpha - e_k) Phi_p
      for (int k = 0; k < D; ++k) {
        if (T.alpha[k] == 0) continue;
        double mk = T.coef * (double)T.alpha[k];
        for (int l = 0; l < D; ++l)
          for (int e = 0; e < T.alpha[l] - (l == k ? 1 : 0); ++e) mk *= w[l];
        if (p & 2) mk = -mk;
        if (p & 1) Pc[k] += mk; else Ps[k] += mk;
      }
    }
    double *o = out + D + 1 + g * (2 * D + 2);
    for (int k = 0; k < D; ++k) {
      o[k] = a.scale * Ps[k];
      o[D + k] = a.scale * Pc[k];
    }
    o[2 * D] = a.scale * Qs;
    o[2 * D + 1] = a.scale * Qc;
  }
}

cudaError_t launch_grad_prefactor(const PrefArgs &a, cudaStream_t st) {
  grad_prefactor_kernel<<<(unsigned)((a.F + 127) / 128), 128, 0, st>>>(a);
  return cudaGetLastError();
}

// CTA: 32 features (lane = feature) x the rows [r0, r1) of one slot; 8 warps split the rows,
// fixed-order warp-tree combine; partials[slot][j][k].  With field groups the row's
// coefficients c_g(x_i) combine the group records first (c_0 = 1).
template <int D, int G>
__global__ void __launch_bounds__(256) grad_reduce_kernel(const GradArgs a) {
  constexpr int R = grad_stride(D, G);
  constexpr int GS = 2 * D + 2;
  __shared__ double sm[8][32][D];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const int64_t r0 = a.row0 + (int64_t)blockIdx.y * a.rows_per_slot;
  int64_t r1 = r0 + a.rows_per_slot;
  if (r1 > a.row1) r1 = a.row1;
  double rec[R];
  const bool on = j < a.F;
#pragma unroll
  for (int s = 0; s < R; ++s) rec[s] = on ? a.pf[j * a.S + s] : 0.0;
  double acc[D];
#pragma unroll
  for (int k = 0; k < D; ++k) acc[k] = 0.0;
  bool bad = false;
  for (int64_t i = r0 + warp; i < r1; i += 8) {
    double x[D];
#pragma unroll
    for (int k = 0; k < D; ++k) x[k] = a.X[i * D + k];
    const double r = a.r[i];
    bad |= !finite(r);
    double c[G + 1];
    c[0] = 1.0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      c[g + 1] = a.fields[i * a.nf + a.gfield[g]];
      bad |= !finite(c[g + 1]);
    }
    double h = rec[D];
#pragma unroll
    for (int k = 0; k < D; ++k) h = fma(rec[k], x[k], h);
    int sgn;
    const double f = halfturn(h, sgn);
    const double u = f * f;
    const double sn = flipsign(sinpi_core(f, u), sgn), cs = flipsign(cospi_core(u), sgn);
    double qs = 0.0, qc = 0.0;
#pragma unroll
    for (int g = 0; g <= G; ++g) {
      qs = fma(c[g], rec[D + 1 + g * GS + 2 * D], qs);
      qc = fma(c[g], rec[D + 1 + g * GS + 2 * D + 1], qc);
    }
    const double q = r * fma(qs, sn, qc * cs);
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double ps = 0.0, pc = 0.0;
#pragma unroll
      for (int g = 0; g <= G; ++g) {
        ps = fma(c[g], rec[D + 1 + g * GS + k], ps);
        pc = fma(c[g], rec[D + 1 + g * GS + D + k], pc);
      }
      acc[k] = fma(r, fma(ps, sn, pc * cs), fma(q, x[k], acc[k]));
    }
  }
  if (bad) atomicOr(a.err, 1u);
#pragma unroll
  for (int k = 0; k < D; ++k) sm[warp][lane][k] = acc[k];
  __syncthreads();
  if (warp == 0 && on) {
    double* dst = a.partials + ((int64_t)(a.slot0 + blockIdx.y) * a.F + j) * D;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      double s = 0.0;
      for (int w = 0; w < 8; ++w) s += sm[w][lane][k];
      dst[k] = s;
    }
  }
}

template <int D>
static cudaError_t go_grad(int G, const GradArgs &a, dim3 grid, cudaStream_t st) {
  switch (G) {
    case 0: grad_reduce_kernel<D, 0><<<grid, 256, 0, st>>>(a); break;
    case 1: grad_reduce_kernel<D, 1><<<grid, 256, 0, st>>>(a); break;
    case 2: grad_reduce_kernel<D, 2><<<grid, 256, 0, st>>>(a); break;
    case 3: grad_reduce_kernel<D, 3><<<grid, 256, 0, st>>>(a); break;
    case 4: grad_reduce_kernel<D, 4><<<grid, 256, 0, st>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_grad_reduce(int D, int G, const GradArgs &a, int slots, cudaStream_t st) {
  const dim3 grid((unsigned)((a.F + 31) / 32), (unsigned)slots);
  switch (D) {
    case 1: return go_grad<1>(G, a, grid, st);
    case 2: return go_grad<2>(G, a, grid, st);
    case 3: return go_grad<3>(G, a, grid, st);
    case 4: return go_grad<4>(G, a, grid, st);
    case 5: return go_grad<5>(G, a, grid, st);
    case 6: return go_grad<6>(G, a, grid, st);
    case 7: return go_grad<7>(G, a, grid, st);
    case 8: return go_grad<8>(G, a, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

// G_kl = 2 sum_j beta_j W^_jl sum_slots V_jk   (one CTA per (k, l); fixed-order tree)
__global__ void grad_final_kernel(int D, int64_t F, int nslots, const double *partials,
                                  const double *beta, const double *Wh, double *G) {
  __shared__ double sm[256];
  const int k = blockIdx.x / D, l = blockIdx.x % D;
  double acc = 0.0;
  for (int64_t j = threadIdx.x; j < F; j += 256) {
    double v = 0.0;
    for (int s = 0; s < nslots; ++s) v += partials[((int64_t)s * F + j) * D + k];
    acc = fma(beta[j] * Wh[j * D + l], v, acc);
  }
  sm[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) sm[threadIdx.x] += sm[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) G[k * D + l] = 2.0 * sm[0];
}

cudaError_t launch_grad_final(int D, int64_t F, int nslots, const double *partials,
                              const double *beta, const double *Wh, double *G, cudaStream_t st) {
  grad_final_kernel<<<D * D, 256, 0, st>>>(D, F, nslots, partials, beta, Wh, G);
  return cudaGetLastError();
}

}  // namespace fls
