// fls_assemble.cuh -- the hot kernel: closed-form operator-matrix assembly (Eq. 2-3).
//
//   A_ij = sum_g c_g(x_i) (Ps_gj sin z_ij + Pc_gj cos z_ij),   z_ij = W_j . x_i + b_j
//
// (Eq. 2 folded per feature by the prefactor kernel; Eq. 3 row blocks).
// HBM-write-bound (8 B per entry) with the FP64 pipe as co-bound (d + 12 FP64 ops per entry
// in the sin-only family, + 1 per coefficient field).
//
// Column-major layout A[j * lda + i] (what cuSOLVER geqrf consumes):
//   CTA = kNT threads owning a kRowsCTA-row tile.  Thread t keeps the x_i (and coefficient
//   fields) of 2*kPairs rows -- the row pairs (p*2*kNT + 2t, +1), p < kPairs -- in registers
//   while the CTA walks a GROUP of kFC-feature chunks (grid.y = feature groups, so X is read
//   from HBM once per group, not once per chunk).  Per chunk the per-feature records
//   [W_j/pi, b'_j/pi, P_j...] are staged in shared memory and read as warp-uniform LDS.128
//   broadcasts.  Every store instruction of a warp writes 64 consecutive rows = 512
//   contiguous bytes of one column as one 16-byte st.global.cs per lane (streaming).
//   kFUnroll features per loop iteration (2*kPairs*kFUnroll independent entries per thread)
//   for FP64-pipe ILP; full tiles run a predicate-free loop, ragged tiles a masked one.
#pragma once
#include <stdio.h>
#include <stdlib.h>

#include <type_traits>

#include "fls_device.cuh"
#include "fls_feat.cuh"
#include "fls_internal.h"

#ifndef FLS_DIAG_NOSTORE
#define FLS_DIAG_NOSTORE 0  // 1: diagnostic build without the full-tile stores (never a product)
#endif
#ifndef FLS_WIDE_C5
#define FLS_WIDE_C5 1  // 0: the C5 class keeps the default 2 features / 4 CTAs (A/B builds)
#endif
#ifndef FLS_FLIP_OUTPUT
#define FLS_FLIP_OUTPUT 0
#endif
#ifndef FLS_STORE_POLICY
#define FLS_STORE_POLICY 0  // full-tile stores: 0 streaming (.cs), 1 write-back, 2 .cg (A/B builds)
#endif
#ifndef FLS_C2_FU1
#define FLS_C2_FU1 1  // 0: the C2 class keeps 2 features per iteration (A/B builds)
#endif
#ifndef FLS_C3_FU1
#define FLS_C3_FU1 1  // 0: the C3 class (d = 5) keeps 2 features per iteration (A/B builds)
#endif
#ifndef FLS_FU1_ALL_G0
#define FLS_FU1_ALL_G0 0  // 1: every d >= 2 constant-coefficient sin class (C4's d = 3 fold) (A/B)
#endif
#ifndef FLS_HOIST
#define FLS_HOIST 0
#endif
#ifndef FLS_C5_FU
#define FLS_C5_FU 4
#endif
#ifndef FLS_XOR_SIGN
#define FLS_XOR_SIGN FLS_FLIP_OUTPUT  // 1: the (-1)^n flip as shift + XOR (A/B builds)
#endif
#ifndef FLS_MINB
#define FLS_MINB 4   // 4 CTAs x 256 threads per SM -> <= 64 registers
#endif
#ifndef FLS_DIAG_CTATIME
#define FLS_DIAG_CTATIME 0  // 1: diagnostic build recording per-CTA timestamps (never a product)
#endif
#ifndef FLS_MINB5
#define FLS_MINB5 3  // d + G = 5 (C3): 3 CTAs -> <= 80 registers
#endif

namespace fls {

#if FLS_DIAG_CTATIME
// per CTA: entry, after the records' wait, after the first chunk's records, end (globaltimer ns),
// SM id, launch segment, (unused), points loaded -- read back by fls_diag_cta
// (tools/cta_timeline.py)
constexpr int kDiagSlots = 8, kDiagCTAs = 65536;
static __device__ unsigned long long g_cta_diag[kDiagSlots * kDiagCTAs];
__device__ __forceinline__ unsigned long long diag_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void diag_mark(int slot, unsigned long long v) {
  if (threadIdx.x == 0 && blockIdx.x < kDiagCTAs) g_cta_diag[blockIdx.x * kDiagSlots + slot] = v;
}
#define FLS_DIAG(slot, v) diag_mark(slot, v)
#else
#define FLS_DIAG(slot, v) ((void)0)
#endif

#ifndef FLS_X_EVICT_LAST
#define FLS_X_EVICT_LAST 0  // 1: point loads with an L2 evict_last policy (A/B builds)
#endif
// the prologue's 16-byte point loads
__device__ __forceinline__ double2 ldg_points(const double2 *p) {
#if FLS_X_EVICT_LAST
  double2 v;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
#else
  return __ldg(p);
#endif
}

template <int D, int G, int KM>
struct EntryMath {
  static constexpr int S = pf_stride(D, G, KM);

  __device__ __forceinline__ static void record(const double *p, double (&rec)[S]) {
#pragma unroll
    for (int s2 = 0; s2 < S / 2; ++s2) {
      const double2 v = reinterpret_cast<const double2 *>(p)[s2];
      rec[2 * s2] = v.x;
      rec[2 * s2 + 1] = v.y;
    }
  }

  // one entry from the feature record and the row's registers
  __device__ __forceinline__ static double entry(const double (&rec)[S], const double (&x)[D],
                                                 const double (&c)[G > 0 ? G : 1]) {
    double h = rec[D];
#pragma unroll
    for (int k = 0; k < D; ++k) h = fma(rec[k], x[k], h);
#if FLS_XOR_SIGN  // A/B build: shift + XOR sign flip
    int sgn;
    const double f = halfturn(h, sgn);
#else
    int nlo;
    const double f = halfturn_n(h, nlo);
#endif
    const double u = f * f;
    if constexpr (KM == KM_SIN) {
      double P = rec[D + 1];
#pragma unroll
      for (int g = 0; g < G; ++g) P = fma(c[g], rec[D + 2 + g], P);
      // (-1)^n on the argument, after u = f^2 is formed: sin is odd, so P sin(pi (-1)^n f) is
      // bit-identical to (-1)^n P sin(pi f), and the XOR then rewrites f's high word in place
      // (the result's register pair feeds the 16-byte store without a move)
#if FLS_FLIP_OUTPUT  // A/B build: the round-1 form (sign applied to the product)
      return flipsign(P * sinpi_core(f, u), sgn);
#elif FLS_XOR_SIGN
      return P * sinpi_core(flipsign(f, sgn), u);
#else
      return P * sinpi_core(addsign(f, nlo), u);
#endif
    } else {
      double Ps = rec[D + 1], Pc = rec[D + 2];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        Ps = fma(c[g], rec[D + 3 + 2 * g], Ps);
        Pc = fma(c[g], rec[D + 4 + 2 * g], Pc);
      }
#if FLS_XOR_SIGN
      return flipsign(fma(Ps, sinpi_core(f, u), Pc * cospi_core(u)), sgn);
#else
      return addsign(fma(Ps, sinpi_core(f, u), Pc * cospi_core(u)), nlo);
#endif
    }
  }
};

// resident CTAs per SM the register budget is sized for (checked against ptxas -v spills):
// sin-only with G <= 1, D + G <= 4 fits 64 registers (4 CTAs: C1, C2, C4, C5), D + G <= 5
// fits 80 (3 CTAs: C3); wider ones get 128 (2 CTAs) or 255 (1 CTA)
// the C5 class (d = 3, one coefficient field, sin family): 4 features per loop iteration at 80
// registers / 3 CTAs per SM (no spills; the 64-register default spilled 20 B) -- interleaved
// sustained 200-step A/B, 3 rounds on one box (tools/ab_variants.sh base narrow):
// 7.020-7.033e11 vs 6.961-6.962e11 entries/s (+0.9%); the same change costs C3 (d = 5) 17%
// and C2 6%, so it is limited to this class
template <int D, int G, int KM>
__host__ __device__ constexpr bool asm_wide_unroll() {
  return FLS_WIDE_C5 && FLS_FUNROLL == 2 && FLS_MINB == 4 && KM == KM_SIN && G == 1 && D == 3;
}
// the C2 class (d = 2, constant coefficients, sin family): 1 feature per iteration -- at 64
// registers the compiler runs the 2-feature body's 8 entries nearly one chain at a time anyway,
// and the 4 outputs of one feature are stored (freeing their registers) before the next;
// 10-step graph, 3 interleaved rounds (tools/ab_small.sh, FLS_FUNROLL=1 build): C2 17.92 ->
// 17.48 us, C1 (d = 1) unchanged, so limited to d = 2; the C3 class (d = 5, 80 registers) too:
// per_config C3 141.6 -> 139.9 us (short window), 167.3 -> 165.9 us sustained (3 rounds,
// tools/per_config_probe.py)
template <int D, int G, int KM>
__host__ __device__ constexpr int asm_funroll() {
  return asm_wide_unroll<D, G, KM>() ? FLS_C5_FU
         : (FLS_C2_FU1 && FLS_FUNROLL == 2 && D == 2 && G == 0 && KM == KM_SIN) ? 1
         : (FLS_C3_FU1 && FLS_FUNROLL == 2 && D == 5 && G == 0 && KM == KM_SIN) ? 1
         : (FLS_FU1_ALL_G0 && FLS_FUNROLL == 2 && D >= 2 && G == 0 && KM == KM_SIN) ? 1
                                                                               : kFUnroll;
}

template <int D, int G, int KM>
constexpr int asm_min_blocks() {
  if (asm_wide_unroll<D, G, KM>()) return 3;
  if (KM != KM_SIN) return D + G >= 9 ? 1 : 2;
  if (G <= 1 && D + G <= 4) return FLS_MINB;
  if (D + G <= 5) return FLS_MINB5;
  return D + G >= 10 ? 1 : 2;
}

// Launch shape: grid = (row tiles, feature groups), a.fpc features per CTA.  Picks the fewest
// feature groups that give >= 2 waves of resident CTAs (148 SMs x asm_min_blocks), then the
// group count in [g, 2g] whose last wave is fullest.  Each CTA keeps >= 16 features (>= kFC
// when the block's point data exceed 32 MB and would not stay in L2 between groups).
template <int D, int G, int KM>
inline dim3 asm_grid(AsmArgs &a) {
  static int sms = 0, waves = 2;  // tools/waves_sweep.sh, variant_sweep_c3.sh: 2 best for C3, flat for C4/C5
  static bool forced = false;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
    if (const char *w = getenv("FLS_ASM_WAVES")) {  // tuning sweeps only
      const int v = atoi(w);
      if (v >= 1 && v <= 64) {
        waves = v;
        forced = true;
      }
    }
  }
  const int64_t span = a.lr1 - (a.lr0 & ~int64_t(kRowAlign - 1));
  const int64_t rt = (span + kRowsCTA - 1) / kRowsCTA;
  const int64_t resident = (int64_t)sms * asm_min_blocks<D, G, KM>();
  const bool big_x = span * (D + G + 1) * 8 > ((int64_t)32 << 20);
  int64_t min_fpc = big_x ? (a.F < kFC ? a.F : kFC) : (a.F < 16 ? a.F : 16);
  // small blocks (C1, C2): 16-feature CTAs cannot fill the waves -> narrower CTAs (>= 2, the
  // features-per-iteration granularity) so the launch spreads over the SMs, each block of the
  // batch getting CTAs in proportion to its rows
  // small launches (<= 2^25 entries, C2): one wave of fatter CTAs -- every CTA pays the fixed
  // cost (launch, x and record loads, two syncs) once; C2 graph step 21.3 -> 20.5 us
  // (tools/small_step_probe.py); larger launches keep the sweep's 2 waves
  const int w_eff = (!forced && a.batch_span * a.F <= (int64_t(1) << 25)) ? 1 : waves;
  int64_t target = w_eff * resident;
  if (!big_x && rt * ((a.F + 15) / 16) < waves * resident) {
    min_fpc = a.F < 2 ? a.F : 2;
    if (a.batch_span > span) target = (target * span + a.batch_span - 1) / a.batch_span;
    const int64_t floor16 = rt * ((a.F + 15) / 16);  // never wider than 16 features per CTA
    if (target < floor16) target = floor16;
  }
  const int64_t gmax = (a.F + min_fpc - 1) / min_fpc;
  int64_t g0 = (target + rt - 1) / rt;
  g0 = g0 < 1 ? 1 : (g0 > gmax ? gmax : g0);
  int64_t best = g0;
  double best_eff = -1.0;
  for (int64_t g = g0; g <= 2 * g0 && g <= gmax; ++g) {
    const int64_t fpc = (((a.F + g - 1) / g) + 1) & ~int64_t(1);
    const int64_t gg = (a.F + fpc - 1) / fpc;
    const double nw = (double)(rt * gg) / (double)resident;
    const double eff = nw / ceil(nw);
    if (eff > best_eff + 1e-3) {
      best_eff = eff;
      best = gg;
    }
  }
  a.fpc = (((a.F + best - 1) / best) + 1) & ~int64_t(1);
  return dim3((unsigned)rt, (unsigned)((a.F + a.fpc - 1) / a.fpc));
}

// Launch plan of a batch (one launch, n row blocks sharing the variant): each block's grid from
// asm_grid, then -- for small launches (<= 2^25 entries, latency-bound: a thread's serial chain
// of fpc features x its rows sets a CTA's time) -- a joint correction, because asm_grid sizes
// each block against the whole wave on its own: C1's 2-row BC block got 63 CTAs of 8 features
// while its 1,000-row PDE block ran 250 CTAs of 2, so the BC CTAs were the critical path.
// FLS_BATCH_PLAN (A/B; tools/ab_small.sh, 10-step graphs, 3 interleaved rounds):
//   1 (default) cap every block's features per CTA at the largest block's: C1 5.92 -> 4.92 us,
//     C2 unchanged (its BC CTAs already carry fewer features than its PDE CTAs);
//   0 per-block grids only;
//   2 one feature count for all blocks, the smallest even one whose CTAs fit one wave: C1 4.92,
//     C2 17.9 -> 19.7 us (C2's PDE CTAs grow from 14 to 18 features);
//   3 equal entries per CTA, relaxed until the CTAs fit one wave: C2 20.5, C1 87 us (its 2-row
//     BC CTAs get 424 features each).
template <int D, int G, int KM>
inline int64_t asm_plan(AsmArgs *blks, int n, AsmBatch &bt, bool fused = false) {
  const char *plan_env = getenv("FLS_BATCH_PLAN");  // read per call: tests switch it
  const int strategy = plan_env && *plan_env ? atoi(plan_env) : 1;
  int64_t span = 0;
  for (int q = 0; q < n; ++q) span += blks[q].lr1 - (blks[q].lr0 & ~int64_t(kRowAlign - 1));
  dim3 g[kMaxBatch];
  for (int q = 0; q < n; ++q) {
    blks[q].batch_span = span;
    g[q] = asm_grid<D, G, KM>(blks[q]);  // sets blks[q].fpc
  }
  const int64_t F = blks[0].F;
  bool same_f = true;
  for (int q = 1; q < n; ++q) same_f = same_f && blks[q].F == F;
  if (n > 1 && strategy > 0 && same_f && F > 0 && span * F <= (int64_t(1) << 25) &&
      !getenv("FLS_ASM_WAVES")) {
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
    const int64_t resident = (int64_t)sms * asm_min_blocks<D, G, KM>();
    int64_t rt_sum = 0;
    for (int q = 0; q < n; ++q) rt_sum += g[q].x;
    auto even_up = [&](int64_t v) { v = v < 2 ? 2 : v; return (v + 1) & ~int64_t(1); };
    int64_t fpc[kMaxBatch];
    bool ok = false;
    if (strategy == 1) {
      int big = 0;
      for (int q = 1; q < n; ++q)
        if (blks[q].lr1 - blks[q].lr0 > blks[big].lr1 - blks[big].lr0) big = q;
      for (int q = 0; q < n; ++q) fpc[q] = blks[q].fpc < blks[big].fpc ? blks[q].fpc : blks[big].fpc;
      ok = true;
    } else if (strategy == 2) {
      for (int64_t f = 2; f <= even_up(F) && !ok; f += 2) {
        if (rt_sum * ((F + f - 1) / f) <= resident) {
          for (int q = 0; q < n; ++q) fpc[q] = f;
          ok = true;
        }
      }
    } else {
      for (int64_t E = (span * F + resident - 1) / resident; !ok && E <= 2 * span * F; E += E / 32 + 1) {
        int64_t total = 0;
        for (int q = 0; q < n; ++q) {
          const int64_t sq = blks[q].lr1 - (blks[q].lr0 & ~int64_t(kRowAlign - 1));
          const int64_t rows = sq < kRowsCTA ? sq : kRowsCTA;
          int64_t f = even_up((E + rows - 1) / rows);
          if (f > even_up(F)) f = even_up(F);
          fpc[q] = f;
          total += (int64_t)g[q].x * ((F + f - 1) / f);
        }
        ok = total <= resident;
      }
    }
    if (ok) {
      for (int q = 0; q < n; ++q) {
        blks[q].fpc = fpc[q];
        g[q].y = (unsigned)((F + fpc[q] - 1) / fpc[q]);
      }
    }
  }
  // segments: block q's features [0, F) as one segment (the plan above), or -- guided tail,
  // FLS_TAIL_PCT percent of its features, FLS_TAIL_FPC features per CTA -- a main segment and
  // a tail segment of narrower CTAs; every tail follows every main segment in the grid, so the
  // hardware dispatches the narrow CTAs last, into the SM slots the main CTAs free.  The
  // per-CTA timeline of C2 (tools/cta_timeline.py: FLS_DIAG_CTATIME build) shows why: the warp
  // schedulers favour the oldest CTAs, so an SM's four first-wave CTAs end at 40-100% of the
  // window and the busy slots fall from 592 to 65 over its last 40%.  Interleaved A/B
  // (tools/ab_tail.py, 10-step graphs, 4 rounds): C2 17.52 -> 17.24 us at 10% / 4 features
  // (5% / 4: 17.41, 10% / 6: 17.43, 10% / 8: 17.63, 20% / 4: 18.35); the fused C1 gets slower
  // (4.94 -> 5.21 us) and so do the multi-wave launches (C3 141 -> 155 us, C4 664 -> 716 us at
  // 10% / 4: their narrow CTAs' prologues cost more than the drain they shorten), so the
  // default tail is for unfused launches of 2^22 .. 2^25 entries (C2) only.
  const char *tp_env = getenv("FLS_TAIL_PCT");
  const char *tf_env = getenv("FLS_TAIL_FPC");
  const bool tail_class = !fused && span * F > (int64_t(1) << 22) && span * F <= (int64_t(1) << 25);
  const int64_t tail_pct = tp_env && *tp_env ? atoll(tp_env) : (tail_class ? 10 : 0);
  const int64_t tail_fpc = tf_env && *tf_env ? atoll(tf_env) : 4;
  AsmArgs seg[kMaxSeg];
  dim3 sg[kMaxSeg];
  int nseg = n;
  for (int q = 0; q < n; ++q) {
    seg[q] = blks[q];
    seg[q].f_begin = 0;
    seg[q].f_end = blks[q].F;
    seg[q].pre_idx = q;
    sg[q] = g[q];
  }
  if (tail_pct > 0 && tail_fpc > 0) {
    for (int q = 0; q < n; ++q) {
      const int64_t Fq = blks[q].F, T = (Fq * tail_pct / 100) & ~int64_t(1);
      if (T < tail_fpc || Fq - T < blks[q].fpc) continue;
      seg[q].f_end = Fq - T;
      sg[q].y = (unsigned)((Fq - T + blks[q].fpc - 1) / blks[q].fpc);
      AsmArgs &t = seg[nseg];
      t = seg[q];
      t.f_begin = Fq - T;
      t.f_end = Fq;
      t.fpc = tail_fpc;
      t.rhs = nullptr;
      sg[nseg] = dim3(g[q].x, (unsigned)((T + tail_fpc - 1) / tail_fpc));
      ++nseg;
    }
  }
  // FLS_PLAN_DEBUG=1 prints each launch's plan (read once).  Measured and rejected: giving every
  // block of a large multi-wave launch the largest block's features per CTA (C3 141.7 -> 145.2
  // us, C4 664 -> 713 us; per_config, 2 rounds)
  static const bool plan_debug = getenv("FLS_PLAN_DEBUG") != nullptr;
  if (plan_debug)
    for (int q = 0; q < nseg; ++q)
      fprintf(stderr, "fls plan: block %d rows %lld tiles %u groups %u fpc %lld features [%lld, %lld)\n",
              seg[q].pre_idx, (long long)(seg[q].lr1 - seg[q].lr0), sg[q].x, sg[q].y,
              (long long)seg[q].fpc, (long long)seg[q].f_begin, (long long)seg[q].f_end);
  bt.n = nseg;
  int64_t total = 0;
  for (int q = 0; q < nseg; ++q) {
    bt.blk[q] = seg[q];
    bt.rt[q] = sg[q].x;
    total += (int64_t)sg[q].x * sg[q].y;
    bt.cta_end[q] = total;
  }
  return total;
}

// full-tile store of one feature column's entries of this thread: two 16-byte streaming stores
// (row pairs 2*kNT apart) or, with kQuad, one 32-byte store of 4 consecutive rows
template <int NQ>
__device__ __forceinline__ void store_full(double *colp, const double (&o)[NQ]) {
#if FLS_DIAG_NOSTORE  // diagnostic build only: keep the values alive, store (almost) nothing
  int bits = 0;
#pragma unroll
  for (int q = 0; q < NQ; ++q) bits ^= __double2hiint(o[q]);
  if (bits == 0x7ff80001) *colp = o[0];
  return;
#endif
  if constexpr (kQuad) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(colp), "d"(o[0]), "d"(o[1]),
                 "d"(o[2]), "d"(o[3])
                 : "memory");
  } else {
#pragma unroll
    for (int pr = 0; pr < NQ / 2; ++pr) {
      double2 *p = reinterpret_cast<double2 *>(colp + pr * (2 * kNT));
#if FLS_STORE_POLICY == 1
      *p = make_double2(o[2 * pr], o[2 * pr + 1]);
#elif FLS_STORE_POLICY == 2
      __stcg(p, make_double2(o[2 * pr], o[2 * pr + 1]));
#else
      __stcs(p, make_double2(o[2 * pr], o[2 * pr + 1]));
#endif
    }
  }
}

// exact phase-range check of one thread's rows against features [f0, f1) (only threads whose
// bound exceeded the limit run it): h as EntryMath::entry computes it
template <int D, int S, int NQ>
__device__ __forceinline__ void phase_check(const double *pf, int64_t f0, int64_t f1,
                                         const double (&x)[NQ][D], const bool (&in)[NQ],
                                         unsigned *err) {
  for (int64_t j = f0; j < f1; ++j) {
    const double *r = pf + j * S;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double h = __ldg(r + D);
#pragma unroll
      for (int k = 0; k < D; ++k) h = fma(__ldg(r + k), x[q][k], h);
      if (in[q] && !(fabs(h) <= kMaxHalfTurns)) {
        atomicOr(err, kErrPhaseRange);
        return;
      }
    }
  }
}

// the fused kernel's exact check: records recomputed per feature (rare path)
template <int D, int NQ>
__device__ __forceinline__ void phase_check_wb(const FusedBatch &fz, int pq, int64_t f0, int64_t f1,
                                               const double (&x)[NQ][D], const bool (&in)[NQ],
                                               unsigned *err) {
  double rec[pf_stride(FLS_MAX_DIM, FLS_MAX_FIELDS, KM_SINCOS)];
  double w[D];
  for (int64_t j = f0; j < f1; ++j) {
#pragma unroll
    for (int k = 0; k < D; ++k) w[k] = feat_normal(j * D + k, D, fz.fb, fz.seed);
    prefactor_rec<>(fz.pre[pq], w, feat_bias(j, fz.seed), rec);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double h = rec[D];
#pragma unroll
      for (int k = 0; k < D; ++k) h = fma(rec[k], x[q][k], h);
      if (in[q] && !(fabs(h) <= kMaxHalfTurns)) {
        atomicOr(err, kErrPhaseRange);
        return;
      }
    }
  }
}

// One launch covers up to kMaxBatch row blocks that share the kernel variant (e.g. a PDE block
// and its identity BC / IC blocks): the 1-D grid is the concatenation of each block's
// (row tile, feature group) CTAs, row tile fastest.
struct NoFuse {};

// Z = NoFuse: the records come from the preceding prefactor launch (a.pf).  Z = FusedBatch: the
// CTA computes the records of each chunk itself (a1 + a2 in the prologue; one launch per call).
template <int D, int G, int KM, class Z = NoFuse>
__global__ void __launch_bounds__(kNT, asm_min_blocks<D, G, KM>())
assemble_cm_kernel(const AsmBatch bt, const Z fz) {
  constexpr bool kFused = !std::is_same<Z, NoFuse>::value;
  using M = EntryMath<D, G, KM>;
  constexpr int S = M::S;
  constexpr int GG = G > 0 ? G : 1;
  constexpr int NQ = 2 * kPairs;  // rows per thread
  static_assert(S % 2 == 0, "pf stride must be even for 16-byte smem reads");
  extern __shared__ __align__(16) double sp[];

  // let the next PDL launch on the stream (the next call's feature / prefactor kernel, which
  // writes nothing before its own griddepcontrol.wait) start while this grid runs
  pdl_trigger();
  FLS_DIAG(0, diag_now());
  int qb = 0;
  while (qb + 1 < bt.n && (int64_t)blockIdx.x >= bt.cta_end[qb]) ++qb;
  const AsmArgs &a = bt.blk[qb];
  const int64_t cta = (int64_t)blockIdx.x - (qb ? bt.cta_end[qb - 1] : 0);
  const int64_t tile = cta % bt.rt[qb], group = cta / bt.rt[qb];
  // this CTA's feature range [f0, f1) (a.fpc features per CTA, chosen by the launcher), walked
  // in shared-memory chunks of at most kFC records
  const int64_t f0 = a.f_begin + group * a.fpc;
  const int64_t f1 = f0 + a.fpc < a.f_end ? f0 + a.fpc : a.f_end;
  // phase-range guard (FLS_MAX_PHASE): |h_ij| <= ||W_j/pi||_1 ||x_i||_inf + |b'_j/pi|.  The
  // feature side is max-reduced over the CTA's records chunk by chunk (s_guard, off the entry
  // path); at the end a thread whose bound exceeds the limit re-checks its rows exactly.
  __shared__ unsigned long long s_guard[2];
  if (threadIdx.x == 0) s_guard[0] = s_guard[1] = 0ull;  // visible after the first chunk sync

  // fused: a1 -- the chunk's normals and biases, one draw per thread (the
  // features_prefactor_kernel draws: bit-identical) into shared memory after the records, both
  // Philox chains side by side; a2 -- one thread per feature folds its record.  Reads nothing
  // from global memory; writes W, b only when wr.
  bool wr = false;
  if constexpr (kFused) wr = fz.write_wb && a.pre_idx == 0 && tile == 0;
  auto fused_chunk = [&](int64_t j0, int nfe, bool write_wb) {
    if constexpr (kFused) {
      double *ws = sp + kFC * S;      // normals (nfe * D), then biases (nfe)
      double *bs = ws + kFC * D;
      for (int t = threadIdx.x; t < nfe * (D + 1); t += kNT) {
        if (t < nfe * D) {
          const int64_t m = j0 * D + t;
          const double w = feat_normal(m, D, fz.fb, fz.seed);
          ws[t] = w;
          if (write_wb) fz.W[m] = w;
        } else {
          const int64_t j = j0 + (t - nfe * D);
          const double bj = feat_bias(j, fz.seed);
          bs[t - nfe * D] = bj;
          if (write_wb) fz.b[j] = bj;
        }
      }
      __syncthreads();
      for (int t = threadIdx.x; t < nfe; t += kNT)
        prefactor_rec<GG + 1>(fz.pre[a.pre_idx], ws + t * D, bs[t], sp + t * S);
    }
  };
  const int nfe0 = (f1 - f0) < kFC ? (int)(f1 - f0) : kFC;
  // the first chunk's records before the wait: with programmatic dependent launch they are
  // drawn while the previous kernel on the stream still runs
  if constexpr (kFused) {
    if (f0 < f1) fused_chunk(f0, nfe0, false);
    // the fused kernel runs ahead of an ARBITRARY predecessor (PDL), which may still be producing
    // X / fields / values or reading A, W, b: no global memory is touched above this line
    pdl_wait();
  }

  // local rows (A-relative) of this thread: rbase + p*2*kNT + {0, 1}; rbase is even.
  // The block's points map to local rows [lr0, lr1): point i = pt0 + (r - lr0).
  const int64_t rbase = (a.lr0 & ~int64_t(kRowAlign - 1)) + tile * kRowsCTA + kRowAlign * threadIdx.x;
  double x[NQ][D];
  double c[NQ][GG];
  double rv[NQ];
  bool in[NQ];
  bool bad = false;
  bool full = a.vec;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int64_t r = kQuad ? rbase + q : rbase + (q >> 1) * (2 * kNT) + (q & 1);
    in[q] = (r >= a.lr0) && (r < a.lr1);
    full = full && in[q];
  }
  // the points of a row pair are 2 D contiguous doubles: D 16-byte loads per pair instead of
  // 2 D 8-byte ones when the pair's first point sits on a 16-byte boundary (X aligned and
  // (pt0 - lr0) D even; rbase is even).  The CTA prologue's point loads were its longest step
  // (C2: 1.6 us of per-CTA latency at the start of each step, tools/cta_timeline.py)
  const int64_t podd = (a.pt0 - a.lr0) & 1;
  const bool xvec = !kQuad && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) && ((podd * D) & 1) == 0;
  const bool cvec = !kQuad && G == 1 && a.nf == 1 && a.gfield[0] == 0 &&
                    ((reinterpret_cast<uintptr_t>(a.fields) & 15) == 0) && podd == 0;
#pragma unroll
  for (int pr = 0; pr < NQ / 2; ++pr) {
    const int q0 = 2 * pr;
    const int64_t r0 = kQuad ? rbase + q0 : rbase + pr * (2 * kNT);
    const int64_t i0 = a.pt0 + (r0 - a.lr0);
    if (xvec && in[q0] && in[q0 + 1]) {
      const double2 *xp = reinterpret_cast<const double2 *>(a.X + i0 * D);
#pragma unroll
      for (int m = 0; m < D; ++m) {
        const double2 v = ldg_points(xp + m);
        x[q0 + (2 * m) / D][(2 * m) % D] = v.x;
        x[q0 + (2 * m + 1) / D][(2 * m + 1) % D] = v.y;
      }
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int k = 0; k < D; ++k) x[q0 + h][k] = in[q0 + h] ? __ldg(a.X + (i0 + h) * D + k) : 0.0;
    }
    if (G > 0 && cvec && in[q0] && in[q0 + 1]) {
      const double2 v = __ldg(reinterpret_cast<const double2 *>(a.fields + i0));
      c[q0][0] = v.x;
      c[q0 + 1][0] = v.y;
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int g = 0; g < GG; ++g)
          c[q0 + h][g] = (G > 0 && in[q0 + h]) ? __ldg(a.fields + (i0 + h) * a.nf + a.gfield[g]) : 0.0;
    }
  }
  if constexpr (kFused) {
    // the rhs values are requested with the points, before anything waits for either (C1
    // 10-step graph 4.91 -> 4.79 us; the same order makes the unfused C2 launch slower,
    // 16.41 -> 16.68 us, so that one keeps the order below -- tools/ab_lib.sh, 3 rounds)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int64_t r = kQuad ? rbase + q : rbase + (q >> 1) * (2 * kNT) + (q & 1);
      const int64_t i = a.pt0 + (r - a.lr0);
      rv[q] = (group == 0 && a.rhs != nullptr && in[q] && a.values) ? __ldg(a.values + i) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
#pragma unroll
      for (int k = 0; k < D; ++k) bad |= !finite(x[q][k]);
#pragma unroll
      for (int g = 0; g < GG; ++g) bad |= !finite(c[q][g]);
      bad |= !finite(rv[q]);
      rv[q] *= a.weight;
    }
  } else {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
#pragma unroll
      for (int k = 0; k < D; ++k) bad |= !finite(x[q][k]);
#pragma unroll
      for (int g = 0; g < GG; ++g) bad |= !finite(c[q][g]);
      const int64_t r = kQuad ? rbase + q : rbase + (q >> 1) * (2 * kNT) + (q & 1);
      const int64_t i = a.pt0 + (r - a.lr0);
      rv[q] = 0.0;
      if (group == 0 && a.rhs != nullptr && in[q]) {
        const double v = a.values ? __ldg(a.values + i) : 0.0;
        bad |= !finite(v);
        rv[q] = a.weight * v;
      }
    }
  }
  // the two-launch path: this grid is launched (PDL) once the prefactor kernel before it has
  // triggered, which it does only after everything ahead of it on the stream completed -- so
  // the points above were safe to read; the records it writes are safe to read from here on
  FLS_DIAG(6, diag_now() + (bad ? 1 : 0));  // (the points have arrived: bad depends on them)
  if constexpr (!kFused) pdl_wait();
  FLS_DIAG(1, diag_now());
  if (group == 0 && a.rhs != nullptr) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int64_t r = kQuad ? rbase + q : rbase + (q >> 1) * (2 * kNT) + (q & 1);
      if (in[q]) a.rhs[r] = rv[q];
    }
  }
  if (bad) atomicOr(a.err, kErrNonFinite);
  double xinf = 0.0;
#pragma unroll
  for (int q = 0; q < NQ; ++q)
#pragma unroll
    for (int k = 0; k < D; ++k) xinf = fmax(xinf, fabs(x[q][k]));
  if constexpr (kFused) {
    if (wr && f0 < f1) {  // the first chunk's W, b (drawn before the wait) go out now
      const double *ws = sp + kFC * S, *bs = ws + kFC * D;
      for (int t = threadIdx.x; t < nfe0 * D; t += kNT) fz.W[f0 * D + t] = ws[t];
      for (int t = threadIdx.x; t < nfe0; t += kNT) fz.b[f0 + t] = bs[t];
    }
  }

  for (int64_t j0 = f0; j0 < f1; j0 += kFC) {
    const int nfe = (f1 - j0) < kFC ? (int)(f1 - j0) : kFC;
    __syncthreads();  // previous chunk's records no longer in use
    if constexpr (kFused) {
      if (j0 != f0) fused_chunk(j0, nfe, wr);
    } else {
      const double2 *src = reinterpret_cast<const double2 *>(a.pf + j0 * S);
      double2 *dst = reinterpret_cast<double2 *>(sp);
      const int n2 = nfe * (S / 2);
      for (int t = threadIdx.x; t < n2; t += kNT) dst[t] = __ldg(src + t);
    }
    __syncthreads();
    if (j0 == f0) FLS_DIAG(2, diag_now());
    if (threadIdx.x < nfe) {
      const double *r = sp + threadIdx.x * S;
      double w1 = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) w1 += fabs(r[k]);
      atomicMax(&s_guard[0], (unsigned long long)__double_as_longlong(w1));
      atomicMax(&s_guard[1], (unsigned long long)__double_as_longlong(fabs(r[D])));
    }
    double *colp = a.A + j0 * a.lda + rbase;
    if (full) {
      int jj = 0;
      constexpr int FU = asm_funroll<D, G, KM>();
#if FLS_HOIST
      const int64_t lda = a.lda;  // a is this block's entry of bt (dynamic index)
      const double *rp = sp;
      for (; jj + FU <= nfe; jj += FU, colp += FU * lda, rp += FU * S) {
#else
      const int64_t lda = a.lda;
      for (; jj + FU <= nfe; jj += FU, colp += FU * a.lda) {
        const double *rp = sp + jj * S;
#endif
        double o[FU][NQ];
#pragma unroll
        for (int u = 0; u < FU; ++u) {
          double rec[S];
          M::record(rp + u * S, rec);
#pragma unroll
          for (int q = 0; q < NQ; ++q) o[u][q] = M::entry(rec, x[q], c[q]);
        }
#pragma unroll
        for (int u = 0; u < FU; ++u) store_full(colp + u * lda, o[u]);
      }
      for (; jj < nfe; ++jj, colp += a.lda) {
        double rec[S];
        M::record(sp + jj * S, rec);
        double o[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) o[q] = M::entry(rec, x[q], c[q]);
        store_full(colp, o);
      }
    } else {
      for (int jj = 0; jj < nfe; ++jj, colp += a.lda) {
        double rec[S];
        M::record(sp + jj * S, rec);
        double o[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) o[q] = M::entry(rec, x[q], c[q]);
        if (kQuad) {
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            if (in[q]) __stcs(colp + q, o[q]);
        } else {
#pragma unroll
          for (int pr = 0; pr < kPairs; ++pr) {
            double *dst = colp + pr * (2 * kNT);
            if (a.vec && in[2 * pr] && in[2 * pr + 1]) {
              __stcs(reinterpret_cast<double2 *>(dst), make_double2(o[2 * pr], o[2 * pr + 1]));
            } else {
              if (in[2 * pr]) __stcs(dst, o[2 * pr]);
              if (in[2 * pr + 1]) __stcs(dst + 1, o[2 * pr + 1]);
            }
          }
        }
      }
    }
  }
  __syncthreads();
#if FLS_DIAG_CTATIME
  {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    FLS_DIAG(3, diag_now());
    FLS_DIAG(4, smid);
    FLS_DIAG(5, qb);
  }
#endif
  const double bound = fma(__longlong_as_double((long long)s_guard[0]), xinf,
                           __longlong_as_double((long long)s_guard[1]));
  if (bound > kMaxHalfTurns) {
    if constexpr (kFused) {
      // no record array in global memory: the records are recomputed (prefactor_rec, the same
      // draw and fold, so h is bit-identical to the entry's)
      phase_check_wb<D, NQ>(fz, a.pre_idx, f0, f1, x, in, a.err);
    } else {
      phase_check<D, S, NQ>(a.pf, f0, f1, x, in, a.err);
    }
  }
}

// launch one batch, with the programmatic-dependent-launch attribute when the caller knows the
// preceding operation on the stream is the prefactor launch of the same call (or an earlier
// assembly batch of it, which writes disjoint rows)
template <class Kern, class Z>
inline cudaError_t asm_launch(Kern kern, unsigned ctas, size_t smem, cudaStream_t st, bool pdl,
                              const AsmBatch &bt, const Z &fz) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctas);
  cfg.blockDim = dim3(kNT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, bt, fz);
}

}  // namespace fls
