// fls_asm_sin.cu -- instantiations of the column-major assembly kernel, KM_SIN family
// (split from the other family so the two compile in parallel).
#include "fls_assemble.cuh"

namespace fls {

template <int D, int G>
static cudaError_t go_sin(AsmArgs *blks, int n, cudaStream_t st, bool pdl,
                          const FusedBatch *fz = nullptr) {
  constexpr int S = pf_stride(D, G, KM_SIN);
  // fused: the chunk's normals and biases follow the records in shared memory
  const size_t smem = (size_t)kFC * (S + (fz ? D + 1 : 0)) * sizeof(double);
  AsmBatch bt;
  const int64_t total = asm_plan<D, G, KM_SIN>(blks, n, bt, fz != nullptr);
  if (fz) {
    if constexpr (G <= 1) {
      auto kern = assemble_cm_kernel<D, G, KM_SIN, FusedBatch>;
      if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
      }
      return asm_launch(kern, (unsigned)total, smem, st, pdl, bt, *fz);
    } else {
      return cudaErrorNotSupported;
    }
  }
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(assemble_cm_kernel<D, G, KM_SIN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  return asm_launch(assemble_cm_kernel<D, G, KM_SIN>, (unsigned)total, smem, st, pdl, bt, NoFuse{});
}

cudaError_t launch_assemble_cm_fused(int D, int G, AsmArgs *blks, int n, const FusedBatch &fz,
                                     cudaStream_t st, bool pdl) {
  if (G > 1) return cudaErrorNotSupported;
#define FLS_FG(d)                                            \
  return G == 0 ? go_sin<d, 0>(blks, n, st, pdl, &fz)        \
                : go_sin<d, 1>(blks, n, st, pdl, &fz);
  switch (D) {
    case 1: FLS_FG(1)
    case 2: FLS_FG(2)
    case 3: FLS_FG(3)
    case 4: FLS_FG(4)
    case 5: FLS_FG(5)
    case 6: FLS_FG(6)
    case 7: FLS_FG(7)
    case 8: FLS_FG(8)
    default: return cudaErrorInvalidValue;
  }
#undef FLS_FG
}

cudaError_t launch_assemble_cm_sin(int D, int G, AsmArgs *blks, int n, cudaStream_t st, bool pdl) {
#define FLS_G(d)                                 \
  switch (G) {                                   \
    case 0: return go_sin<d, 0>(blks, n, st, pdl);    \
    case 1: return go_sin<d, 1>(blks, n, st, pdl);    \
    case 2: return go_sin<d, 2>(blks, n, st, pdl);    \
    case 3: return go_sin<d, 3>(blks, n, st, pdl);    \
    case 4: return go_sin<d, 4>(blks, n, st, pdl);    \
    default: return cudaErrorInvalidValue;       \
  }
  switch (D) {
    case 1: FLS_G(1)
    case 2: FLS_G(2)
    case 3: FLS_G(3)
    case 4: FLS_G(4)
    case 5: FLS_G(5)
    case 6: FLS_G(6)
    case 7: FLS_G(7)
    case 8: FLS_G(8)
    default: return cudaErrorInvalidValue;
  }
#undef FLS_G
}

}  // namespace fls

#if FLS_DIAG_CTATIME
// diagnostic builds only: copy the per-CTA timestamps of the KM_SIN kernels to the host
extern "C" __attribute__((visibility("default"))) int fls_diag_cta(void *host, long long n) {
  const long long cap = (long long)fls::kDiagSlots * fls::kDiagCTAs * 8;
  if (n > cap) n = cap;
  return (int)cudaMemcpyFromSymbol(host, fls::g_cta_diag, (size_t)n);
}
#endif
