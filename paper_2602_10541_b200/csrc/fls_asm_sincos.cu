// fls_asm_sincos.cu -- instantiations of the column-major assembly kernel, KM_SINCOS family
// (split from the other family so the two compile in parallel).
#include "fls_assemble.cuh"

namespace fls {

template <int D, int G>
static cudaError_t go_sincos(AsmArgs *blks, int n, cudaStream_t st, bool pdl) {
  constexpr int S = pf_stride(D, G, KM_SINCOS);
  const size_t smem = (size_t)kFC * S * sizeof(double);
  AsmBatch bt;
  const int64_t total = asm_plan<D, G, KM_SINCOS>(blks, n, bt);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(assemble_cm_kernel<D, G, KM_SINCOS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  return asm_launch(assemble_cm_kernel<D, G, KM_SINCOS>, (unsigned)total, smem, st, pdl, bt, NoFuse{});
}

cudaError_t launch_assemble_cm_sincos(int D, int G, AsmArgs *blks, int n, cudaStream_t st, bool pdl) {
#define FLS_G(d)                                 \
  switch (G) {                                   \
    case 0: return go_sincos<d, 0>(blks, n, st, pdl);    \
    case 1: return go_sincos<d, 1>(blks, n, st, pdl);    \
    case 2: return go_sincos<d, 2>(blks, n, st, pdl);    \
    case 3: return go_sincos<d, 3>(blks, n, st, pdl);    \
    case 4: return go_sincos<d, 4>(blks, n, st, pdl);    \
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
