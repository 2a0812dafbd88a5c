// tcgen05 GEMM instantiations for the store_f32 epilogue (see gemm_impl.cuh).
#include "gemm_impl.cuh"

namespace wipes {
cudaError_t launch_gemm_e0(const wipes_gemm_args& g, cudaStream_t s) {
  return launch_epi<WIPES_GEMM_EPI_STORE_F32>(g, s);
}
}  // namespace wipes
