// tcgen05 GEMM instantiations for the bias_relu_bf16 epilogue (see gemm_impl.cuh).
#include "gemm_impl.cuh"

namespace wipes {
cudaError_t launch_gemm_e2(const wipes_gemm_args& g, cudaStream_t s) {
  return launch_epi<WIPES_GEMM_EPI_BIAS_RELU_BF16>(g, s);
}
}  // namespace wipes
