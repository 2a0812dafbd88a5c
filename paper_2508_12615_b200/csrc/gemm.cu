// tcgen05 GEMM entry: dispatch on the epilogue (the kernels are instantiated
// in gemm_e*.cu from gemm_impl.cuh).
#include "common.cuh"

namespace wipes {

cudaError_t launch_gemm_e0(const wipes_gemm_args& g, cudaStream_t s);
cudaError_t launch_gemm_e1(const wipes_gemm_args& g, cudaStream_t s);
cudaError_t launch_gemm_e2(const wipes_gemm_args& g, cudaStream_t s);
cudaError_t launch_gemm_e3(const wipes_gemm_args& g, cudaStream_t s);
cudaError_t launch_gemm_e4(const wipes_gemm_args& g, cudaStream_t s);

cudaError_t launch_gemm(const wipes_gemm_args& g, cudaStream_t s) {
  switch (g.epilogue) {
    case WIPES_GEMM_EPI_STORE_F32: return launch_gemm_e0(g, s);
    case WIPES_GEMM_EPI_BIAS_F32: return launch_gemm_e1(g, s);
    case WIPES_GEMM_EPI_BIAS_RELU_BF16: return launch_gemm_e2(g, s);
    case WIPES_GEMM_EPI_MASK_BF16: return launch_gemm_e3(g, s);
    default: return launch_gemm_e4(g, s);
  }
}

}  // namespace wipes
