// NEXT-2: the image-fitting step around the rasterizer — the
// L2 objective with its image gradient, and Adam with the parameter
// activations fused in (include/wipes.h "NEXT-2").
//
// Both kernels are HBM-bound streaming passes sized as a fixed grid (a
// multiple of the SM count, independent of the data) so that the FP64 loss
// reduction has a fixed order (run-to-run deterministic) and both are
// graph-capturable: the Adam step counter and the reduction tickets live in
// device memory, and the last CTA to finish resets its ticket.
#include <cmath>

#include "common.cuh"

namespace wipes {

namespace {

constexpr int kTrainThreads = 256;
constexpr int kLossBlocks = 148 * 8;  // fixed grid: fixed reduction order

struct TrainScratch {
  unsigned int loss_ticket, adam_ticket;
  unsigned int pad[14];
  double partial[kLossBlocks];
};

__device__ __forceinline__ double block_sum(double x, double* sm) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if (lane == 0) sm[wid] = x;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kTrainThreads / 32; ++w) t += sm[w];
  __syncthreads();
  return t;  // valid in thread 0
}

// loss = (1/n) sum d^2, dL/dC = (2/n) d, d = image - target.
__global__ void __launch_bounds__(kTrainThreads) k_loss_l2(const float* __restrict__ img,
                                                           const float* __restrict__ tgt,
                                                           int64_t n, float scale,
                                                           float* __restrict__ grad,
                                                           double* loss, TrainScratch* sc) {
  __shared__ double sm[kTrainThreads / 32];
  __shared__ bool last;
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float d = __fsub_rn(img[i], tgt[i]);
    grad[i] = __fmul_rn(scale, d);
    acc += (double)d * (double)d;
  }
  const double bsum = block_sum(acc, sm);
  if (threadIdx.x == 0) {
    sc->partial[blockIdx.x] = bsum;
    __threadfence();
    last = atomicAdd(&sc->loss_ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double t = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
    t += ((volatile double*)sc->partial)[b];
  const double tot = block_sum(t, sm);
  if (threadIdx.x == 0) {
    *loss = tot / (double)n;
    sc->loss_ticket = 0;
  }
}

struct AdamArgs {
  wipes_adam_group g[WIPES_MAX_ADAM_GROUPS];
  int64_t prefix[WIPES_MAX_ADAM_GROUPS + 1];
  int32_t ng, activate_only;
  float b1, b2, eps;
  int64_t* step;
  const int32_t* guard;
  TrainScratch* sc;
};

__device__ __forceinline__ float sigmoid(float x) { return 1.f / (1.f + expf(-x)); }

__global__ void __launch_bounds__(kTrainThreads) k_adam(const __grid_constant__ AdamArgs a) {
  __shared__ float bc[2];
  __shared__ bool skip, last;
  if (threadIdx.x == 0) {
    skip = a.guard && *(volatile const int32_t*)a.guard != 0;
    if (!a.activate_only && !skip) {
      const double t = (double)(*(volatile int64_t*)a.step + 1);
      bc[0] = (float)(1.0 / (1.0 - pow((double)a.b1, t)));  // 1 / (1 - b1^t)
      bc[1] = (float)(1.0 / (1.0 - pow((double)a.b2, t)));
    }
  }
  __syncthreads();
  if (!skip) {
    const int64_t total = a.prefix[a.ng];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
      int k = 0;
      while (i >= a.prefix[k + 1]) ++k;
      const wipes_adam_group& G = a.g[k];
      const int64_t j = i - a.prefix[k];
      float p = G.param[j];
      if (!a.activate_only) {
        float g = G.grad[j];
        if (G.activation == WIPES_ACT_SIGMOID) {
          const float s = sigmoid(p);
          g = g * (s * (1.f - s));
        }
        const float m = a.b1 * G.m[j] + (1.f - a.b1) * g;
        const float v = a.b2 * G.v[j] + (1.f - a.b2) * (g * g);
        G.m[j] = m;
        G.v[j] = v;
        const float mh = m * bc[0], vh = v * bc[1];
        p = p - G.lr * mh / (sqrtf(vh) + a.eps);
        G.param[j] = p;
      }
      if (G.activation == WIPES_ACT_SIGMOID && G.act) G.act[j] = sigmoid(p);
    }
  }
  if (a.activate_only) return;
  // the last CTA advances the step counter (every CTA has read it by now)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&a.sc->adam_ticket, 1u) == gridDim.x - 1;
    if (last) {
      a.sc->adam_ticket = 0;
      if (!skip) *a.step = *(volatile int64_t*)a.step + 1;
    }
  }
}

}  // namespace

size_t train_scratch_bytes() { return sizeof(TrainScratch); }

cudaError_t launch_loss_l2(const float* img, const float* tgt, int64_t n, float* grad,
                           double* loss, void* scratch, cudaStream_t s) {
  const int64_t need = (n + kTrainThreads - 1) / kTrainThreads;
  const int grid = (int)(need < kLossBlocks ? (need > 0 ? need : 1) : kLossBlocks);
  const float scale = (float)(2.0 / (double)(n > 0 ? n : 1));
  launch_begin(K_LOSS, s);
  k_loss_l2<<<grid, kTrainThreads, 0, s>>>(img, tgt, n, scale, grad, loss,
                                           (TrainScratch*)scratch);
  launch_end(K_LOSS, s);
  return cudaGetLastError();
}

cudaError_t launch_adam(const wipes_adam_group* groups, int ng, float b1, float b2, float eps,
                        int64_t* step, const int32_t* guard, void* scratch, int activate_only,
                        cudaStream_t s) {
  AdamArgs a;
  a.ng = ng;
  a.prefix[0] = 0;
  for (int k = 0; k < ng; ++k) {
    a.g[k] = groups[k];
    a.prefix[k + 1] = a.prefix[k] + groups[k].n;
  }
  a.activate_only = activate_only;
  a.b1 = b1; a.b2 = b2; a.eps = eps;
  a.step = step; a.guard = guard;
  a.sc = (TrainScratch*)scratch;
  const int64_t need = (a.prefix[ng] + kTrainThreads - 1) / kTrainThreads;
  const int grid = (int)(need < 148 * 8 ? (need > 0 ? need : 1) : 148 * 8);
  launch_begin(K_ADAM, s);
  k_adam<<<grid, kTrainThreads, 0, s>>>(a);
  launch_end(K_ADAM, s);
  return cudaGetLastError();
}

}  // namespace wipes
