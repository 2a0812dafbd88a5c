// tcgen05 GEMM with fused epilogues (NEXT-4 building block; see gemm_tc.cuh).
#include "gemm_tc.cuh"

namespace wipes {

namespace {

using namespace tc;

template <int NT>
struct GemmSmem {
  __nv_bfloat16 a[2][kM * kKC];
  __nv_bfloat16 b[2][NT * kKC];
  uint64_t bar[2];
  uint32_t tmem;
};

// Stage one operand tile (R rows x kKC) of chunk k0 into the canonical layout.
template <int R, bool MN>
__device__ __forceinline__ void stage(__nv_bfloat16* dst, const __nv_bfloat16* src, int64_t ld,
                                      int64_t r0, int64_t rows, int64_t k0, int64_t K, int tid) {
  constexpr int kChunks = R * (kKC / 8);
#pragma unroll 4
  for (int c = tid; c < kChunks; c += kThreads) {
    int r, kk, off;
    const __nv_bfloat16* s;
    bool ok;
    if (!MN) {  // 16 B = 8 consecutive k of row r
      r = c >> 3;
      const int kc = c & 7;
      kk = 8 * kc;
      off = (((r >> 3) * 8 + kc) << 7) + ((r & 7) << 4);
      ok = r0 + r < rows && k0 + kk < K;
      s = src + (ok ? (r0 + r) * ld + k0 + kk : 0);
    } else {    // 16 B = 8 consecutive rows at one k
      const int g = c % (R / 8);
      kk = c / (R / 8);
      r = 8 * g;
      off = ((g * 8 + (kk >> 3)) << 7) + ((kk & 7) << 4);
      ok = r0 + r < rows && k0 + kk < K;
      s = src + (ok ? (k0 + kk) * ld + r0 + r : 0);
    }
    cp16(reinterpret_cast<char*>(dst) + off, s, ok);
  }
}

template <int NT, bool AMN, bool BMN, int EPI>
__global__ void __launch_bounds__(kThreads) k_gemm(const wipes_gemm_args g) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  GemmSmem<NT>& sm = *reinterpret_cast<GemmSmem<NT>*>(smem_raw);
  constexpr int kCols = NT <= 32 ? 32 : (NT <= 64 ? 64 : (NT <= 128 ? 128 : 256));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = (int64_t)blockIdx.x * kM, n0 = (int64_t)blockIdx.y * NT;
  // this CTA's K range (split-K over gridDim.z, whole chunks)
  const int64_t nchunk_all = (g.K + kKC - 1) / kKC;
  const int64_t per = (nchunk_all + gridDim.z - 1) / gridDim.z;
  const int64_t c_lo = per * blockIdx.z;
  const int64_t c_hi = c_lo + per < nchunk_all ? c_lo + per : nchunk_all;
  const __nv_bfloat16* A = reinterpret_cast<const __nv_bfloat16*>(g.A);
  const __nv_bfloat16* B = reinterpret_cast<const __nv_bfloat16*>(g.B);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&sm.tmem)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&sm.bar[0], 1);
    mbar_init(&sm.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  const uint32_t idesc = instr_desc(NT, AMN, BMN);
  uint32_t phase[2] = {0, 0};

  const int64_t nch = c_hi - c_lo;
  if (nch > 0) {
    stage<kM, AMN>(sm.a[0], A, g.lda, m0, g.M, c_lo * kKC, g.K, tid);
    stage<NT, BMN>(sm.b[0], B, g.ldb, n0, g.N, c_lo * kKC, g.K, tid);
    cp_commit();
  }
  for (int64_t c = 0; c < nch; ++c) {
    const int buf = (int)(c & 1);
    if (c + 1 < nch) {
      const int nb = buf ^ 1;
      if (c >= 1) {  // buffer nb was read by the MMAs of chunk c - 1
        mbar_wait(&sm.bar[nb], phase[nb]);
        phase[nb] ^= 1;
      }
      const int64_t k0 = (c_lo + c + 1) * kKC;
      stage<kM, AMN>(sm.a[nb], A, g.lda, m0, g.M, k0, g.K, tid);
      stage<NT, BMN>(sm.b[nb], B, g.ldb, n0, g.N, k0, g.K, tid);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    fence_proxy_async();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t a0 = smem_u32(sm.a[buf]), b0 = smem_u32(sm.b[buf]);
#pragma unroll
      for (int j = 0; j < kKC / 16; ++j)
        mma_bf16(tmem, smem_desc(a0 + 256 * j, 128, 1024), smem_desc(b0 + 256 * j, 128, 1024),
                 idesc, (c > 0 || j > 0) ? 1u : 0u);
      mma_commit(&sm.bar[buf]);
    }
  }
  // the last chunk's commit covers all earlier MMAs
  if (nch > 0) {
    const int lb = (int)((nch - 1) & 1);
    mbar_wait(&sm.bar[lb], phase[lb]);
  }
  tc_fence_after();

  // ---- epilogue: warp w owns rows 32w..32w+31 of the tile ------------------
  const int64_t m = m0 + 32 * warp + lane;
  const bool mrow = m < g.M;
#pragma unroll 1
  for (int cb = 0; cb < NT / 32 + (NT % 32 ? 1 : 0); ++cb) {
    float v[32];
    if (nch > 0) {
      tmem_ld32(tmem + ((uint32_t)(32 * warp) << 16) + (uint32_t)(32 * cb), v);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
    }
    if (!mrow) continue;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int64_t n = n0 + 32 * cb + i;
      if (32 * cb + i >= NT || n >= g.N) break;
      float x = v[i];
      if (EPI == WIPES_GEMM_EPI_STORE_F32) {
        reinterpret_cast<float*>(g.C)[m * g.ldc + n] = x;
      } else if (EPI == WIPES_GEMM_EPI_BIAS_F32) {
        reinterpret_cast<float*>(g.C)[m * g.ldc + n] = x + g.bias[n];
      } else if (EPI == WIPES_GEMM_EPI_BIAS_RELU_BF16) {
        x = fmaxf(x + g.bias[n], 0.f);
        reinterpret_cast<__nv_bfloat16*>(g.C)[m * g.ldc + n] = __float2bfloat16_rn(x);
      } else if (EPI == WIPES_GEMM_EPI_MASK_BF16) {
        const float mk = __bfloat162float(
            reinterpret_cast<const __nv_bfloat16*>(g.mask)[m * g.ldm + n]);
        reinterpret_cast<__nv_bfloat16*>(g.C)[m * g.ldc + n] =
            __float2bfloat16_rn(mk > 0.f ? x : 0.f);
      } else {  // WIPES_GEMM_EPI_ATOMIC_F32
        atomicAdd(reinterpret_cast<float*>(g.C) + m * g.ldc + n, x);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
}

template <int NT, bool AMN, bool BMN, int EPI>
cudaError_t launch_nt(const wipes_gemm_args& g, cudaStream_t s) {
  auto k = k_gemm<NT, AMN, BMN, EPI>;
  const int smem = (int)sizeof(GemmSmem<NT>) + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid((unsigned)((g.M + kM - 1) / kM), (unsigned)((g.N + NT - 1) / NT),
            (unsigned)(g.split_k > 0 ? g.split_k : 1));
  launch_begin(K_GEMM, s);
  k<<<grid, kThreads, smem, s>>>(g);
  launch_end(K_GEMM, s);
  return cudaGetLastError();
}

template <bool AMN, bool BMN, int EPI>
cudaError_t launch_maj(const wipes_gemm_args& g, cudaStream_t s) {
  if (g.N <= 16) return launch_nt<16, AMN, BMN, EPI>(g, s);
  if (g.N <= 64) return launch_nt<64, AMN, BMN, EPI>(g, s);
  if (g.N <= 128) return launch_nt<128, AMN, BMN, EPI>(g, s);
  return launch_nt<256, AMN, BMN, EPI>(g, s);
}

template <int EPI>
cudaError_t launch_epi(const wipes_gemm_args& g, cudaStream_t s) {
  if (!g.a_mn_major && !g.b_mn_major) return launch_maj<false, false, EPI>(g, s);
  if (!g.a_mn_major && g.b_mn_major) return launch_maj<false, true, EPI>(g, s);
  if (g.a_mn_major && !g.b_mn_major) return launch_maj<true, false, EPI>(g, s);
  return launch_maj<true, true, EPI>(g, s);
}

}  // namespace

cudaError_t launch_gemm(const wipes_gemm_args& g, cudaStream_t s) {
  switch (g.epilogue) {
    case WIPES_GEMM_EPI_STORE_F32: return launch_epi<WIPES_GEMM_EPI_STORE_F32>(g, s);
    case WIPES_GEMM_EPI_BIAS_F32: return launch_epi<WIPES_GEMM_EPI_BIAS_F32>(g, s);
    case WIPES_GEMM_EPI_BIAS_RELU_BF16: return launch_epi<WIPES_GEMM_EPI_BIAS_RELU_BF16>(g, s);
    case WIPES_GEMM_EPI_MASK_BF16: return launch_epi<WIPES_GEMM_EPI_MASK_BF16>(g, s);
    default: return launch_epi<WIPES_GEMM_EPI_ATOMIC_F32>(g, s);
  }
}

}  // namespace wipes
