// tcgen05 GEMM with fused epilogues (NEXT-4 building block; see gemm_tc.cuh):
// the persistent warp-specialised kernel, included by one translation unit per
// epilogue (gemm_e*.cu) so the 80 instantiations compile in parallel.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "gemm_tc.cuh"

namespace wipes {

namespace {

using namespace tc;

// Stage one operand tile (R rows x kKC) of chunk k0 into the canonical layout.
template <int R, bool MN, int NTHR = kThreads>
__device__ __forceinline__ void stage(__nv_bfloat16* dst, const __nv_bfloat16* src, int64_t ld,
                                      int64_t r0, int64_t rows, int64_t k0, int64_t K, int tid) {
  // 16-byte slots to visit: K-major R x 8 chunks; MN-major 8 k-blocks x
  // ceil(G/4) group quads x 32 lanes (lanes of a partial quad stay idle)
  constexpr int kChunks = MN ? 8 * ((R / 8 + 3) / 4) * 32 : R * (kKC / 8);
  // Thread -> chunk mapping: each quarter-warp (8 lanes, one shared-memory
  // phase of 16-byte accesses) covers the 8 rows of a core matrix, i.e. the 8
  // distinct 16-byte bank groups (conflict-free), while 4 lanes along the
  // contiguous dimension keep 64 contiguous bytes per global row segment.
#pragma unroll 4
  for (int c = tid; c < kChunks; c += NTHR) {
    const int q = c >> 5, ln = c & 31;
    int r, kk, off;
    const __nv_bfloat16* s;
    bool ok;
    if (!MN) {  // 16 B = 8 consecutive k of row r
      r = (q >> 1) * 8 + (ln & 7);
      const int kc = (q & 1) * 4 + (ln >> 3);
      kk = 8 * kc;
      off = (((r >> 3) * 8 + kc) << 7) + ((r & 7) << 4);
      ok = r0 + r < rows && k0 + kk < K;
      s = src + (ok ? (r0 + r) * ld + k0 + kk : 0);
    } else {    // 16 B = 8 consecutive rows (MN) at one k
      constexpr int G = R / 8;               // MN groups of 8
      // q enumerates (k block of 8, group quad); lanes: (k & 7, group within quad)
      const int kb = q / ((G + 3) / 4), gq = q % ((G + 3) / 4);
      const int g = gq * 4 + (ln >> 3);
      kk = kb * 8 + (ln & 7);
      r = 8 * g;
      off = ((g * 8 + (kk >> 3)) << 7) + ((kk & 7) << 4);
      ok = g < G && r0 + r < rows && k0 + kk < K;
      s = src + (ok ? (k0 + kk) * ld + r0 + r : 0);
      if (g >= G) continue;
    }
    cp16(reinterpret_cast<char*>(dst) + off, s, ok);
  }
}

// ---------------------------------------------------------------------------
// Persistent, warp-specialised variant (one CTA per SM):
//   warps 0..P-1  producers: cp.async A/B chunks into a kStages ring; each
//                 thread's cp.async completion arrives on full[s] (noinc);
//   warp P        one lane issues tcgen05.mma per chunk, commits the chunk to
//                 empty[s] and the finished tile to tfull[acc];
//   warp P+1      owns the TMEM allocation (2 accumulators of NT columns);
//   warps P+2..   4 epilogue warps (TMEM lanes 32 (w mod 4)..): drain
//                 accumulator acc while the MMA warp fills the other one,
//                 then arrive on tempty[acc].
// Tiles t = blockIdx.x + i gridDim.x enumerate (m tile, n tile, k split).
// ---------------------------------------------------------------------------
#ifndef WIPES_GEMM_PROD_WARPS
#define WIPES_GEMM_PROD_WARPS 2
#endif
#ifndef WIPES_GEMM_EPI_WARPS
#define WIPES_GEMM_EPI_WARPS 8
#endif
constexpr int kProdWarps = WIPES_GEMM_PROD_WARPS;
constexpr int kEpiWarps = WIPES_GEMM_EPI_WARPS;  // 4 or 8 (two per TMEM lane quarter)
constexpr int kProd = 32 * kProdWarps;
constexpr int kMmaWarp = kProdWarps, kAllocWarp = kProdWarps + 1, kEpiWarp0 = kProdWarps + 2;
constexpr int kWsThreads = 32 * (kProdWarps + 2 + kEpiWarps);
static_assert(kEpiWarp0 % 4 == 0, "epilogue warps must start at a multiple of 4 (TMEM lanes)");
constexpr int kMaxStages = 4;
constexpr int kSmemMax = 227 * 1024;

// Runtime carve of the dynamic shared memory (1024-aligned base):
//   A ring  [stages][128 x 64] bf16,
//   B       [stages][NT x 64] (streamed) or [all K chunks][NT x 64] (resident),
//   barriers full/empty[kMaxStages], tfull/tempty[2], bfull, TMEM address.
struct WsCarve {
  uint32_t a, b, stg, bar, stages, bres, bytes;
};
// per epilogue warp: one 32 x 32 fp32 output block + one 32 x 32 bf16 mask block
constexpr uint32_t kStgWarpBytes = 32 * 32 * 4 + 32 * 32 * 2;
constexpr uint32_t kStgBytes = 8 * kStgWarpBytes;

// B bytes per K chunk: NT x 64 bf16; an MN-major TMA panel is whole 64-wide
// atoms (64 x 64 bf16 = 8 KB each).
template <int NT, bool BMN, bool TMA>
__host__ __device__ constexpr uint32_t b_chunk_bytes() {
  return (TMA && BMN) ? (uint32_t)((NT + 63) / 64) * 8192u : (uint32_t)NT * kKC * 2;
}

template <int NT, bool BMN = false, bool TMA = false>
__host__ __device__ inline WsCarve ws_carve(int64_t K, int64_t split) {
  WsCarve c;
  const uint32_t a_st = kM * kKC * 2, b_st = b_chunk_bytes<NT, BMN, TMA>();
  const int64_t nch = (K + kKC - 1) / kKC;
  const uint32_t tail = 1024 + kStgBytes;  // output staging + barriers + tmem slot
  const uint64_t bres_bytes = (uint64_t)nch * b_st;
  const uint64_t budget = kSmemMax - 1024;  // the launch adds 1 KB for the 1024-B alignment
  c.bres = 0;
  {  // streamed B: as many (A + B) stages as fit
    const uint64_t st = (budget - tail) / (a_st + b_st);
    c.stages = (uint32_t)(st < kMaxStages ? st : kMaxStages);
  }
  if (split <= 1 && bres_bytes + 2ull * a_st + tail <= budget) {  // resident B
    c.bres = 1;
    const uint64_t left = budget - bres_bytes - tail;
    c.stages = (uint32_t)(left / a_st < kMaxStages ? left / a_st : kMaxStages);
  }
  c.a = 0;
  c.b = c.stages * a_st;
  c.stg = c.b + (uint32_t)(c.bres ? bres_bytes : (uint64_t)c.stages * b_st);
  c.bar = c.stg + kStgBytes;
  c.bytes = c.bar + 1024;
  return c;
}

// Epilogue of one 128 x NT tile for epilogue warp ew (rows 32 ew + lane):
// each thread owns one output row and writes its 32-column segments directly
// with 16-byte vector stores (bias loads are warp-uniform broadcasts); a
// partial last segment or a misaligned destination falls back to scalars.
template <int NT, int EPI>
__device__ __forceinline__ void epilogue_tile(const wipes_gemm_args& g, int cb0, int cb1,
                                              uint32_t tacc, int ew, int lane, int64_t m0,
                                              int64_t n0, bool have, const void* tcmap,
                                              unsigned char* stg, const void* tmmap,
                                              uint64_t* mbar, uint32_t& mphase) {
  unsigned char* mstg = stg + 32 * 32 * 4;  // mask block (bf16, row-major)
  const int64_t m = m0 + 32 * ew + lane;
  const bool mrow = m < g.M;
  constexpr bool kBf16Out = EPI == WIPES_GEMM_EPI_BIAS_RELU_BF16 || EPI == WIPES_GEMM_EPI_MASK_BF16;
  const bool cvec = ((uintptr_t)g.C % 16 == 0) && (g.ldc % (kBf16Out ? 8 : 4) == 0);
  const bool mvec = EPI != WIPES_GEMM_EPI_MASK_BF16 ||
                    (((uintptr_t)g.mask % 16 == 0) && (g.ldm % 8 == 0));
#pragma unroll 1
  for (int cb = cb0; cb < cb1; ++cb) {
    float v[32];
    const bool tm = EPI == WIPES_GEMM_EPI_MASK_BF16 && tmmap != nullptr &&
                    32 * cb < NT && n0 + 32 * cb < g.N;
    if (tm) {  // fetch this block's ReLU mask with TMA while the accumulator is read
      __syncwarp();
      if (lane == 0) {
        mbar_expect_tx(mbar, 32 * 32 * 2);
        tma_load_2d(mstg, tmmap, (int)(n0 + 32 * cb), (int)(m0 + 32 * ew), mbar);
      }
    }
    if (have) {
      tmem_ld32(tacc + ((uint32_t)(32 * ew) << 16) + (uint32_t)(32 * cb), v);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
      if (EPI == WIPES_GEMM_EPI_ATOMIC_F32) continue;
    }
    const int tc = 32 * cb;
    const int64_t n = n0 + tc;
    if (tc >= NT || n >= g.N) continue;  // warp-uniform
    const bool full = tc + 32 <= NT && n + 32 <= g.N;
    const int nv = full ? 32 : (int)((g.N - n) < (NT - tc) ? (g.N - n) : (NT - tc));
    if (!mrow) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
    }
    if (EPI == WIPES_GEMM_EPI_BIAS_F32 || EPI == WIPES_GEMM_EPI_BIAS_RELU_BF16) {
      if (full && ((uintptr_t)(g.bias + n) % 16 == 0)) {
        const float4* b4 = reinterpret_cast<const float4*>(g.bias + n);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 b = __ldg(b4 + q);
          v[4 * q] += b.x; v[4 * q + 1] += b.y; v[4 * q + 2] += b.z; v[4 * q + 3] += b.w;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < nv) v[i] += g.bias[n + i];
      }
    }
    if (EPI == WIPES_GEMM_EPI_BIAS_RELU_BF16) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
    }
    if (tm) {
      mbar_wait(mbar, mphase);
      mphase ^= 1u;
      const uint4* mr = reinterpret_cast<const uint4*>(mstg + lane * 64);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 u = mr[q];
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const __nv_bfloat162 pr = *reinterpret_cast<const __nv_bfloat162*>(&w[h]);
          v[8 * q + 2 * h] = __low2float(pr) > 0.f ? v[8 * q + 2 * h] : 0.f;
          v[8 * q + 2 * h + 1] = __high2float(pr) > 0.f ? v[8 * q + 2 * h + 1] : 0.f;
        }
      }
    } else if (EPI == WIPES_GEMM_EPI_MASK_BF16 && mrow) {
      const __nv_bfloat16* mp = reinterpret_cast<const __nv_bfloat16*>(g.mask) + m * g.ldm + n;
      if (full && mvec) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 u = *reinterpret_cast<const uint4*>(mp + 8 * q);
          const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const __nv_bfloat162 pr = *reinterpret_cast<const __nv_bfloat162*>(&w[h]);
            v[8 * q + 2 * h] = __low2float(pr) > 0.f ? v[8 * q + 2 * h] : 0.f;
            v[8 * q + 2 * h + 1] = __high2float(pr) > 0.f ? v[8 * q + 2 * h + 1] : 0.f;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < nv) v[i] = __bfloat162float(mp[i]) > 0.f ? v[i] : 0.f;
      }
    }
    if (g.colsum) {
      // column sums over the warp's 32 rows by reduce-scatter (31 shuffles):
      // at each halving the lane with bit sz set keeps the upper half, so
      // lane l ends with the sum of column l of this block
      float w[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) w[i] = (i < nv) ? v[i] : 0.f;
#pragma unroll
      for (int sz = 16; sz >= 1; sz >>= 1) {
        const bool up = lane & sz;
#pragma unroll
        for (int i = 0; i < sz; ++i) {
          const float send = up ? w[i] : w[i + sz];
          const float keep = up ? w[i + sz] : w[i];
          w[i] = keep + __shfl_xor_sync(0xffffffffu, send, sz);
        }
      }
      if (lane < nv) atomicAdd(g.colsum + n + lane, w[0]);
    }
    if (EPI != WIPES_GEMM_EPI_ATOMIC_F32 && tcmap) {
      // stage the 32 x 32 block row-major in shared memory and let TMA write it
      // (out-of-range rows/columns are clipped by the tensor map bounds)
      if (lane == 0) bulk_wait_read();  // the previous block's store has read the buffer
      __syncwarp();
      if (kBf16Out && g.split3 > 0) {
        // split-bf16 triple through TMA: hi staged at stg, lo at stg + 2 KB
        uint4* row = reinterpret_cast<uint4*>(stg + lane * 64);
        uint4* rowl = reinterpret_cast<uint4*>(stg + 2048 + lane * 64);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 uh, ul;
          uint32_t* wh = reinterpret_cast<uint32_t*>(&uh);
          uint32_t* wl = reinterpret_cast<uint32_t*>(&ul);
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const float a = v[8 * q + 2 * h], b = v[8 * q + 2 * h + 1];
            const __nv_bfloat162 hi = __floats2bfloat162_rn(a, b);
            const __nv_bfloat162 lo =
                __floats2bfloat162_rn(a - __low2float(hi), b - __high2float(hi));
            wh[h] = *reinterpret_cast<const uint32_t*>(&hi);
            wl[h] = *reinterpret_cast<const uint32_t*>(&lo);
          }
          row[q] = uh;
          rowl[q] = ul;
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          const int rr = (int)(m0 + 32 * ew);
          tma_store_2d(tcmap, (int)n, rr, stg);
          tma_store_2d(tcmap, (int)(n + g.split3), rr, stg);
          tma_store_2d(tcmap, (int)(n + 2 * g.split3), rr, stg + 2048);
          bulk_commit();
        }
        continue;
      } else if (kBf16Out) {
        uint4* row = reinterpret_cast<uint4*>(stg + lane * 64);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const __nv_bfloat162 pr = __floats2bfloat162_rn(v[8 * q + 2 * h], v[8 * q + 2 * h + 1]);
            w[h] = *reinterpret_cast<const uint32_t*>(&pr);
          }
          row[q] = u;
        }
      } else {
        float4* row = reinterpret_cast<float4*>(stg + lane * 128);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          row[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tcmap, (int)n, (int)(m0 + 32 * ew), stg);
        bulk_commit();
      }
      continue;
    }
    if (!mrow) continue;
    if (EPI == WIPES_GEMM_EPI_ATOMIC_F32) {
      float* cp = reinterpret_cast<float*>(g.C) + m * g.ldc + n;
      if (full && cvec) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          atomicAdd(reinterpret_cast<float4*>(cp) + q,
                    make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < nv) atomicAdd(cp + i, v[i]);
      }
    } else if (kBf16Out && g.split3 > 0) {
      // split-bf16 triple (R38): hi at n and n + split3, lo at n + 2 split3
      __nv_bfloat16* cp = reinterpret_cast<__nv_bfloat16*>(g.C) + m * g.ldc + n;
      const int64_t s3 = g.split3;
      if (full && cvec && (s3 % 8) == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 uh, ul;
          uint32_t* wh = reinterpret_cast<uint32_t*>(&uh);
          uint32_t* wl = reinterpret_cast<uint32_t*>(&ul);
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const float a = v[8 * q + 2 * h], b = v[8 * q + 2 * h + 1];
            const __nv_bfloat162 hi = __floats2bfloat162_rn(a, b);
            const __nv_bfloat162 lo =
                __floats2bfloat162_rn(a - __low2float(hi), b - __high2float(hi));
            wh[h] = *reinterpret_cast<const uint32_t*>(&hi);
            wl[h] = *reinterpret_cast<const uint32_t*>(&lo);
          }
          reinterpret_cast<uint4*>(cp)[q] = uh;
          reinterpret_cast<uint4*>(cp + s3)[q] = uh;
          reinterpret_cast<uint4*>(cp + 2 * s3)[q] = ul;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < nv) {
            const __nv_bfloat16 hi = __float2bfloat16_rn(v[i]);
            cp[i] = hi;
            cp[i + s3] = hi;
            cp[i + 2 * s3] = __float2bfloat16_rn(v[i] - __bfloat162float(hi));
          }
      }
    } else if (kBf16Out) {
      __nv_bfloat16* cp = reinterpret_cast<__nv_bfloat16*>(g.C) + m * g.ldc + n;
      if (full && cvec) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const __nv_bfloat162 pr = __floats2bfloat162_rn(v[8 * q + 2 * h], v[8 * q + 2 * h + 1]);
            w[h] = *reinterpret_cast<const uint32_t*>(&pr);
          }
          reinterpret_cast<uint4*>(cp)[q] = u;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < nv) cp[i] = __float2bfloat16_rn(v[i]);
      }
    } else {
      float* cp = reinterpret_cast<float*>(g.C) + m * g.ldc + n;
      if (full && cvec) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          reinterpret_cast<float4*>(cp)[q] =
              make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < nv) cp[i] = v[i];
      }
    }
  }
}

// Kernel parameters: the ABI arguments plus, for the TMA path, one tensor map
// per operand (128-byte swizzle; K-major boxes 64 x rows, MN-major boxes
// 64 x 64) built on the host.
struct GemmParams {
  wipes_gemm_args g;
  CUtensorMap ta, tb, tc, tm;
  int32_t tstore;  // 1: the epilogue writes C with TMA stores through tc
  int32_t tmask;   // 1: the ReLU mask is fetched with TMA through tm
};

template <int NT, bool AMN, bool BMN, int EPI, bool TMA>
__global__ void __launch_bounds__(kWsThreads, 1) k_gemm_ws(const __grid_constant__ GemmParams P) {
  const wipes_gemm_args& g = P.g;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  constexpr int kCols = NT <= 32 ? 32 : (NT <= 64 ? 64 : (NT <= 128 ? 128 : 256));
  constexpr int kAlloc = 2 * kCols;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t mtiles = (g.M + kM - 1) / kM, ntiles = (g.N + NT - 1) / NT;
  const int64_t splits = g.split_k > 0 ? g.split_k : 1;
  const int64_t tiles = mtiles * ntiles * splits;
  const int64_t nchunk_all = (g.K + kKC - 1) / kKC;
  const int64_t per = (nchunk_all + splits - 1) / splits;
  const __nv_bfloat16* A = reinterpret_cast<const __nv_bfloat16*>(g.A);
  const __nv_bfloat16* B = reinterpret_cast<const __nv_bfloat16*>(g.B);
  // B stays resident (loaded once per CTA) when there is one N tile and no K split
  const WsCarve cv = ws_carve<NT, BMN, TMA>(g.K, (splits > 1 || ntiles > 1) ? 2 : 1);
  const int S = (int)cv.stages;
  // 128-byte swizzle atoms need 1024-byte aligned buffers (the launch adds 1 KB)
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __nv_bfloat16* sa = reinterpret_cast<__nv_bfloat16*>(base + cv.a);
  __nv_bfloat16* sb = reinterpret_cast<__nv_bfloat16*>(base + cv.b);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + cv.bar);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* bfull = tempty + 2;
  uint64_t* mbars = bfull + 1;  // one per epilogue warp (TMA mask loads)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbars + 8);
  constexpr int kAst = kM * kKC;                                // A elements per stage
  constexpr int kBst = b_chunk_bytes<NT, BMN, TMA>() / 2;      // B elements per chunk

  if (warp == kAllocWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "n"(kAlloc));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < kMaxStages; ++i) {
      mbar_init(&full[i], TMA ? 1 : kProd);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 32 * kEpiWarps);
    }
    mbar_init(bfull, TMA ? 1 : kProd);
    for (int i = 0; i < 8; ++i) mbar_init(&mbars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  auto tile_coords = [&](int64_t t, int64_t& m0, int64_t& n0, int64_t& c_lo, int64_t& nch) {
    const int64_t mt = t % mtiles, nt = (t / mtiles) % ntiles, ks = t / (mtiles * ntiles);
    m0 = mt * kM;
    n0 = nt * NT;
    c_lo = per * ks;
    const int64_t c_hi = c_lo + per < nchunk_all ? c_lo + per : nchunk_all;
    nch = c_hi > c_lo ? c_hi - c_lo : 0;
  };

  // TMA loads of one K chunk: K-major = one box (64 K x rows); MN-major = one
  // 64 x 64 box per 64-wide M/N atom.
  auto tma_a = [&](__nv_bfloat16* dst, int64_t m0, int64_t k0, uint64_t* bar) {
    if (!AMN) tma_load_2d(dst, &P.ta, (int)k0, (int)m0, bar);
    else
      for (int q = 0; q < kM / 64; ++q) tma_load_2d(dst + q * 4096, &P.ta, (int)(m0 + 64 * q), (int)k0, bar);
  };
  auto tma_b = [&](__nv_bfloat16* dst, int64_t n0, int64_t k0, uint64_t* bar) {
    if (!BMN) tma_load_2d(dst, &P.tb, (int)k0, (int)n0, bar);
    else
      for (int q = 0; q < (NT + 63) / 64; ++q)
        tma_load_2d(dst + q * 4096, &P.tb, (int)(n0 + 64 * q), (int)k0, bar);
  };
  constexpr uint32_t kABytes = kM * kKC * 2, kBBytes = b_chunk_bytes<NT, BMN, TMA>();

  if (TMA && warp == 0) {  // ------------------------------ TMA producer (1 lane)
    if (lane == 0) {
      int64_t it = 0, loaded_n0 = -1;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        int64_t m0, n0, c_lo, nch;
        tile_coords(t, m0, n0, c_lo, nch);
        if (cv.bres && n0 != loaded_n0) {
          mbar_expect_tx(bfull, (uint32_t)(nchunk_all * kBBytes));
          for (int64_t c = 0; c < nchunk_all; ++c) tma_b(sb + c * kBst, n0, c * kKC, bfull);
          loaded_n0 = n0;
        }
        for (int64_t c = 0; c < nch; ++c, ++it) {
          const int st = (int)(it % S);
          const uint32_t round = (uint32_t)(it / S);
          mbar_wait(&empty[st], (round & 1u) ^ 1u);
          const int64_t k0 = (c_lo + c) * kKC;
          mbar_expect_tx(&full[st], kABytes + (cv.bres ? 0u : kBBytes));
          tma_a(sa + st * kAst, m0, k0, &full[st]);
          if (!cv.bres) tma_b(sb + st * kBst, n0, k0, &full[st]);
        }
      }
    }
  } else if (!TMA && warp < kProdWarps) {  // --------------------- producers
    int64_t it = 0, loaded_n0 = -1;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      int64_t m0, n0, c_lo, nch;
      tile_coords(t, m0, n0, c_lo, nch);
      if (cv.bres && n0 != loaded_n0) {
        // load the resident B panel once (single N tile); the MMA warp waits
        // on bfull before its first MMA
        for (int64_t c = 0; c < nchunk_all; ++c)
          stage<NT, BMN, kProd>(sb + c * kBst, B, g.ldb, n0, g.N, c * kKC, g.K, tid);
        cp_async_arrive(bfull);
        loaded_n0 = n0;
      }
      for (int64_t c = 0; c < nch; ++c, ++it) {
        const int st = (int)(it % S);
        const uint32_t round = (uint32_t)(it / S);
        mbar_wait(&empty[st], (round & 1u) ^ 1u);
        const int64_t k0 = (c_lo + c) * kKC;
        stage<kM, AMN, kProd>(sa + st * kAst, A, g.lda, m0, g.M, k0, g.K, tid);
        if (!cv.bres) stage<NT, BMN, kProd>(sb + st * kBst, B, g.ldb, n0, g.N, k0, g.K, tid);
        cp_async_arrive(&full[st]);
      }
    }
  } else if (warp == kMmaWarp) {  // ------------------------------- MMA issuer
    const uint32_t idesc = instr_desc(NT, AMN, BMN);
    int64_t it = 0, tcount = 0, loaded_n0 = -1;
    uint32_t bphase = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++tcount) {
      int64_t m0, n0, c_lo, nch;
      tile_coords(t, m0, n0, c_lo, nch);
      if (cv.bres && n0 != loaded_n0) {  // once: resident mode has one N tile
        mbar_wait(bfull, bphase);
        bphase ^= 1u;
        loaded_n0 = n0;
      }
      const int acc = (int)(tcount & 1);
      const uint32_t tround = (uint32_t)(tcount >> 1);
      mbar_wait(&tempty[acc], (tround & 1u) ^ 1u);
      tc_fence_after();
      const uint32_t d = tmem + (uint32_t)(acc * kCols);
      for (int64_t c = 0; c < nch; ++c, ++it) {
        const int st = (int)(it % S);
        const uint32_t round = (uint32_t)(it / S);
        mbar_wait(&full[st], round & 1u);
        if (!TMA) fence_proxy_async();  // cp.async (generic proxy) -> tensor core reads
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a0 = smem_u32(sa + st * kAst);
          const uint32_t b0 = smem_u32(sb + (cv.bres ? (c_lo + c) : st) * kBst);
#pragma unroll
          for (int j = 0; j < kKC / 16; ++j) {
            uint64_t da, db;
            if (TMA) {  // 128-byte swizzled tiles written by TMA
              da = AMN ? smem_desc_sw128(a0 + 2048 * j, 8192, 1024)
                       : smem_desc_sw128(a0 + 32 * j, 16, 1024);
              db = BMN ? smem_desc_sw128(b0 + 2048 * j, 8192, 1024)
                       : smem_desc_sw128(b0 + 32 * j, 16, 1024);
            } else {
              da = smem_desc(a0 + 256 * j, 128, 1024);
              db = smem_desc(b0 + 256 * j, 128, 1024);
            }
            mma_bf16(d, da, db, idesc, (c > 0 || j > 0) ? 1u : 0u);
          }
          mma_commit(&empty[st]);
        }
        __syncwarp();
      }
      if (lane == 0) mma_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if (warp >= kEpiWarp0) {  // ------------------------------- epilogue
    const int e = warp - kEpiWarp0;
    const int ew = e & 3;  // TMEM lane quarter (warp % 4)
    constexpr int kBlocks = (NT + 31) / 32;
    const int half = e >> 2, nh = kEpiWarps / 4;
    const int cb0 = kBlocks * half / nh, cb1 = kBlocks * (half + 1) / nh;
    int64_t tcount = 0;
    uint32_t mphase = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++tcount) {
      int64_t m0, n0, c_lo, nch;
      tile_coords(t, m0, n0, c_lo, nch);
      const int acc = (int)(tcount & 1);
      mbar_wait(&tfull[acc], (uint32_t)((tcount >> 1) & 1));
      tc_fence_after();
      epilogue_tile<NT, EPI>(g, cb0, cb1, tmem + (uint32_t)(acc * kCols), ew, lane, m0, n0,
                             nch > 0, P.tstore ? (const void*)&P.tc : nullptr,
                             base + cv.stg + e * kStgWarpBytes,
                             P.tmask ? (const void*)&P.tm : nullptr, &mbars[e], mphase);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
    if (P.tstore && lane == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kAllocWarp)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "n"(kAlloc));
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Tensor map of a bf16 operand with `rows` M/N rows and K columns.
bool make_tmap(CUtensorMap* m, const void* ptr, bool mn, int64_t rows, int64_t K, int64_t ld,
               int box_rows) {
  auto enc = tmap_encoder();
  if (!enc) return false;
  cuuint64_t dims[2], strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2], es[2] = {1, 1};
  if (!mn) { dims[0] = (cuuint64_t)K; dims[1] = (cuuint64_t)rows; box[0] = 64; box[1] = (cuuint32_t)box_rows; }
  else { dims[0] = (cuuint64_t)rows; dims[1] = (cuuint64_t)K; box[0] = 64; box[1] = 64; }
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Output tensor map: C [M, N] (row pitch ldc), 32 x 32 boxes, no swizzle.
bool make_out_tmap(CUtensorMap* m, const void* ptr, bool bf16, int64_t M, int64_t N, int64_t ldc) {
  auto enc = tmap_encoder();
  const int esz = bf16 ? 2 : 4;
  if (!enc || (uintptr_t)ptr % 16 != 0 || (ldc * esz) % 16 != 0) return false;
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M}, strides[1] = {(cuuint64_t)(ldc * esz)};
  cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
  return enc(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
             const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NT, bool AMN, bool BMN, int EPI, bool TMA>
cudaError_t launch_ws_t(const GemmParams& P, cudaStream_t s) {
  const wipes_gemm_args& g = P.g;
  auto k = k_gemm_ws<NT, AMN, BMN, EPI, TMA>;
  static int sms = 0;
  if (!sms) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemMax);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int64_t ntiles = (g.N + NT - 1) / NT;
  const int64_t splits = g.split_k > 0 ? g.split_k : 1;
  const WsCarve cv = ws_carve<NT, BMN, TMA>(g.K, (splits > 1 || ntiles > 1) ? 2 : 1);
  const int64_t tiles = ((g.M + kM - 1) / kM) * ntiles * splits;
  const unsigned grid = (unsigned)(tiles < sms ? tiles : sms);
  launch_begin(K_GEMM, s);
  k<<<grid, kWsThreads, cv.bytes + 1024, s>>>(P);
  launch_end(K_GEMM, s);
  return cudaGetLastError();
}

template <int NT, bool AMN, bool BMN, int EPI>
cudaError_t launch_ws(const wipes_gemm_args& g, cudaStream_t s) {
  GemmParams P;
  P.g = g;
  std::memset(&P.ta, 0, sizeof(P.ta));
  std::memset(&P.tb, 0, sizeof(P.tb));
  // TMA needs 16-byte aligned bases and row pitches (the ABI requires both)
  if (!make_tmap(&P.ta, g.A, AMN, g.M, g.K, g.lda, kM) ||
      !make_tmap(&P.tb, g.B, BMN, g.N, g.K, g.ldb, NT))
    return cudaErrorInvalidValue;
  std::memset(&P.tc, 0, sizeof(P.tc));
  std::memset(&P.tm, 0, sizeof(P.tm));
  P.tmask = EPI == WIPES_GEMM_EPI_MASK_BF16 && make_out_tmap(&P.tm, g.mask, true, g.M, g.N, g.ldm);
  // split3: one map over the three blocks (3 split3 columns); only when the
  // blocks are whole 32-column boxes (a partial box would spill into the next block)
  const bool s3ok = g.split3 == 0 || (g.N == g.split3 && g.N % 32 == 0);
  P.tstore = EPI != WIPES_GEMM_EPI_ATOMIC_F32 && s3ok &&
             make_out_tmap(&P.tc, g.C,
                           EPI == WIPES_GEMM_EPI_BIAS_RELU_BF16 || EPI == WIPES_GEMM_EPI_MASK_BF16,
                           g.M, g.split3 ? 3 * g.split3 : g.N, g.ldc);
#ifdef WIPES_GEMM_CPASYNC  // cp.async staging variant (experiments / cross-checks)
  return launch_ws_t<NT, AMN, BMN, EPI, false>(P, s);
#else
  return launch_ws_t<NT, AMN, BMN, EPI, true>(P, s);
#endif
}

template <int NT, bool AMN, bool BMN, int EPI>
cudaError_t launch_nt(const wipes_gemm_args& g, cudaStream_t s) {
  return launch_ws<NT, AMN, BMN, EPI>(g, s);
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
}  // namespace wipes
