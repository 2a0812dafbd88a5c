// NEXT-4 fused forward of the deformation field (DESIGN.md NEXT-4): every
// layer of one 128-row tile runs back to back with the activations kept in
// shared memory, so HBM sees only the canonical parameters in and the frame
// rows out (plus, when training, one store of each layer's activations for
// the backward).
//
// One CTA per SM, persistent over 128-row tiles:
//   warp 0      TMA producer: streams every layer's bf16 weights (K chunks of
//               64, 128-byte swizzle) through a ring (weights do not depend on
//               the tile, so it runs a layer or more ahead);
//   warp 1      one lane issues tcgen05.mma (M = 128, N = width or 16) per
//               chunk: A = the activation tile in shared memory, B = the ring
//               stage; commits each chunk to empty[s] and each layer to accf;
//   warp 2      owns the TMEM accumulator (256 columns);
//   warps 4-11  epilogue (two warps per TMEM lane quarter, one per column
//               half): the positional encoding at tile start, then per layer
//               bias + ReLU -> bf16 -> the activation tile (written in the
//               SW128 K-major layout the next MMA reads), optional TMA stores
//               of the activations, and the head's apply into the frame rows.
// Activation tile X: 6 chunks of [128 rows x 64 bf16]: chunks 0-1 hold the
// encoding (zero padded to 128 columns), chunks 2-5 hold h (width <= 256).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

#include "gemm_tc.cuh"

namespace wipes {

namespace {

using namespace tc;

constexpr int kFMaxD = 8;
constexpr int kFMaxFrames = 128;
constexpr int kFStages = 4;  // a whole 256-wide layer of weights in flight (224 KB with X)
#ifndef WIPES_FWD_EPI_WARPS
#define WIPES_FWD_EPI_WARPS 16
#endif
constexpr int kFEpiWarps = WIPES_FWD_EPI_WARPS;  // forward epilogue: 4 per TMEM lane quarter
constexpr int kFParts = kFEpiWarps / 4;          // column parts per lane quarter
constexpr int kFThreads = 32 * (4 + kFEpiWarps);
constexpr int kBEpiWarps = 8;                    // layer backward epilogue
constexpr uint32_t kXChunk = 128 * 64 * 2;  // 16 KB

struct FusedArgs {
  int32_t W, D, skip, Lx, Lt, E8, catw, train, shc;
  int64_t N, M;
  float t[kFMaxFrames];
  const float* theta;
  int64_t thb[kFMaxD], thbh;
  wipes_params canon, frame;
  float* out;  // [M, 16] head outputs (training)
  CUtensorMap wl[kFMaxD + 1];  // weights per layer (the skip layer's h part in wl[kFMaxD])
  CUtensorMap wh;              // head weights [16, W]
  CUtensorMap hs[kFMaxD];      // activation stores (training)
  CUtensorMap cate, cath;      // concat buffer: encoding part / h part (training)
};

// The K chunks of layer l (l == D: head) and which X chunk / weight map / k0 each uses.
__device__ __forceinline__ int layer_chunks(const FusedArgs& a, int l) {
  if (l == a.D) return a.W / 64;
  if (l == 0) return 2;
  if (l == a.skip + 1) return 2 + a.W / 64;
  return a.W / 64;
}

__device__ __forceinline__ void chunk_info(const FusedArgs& a, int l, int c, int& xchunk,
                                           const CUtensorMap*& map, int& k0) {
  if (l == a.D) { xchunk = 2 + c; map = &a.wh; k0 = 64 * c; return; }
  if (l == 0) { xchunk = c; map = &a.wl[0]; k0 = 64 * c; return; }
  if (l == a.skip + 1) {
    if (c < 2) { xchunk = c; map = &a.wl[l]; k0 = 64 * c; }
    else { xchunk = c; map = &a.wl[kFMaxD]; k0 = 64 * (c - 2); }
    return;
  }
  xchunk = 2 + c; map = &a.wl[l]; k0 = 64 * c;
}

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// store 8 bf16 (one 16-byte unit) of row r, column c0 (multiple of 8) into X
__device__ __forceinline__ void x_store8(unsigned char* X, int r, int c0, const uint4& u) {
  const int chunk = c0 >> 6, unit = (c0 & 63) >> 3;
  *reinterpret_cast<uint4*>(X + chunk * kXChunk + r * 128 + ((unit ^ (r & 7)) << 4)) = u;
}

__device__ __forceinline__ uint4 pack8(const float* v) {
  uint4 u;
  uint32_t* w = reinterpret_cast<uint32_t*>(&u);
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const __nv_bfloat162 p = __floats2bfloat162_rn(v[2 * h], v[2 * h + 1]);
    w[h] = *reinterpret_cast<const uint32_t*>(&p);
  }
  return u;
}

__global__ void __launch_bounds__(kFThreads, 1) k_mlp_fused_fwd(const __grid_constant__ FusedArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* X = base;                                  // 6 x 16 KB
  unsigned char* ring = base + 6 * kXChunk;                 // kFStages x (256 x 64 bf16)
  constexpr uint32_t kStage = 256 * 64 * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kFStages * kStage);
  uint64_t* empty = full + kFStages;
  uint64_t* xready = empty + kFStages;
  uint64_t* accf = xready + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accf + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tiles = (a.M + 127) / 128;

  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < kFStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(xready, 1);
    mbar_init(accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {  // ------------------------------------------- TMA producer
    if (lane == 0) {
      int64_t it = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x)
        for (int l = 0; l <= a.D; ++l) {
          const int nch = layer_chunks(a, l);
          for (int c = 0; c < nch; ++c, ++it) {
            const int st = (int)(it % kFStages);
            const uint32_t round = (uint32_t)(it / kFStages);
            mbar_wait(&empty[st], (round & 1u) ^ 1u);
            int xc, k0;
            const CUtensorMap* map;
            chunk_info(a, l, c, xc, map, k0);
            mbar_expect_tx(&full[st], l == a.D ? 16 * 128 : (uint32_t)a.W * 128);
            tma_load_2d(ring + st * kStage, map, k0, 0, &full[st]);
          }
        }
    }
  } else if (warp == 1) {  // -------------------------------------- MMA issuer
    const uint32_t id_l = instr_desc(a.W, false, false), id_h = instr_desc(16, false, false);
    int64_t it = 0;
    uint32_t xph = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x)
      for (int l = 0; l <= a.D; ++l) {
        mbar_wait(xready, xph);
        xph ^= 1u;
        tc_fence_after();
        const int nch = layer_chunks(a, l);
        for (int c = 0; c < nch; ++c, ++it) {
          const int st = (int)(it % kFStages);
          const uint32_t round = (uint32_t)(it / kFStages);
          mbar_wait(&full[st], round & 1u);
          tc_fence_after();
          if (lane == 0) {
            int xc, k0;
            const CUtensorMap* map;
            chunk_info(a, l, c, xc, map, k0);
            const uint32_t a0 = smem_u32(X + xc * kXChunk), b0 = smem_u32(ring + st * kStage);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              mma_bf16(tmem, smem_desc_sw128(a0 + 32 * j, 16, 1024),
                       smem_desc_sw128(b0 + 32 * j, 16, 1024), l == a.D ? id_h : id_l,
                       (c > 0 || j > 0) ? 1u : 0u);
            mma_commit(&empty[st]);
          }
          __syncwarp();
        }
        if (lane == 0) mma_commit(accf);
        __syncwarp();
      }
  } else if (warp >= 4) {  // -------------------------------------- epilogue
    const int e = warp - 4, q = e & 3, half = e >> 2;  // half: column part 0 .. kFParts - 1
    const int r = 32 * q + lane;  // tile row = TMEM lane
    const int nb = a.W / 32, cb0 = half * nb / kFParts, cb1 = (half + 1) * nb / kFParts;
    const bool issuer = (e == 0 && lane == 0);
    uint32_t aph = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int64_t m0 = t * 128, m = m0 + r;
      const bool mrow = m < a.M;
      // ---- positional encoding of row r into X chunks 0-1 (zero padded) ----
      if (issuer) bulk_wait_read();  // previous tile's stores have read X
      named_sync(1, 32 * kFEpiWarps);
      if (half == 0) {
        float x[3] = {0.f, 0.f, 0.f}, tt = 0.f;
        if (mrow) {
          const int64_t f = m / a.N, i = m - f * a.N;
          x[0] = a.canon.mean[3 * i]; x[1] = a.canon.mean[3 * i + 1]; x[2] = a.canon.mean[3 * i + 2];
          tt = a.t[f];
        }
        float buf[8];
        int n = 0, c0 = 0;
        auto push = [&](float v) {
          buf[n++] = v;
          if (n == 8) { x_store8(X, r, c0, pack8(buf)); c0 += 8; n = 0; }
        };
        for (int d = 0; d < 3; ++d) push(x[d]);
        for (int k = 0; k < a.Lx; ++k) {
          float sn[3], cs[3];
          for (int d = 0; d < 3; ++d) sincosf((float)(1 << k) * x[d], &sn[d], &cs[d]);
          for (int d = 0; d < 3; ++d) push(sn[d]);
          for (int d = 0; d < 3; ++d) push(cs[d]);
        }
        push(tt);
        for (int k = 0; k < a.Lt; ++k) {
          float sn, cs;
          sincosf((float)(1 << k) * tt, &sn, &cs);
          push(sn);
          push(cs);
        }
        while (c0 < 128) push(0.f);
      }
      fence_proxy_async();
      named_sync(1, 32 * kFEpiWarps);
      if (issuer) {
        if (a.train) {
          tma_store_2d(&a.cate, 0, (int)m0, X);
          tma_store_2d(&a.cate, 64, (int)m0, X + kXChunk);
          bulk_commit();
        }
        mbar_arrive(xready);
      }
      // ---- layers -----------------------------------------------------------
      for (int l = 0; l <= a.D; ++l) {
        mbar_wait(accf, aph);
        aph ^= 1u;
        tc_fence_after();
        if (l < a.D) {
          if (issuer) bulk_wait_read();  // X chunks 2-5 free of pending stores
          named_sync(1, 32 * kFEpiWarps);
          const float* bias = a.theta + a.thb[l];
          for (int cb = cb0; cb < cb1; ++cb) {
            float v[32];
            tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(32 * cb), v);
            const float4* b4 = reinterpret_cast<const float4*>(bias + 32 * cb);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const float4 b = __ldg(b4 + k);
              v[4 * k] = fmaxf(v[4 * k] + b.x, 0.f);
              v[4 * k + 1] = fmaxf(v[4 * k + 1] + b.y, 0.f);
              v[4 * k + 2] = fmaxf(v[4 * k + 2] + b.z, 0.f);
              v[4 * k + 3] = fmaxf(v[4 * k + 3] + b.w, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) x_store8(X + 2 * kXChunk, r, 32 * cb + 8 * u, pack8(v + 8 * u));
          }
          tc_fence_before();
          fence_proxy_async();
          named_sync(1, 32 * kFEpiWarps);
          if (issuer) {
            if (a.train) {
              const CUtensorMap* hm = l == a.skip ? &a.cath : &a.hs[l];
              for (int j = 0; j < a.W / 64; ++j)
                tma_store_2d(hm, 64 * j, (int)m0, X + (2 + j) * kXChunk);
              bulk_commit();
            }
            mbar_arrive(xready);
          }
        } else {  // head: bias, then the frame rows (and the outputs for the backward)
          float v[32];
          tmem_ld32(tmem + ((uint32_t)(32 * q) << 16), v);
          tc_fence_before();
          if (half == 0 && mrow) {
            const int64_t i = m % a.N;
            for (int k = 0; k < 13; ++k) v[k] += a.theta[a.thbh + k];
            float* fm = const_cast<float*>(a.frame.mean);
            float* fq = const_cast<float*>(a.frame.quat);
            float* fs = const_cast<float*>(a.frame.scale);
            float* ff = const_cast<float*>(a.frame.freq);
            for (int d = 0; d < 3; ++d) fm[3 * m + d] = a.canon.mean[3 * i + d] + v[d];
            for (int d = 0; d < 4; ++d) fq[4 * m + d] = a.canon.quat[4 * i + d] + v[3 + d];
            for (int d = 0; d < 3; ++d) fs[3 * m + d] = a.canon.scale[3 * i + d] * expf(v[7 + d]);
            for (int d = 0; d < 3; ++d) ff[3 * m + d] = a.canon.freq[3 * i + d] + v[10 + d];
            if (a.canon.phase && a.frame.phase) const_cast<float*>(a.frame.phase)[m] = a.canon.phase[i];
            if (a.canon.opacity && a.frame.opacity)
              const_cast<float*>(a.frame.opacity)[m] = a.canon.opacity[i];
            if (a.canon.color && a.frame.color)
              for (int d = 0; d < 3; ++d)
                const_cast<float*>(a.frame.color)[3 * m + d] = a.canon.color[3 * i + d];
            if (a.canon.sh && a.frame.sh)
              for (int d = 0; d < 3 * a.shc; ++d)
                const_cast<float*>(a.frame.sh)[3 * a.shc * m + d] = a.canon.sh[3 * a.shc * i + d];
            if (a.train) {
              float4* o = reinterpret_cast<float4*>(a.out + m * 16);
              o[0] = make_float4(v[0], v[1], v[2], v[3]);
              o[1] = make_float4(v[4], v[5], v[6], v[7]);
              o[2] = make_float4(v[8], v[9], v[10], v[11]);
              o[3] = make_float4(v[12], 0.f, 0.f, 0.f);
            }
          }
        }
      }
    }
    if (issuer) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

// ---------------------------------------------------------------------------
// Fused backward of one hidden layer (width 256): the two GEMMs of a layer's
// backward read the same operands (dz_l and the layer input h_(l-1), which is
// also the ReLU mask), so one pass computes both:
//   dz_(l-1) = (dz_l W_l) * (h_(l-1) > 0)      [M, 256] bf16
//   dW_l     = dz_l^T h_(l-1)                   [256, 256] fp32 (per-group partials)
//   db_(l-1) = colsum(dz_(l-1))                 (per-group partials)
// CTA pairs ("groups") walk the same 128-row tiles; member m owns input
// columns [128 m, 128 m + 128): its slice of dW (all 256 rows), the same
// columns of dz_(l-1), and the matching half of the mask. Both members load
// the whole dz tile (the second read hits L2), so HBM sees dz and h once and
// dz_(l-1) once per layer, against twice and once for the two-GEMM schedule.
// Per CTA: W slice resident (64 KB, MN-major B of the dIn MMA), dz tiles in a
// ring of 3 x 32 KB halves (K-major A of dIn, MN-major A of dW: the same
// SW128 bytes serve both), h tiles in a ring of 2 x 32 KB (MN-major B of dW,
// mask of the epilogue). TMEM: dIn accumulator double-buffered (2 x 128
// columns) + dW halves (2 x 128 columns, accumulated over all the group's tiles).
constexpr int kBThreads = 32 * (4 + kBEpiWarps);
constexpr uint32_t kHalf = 32768;  // 128 rows x 128 columns bf16 (two SW128 boxes)

struct BwdArgs {
  int64_t M;
  int32_t groups;
  float* wpart;
  float* bpart;
  __nv_bfloat16* dzo;
  CUtensorMap tdz, tact, tw;
};

__global__ void __launch_bounds__(kBThreads, 1) k_mlp_bwd_layer(const __grid_constant__ BwdArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* Wsl = base;                 // 2 boxes [256 rows (out) x 64 in]
  unsigned char* dzr = base + 2 * kHalf;     // 3 x 32 KB
  unsigned char* actr = dzr + 3 * kHalf;     // 2 x 32 KB
  uint64_t* fdz = reinterpret_cast<uint64_t*>(actr + 2 * kHalf);
  uint64_t* edz = fdz + 3;
  uint64_t* fact = edz + 3;
  uint64_t* eact = fact + 2;
  uint64_t* accf = eact + 2;
  uint64_t* acce = accf + 2;
  uint64_t* wbar = acce + 2;
  uint64_t* dwdone = wbar + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dwdone + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int member = blockIdx.x & 1, grp = blockIdx.x >> 1;
  const int c0 = 128 * member;
  const int64_t tiles = (a.M + 127) / 128;

  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) { mbar_init(&fdz[i], 1); mbar_init(&edz[i], 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&fact[i], 1);
      mbar_init(&eact[i], 1 + kBEpiWarps);  // the dW MMAs and the epilogue's mask reads
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], kBEpiWarps);
    }
    mbar_init(wbar, 1);
    mbar_init(dwdone, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {  // ------------------------------------------- TMA producer
    if (lane == 0) {
      mbar_expect_tx(wbar, 2 * kHalf);
      tma_load_2d(Wsl, &a.tw, c0, 0, wbar);
      tma_load_2d(Wsl + kHalf, &a.tw, c0 + 64, 0, wbar);
      int64_t k = 0;
      for (int64_t t = grp; t < tiles; t += a.groups, ++k) {
        const int m0 = (int)(t * 128);
        for (int h = 0; h < 2; ++h) {
          const int64_t q = 2 * k + h;
          const int st = (int)(q % 3);
          mbar_wait(&edz[st], ((uint32_t)(q / 3) & 1u) ^ 1u);
          mbar_expect_tx(&fdz[st], kHalf);
          tma_load_2d(dzr + st * kHalf, &a.tdz, 128 * h, m0, &fdz[st]);
          tma_load_2d(dzr + st * kHalf + kHalf / 2, &a.tdz, 128 * h + 64, m0, &fdz[st]);
          if (h == 0) {  // the mask/B tile between the two dz halves (MMA order)
            const int sa = (int)(k & 1);
            mbar_wait(&eact[sa], ((uint32_t)(k >> 1) & 1u) ^ 1u);
            mbar_expect_tx(&fact[sa], kHalf);
            tma_load_2d(actr + sa * kHalf, &a.tact, c0, m0, &fact[sa]);
            tma_load_2d(actr + sa * kHalf + kHalf / 2, &a.tact, c0 + 64, m0, &fact[sa]);
          }
        }
      }
    }
  } else if (warp == 1) {  // -------------------------------------- MMA issuer
    // dIn is computed transposed, D[i, r] = sum_j W[j, i] dz[r, j] (A = the W slice,
    // MN-major; B = the dz tile, K-major), so TMEM lanes are columns and the
    // epilogue's stores and column sums run along rows
    const uint32_t id_in = instr_desc(128, true, false), id_w = instr_desc(128, true, true);
    mbar_wait(wbar, 0);
    tc_fence_after();
    const uint32_t wb = smem_u32(Wsl);
    int64_t k = 0;
    for (int64_t t = grp; t < tiles; t += a.groups, ++k) {
      const int b = (int)(k & 1), sa = (int)(k & 1);
      const uint32_t tin = tmem + 128u * b;
      mbar_wait(&acce[b], ((uint32_t)(k >> 1) & 1u) ^ 1u);  // epilogue drained buffer b
      tc_fence_after();
      for (int h = 0; h < 2; ++h) {
        const int64_t q = 2 * k + h;
        const int st = (int)(q % 3);
        mbar_wait(&fdz[st], (uint32_t)(q / 3) & 1u);
        tc_fence_after();
        const uint32_t dzb = smem_u32(dzr + st * kHalf);
        if (lane == 0) {
          // dIn^T: K = dz features 128 h .. 128 h + 127 (two K-major boxes)
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            const int ks = 8 * h + s;  // global K16 step (out features 16 ks ..)
            mma_bf16(tin, smem_desc_sw128(wb + 2048 * ks, kHalf, 1024),
                     smem_desc_sw128(dzb + (s >> 2) * (kHalf / 2) + 32 * (s & 3), 16, 1024), id_in,
                     ks > 0 ? 1u : 0u);
          }
          if (h == 1) mma_commit(&accf[b]);
        }
        __syncwarp();
        if (h == 0) {
          mbar_wait(&fact[sa], (uint32_t)(k >> 1) & 1u);
          tc_fence_after();
        }
        const uint32_t acb = smem_u32(actr + sa * kHalf);
        if (lane == 0) {
          // dW half h: M = out features (MN-major dz), N = in columns (MN-major act), K = rows
#pragma unroll
          for (int s = 0; s < 8; ++s)
            mma_bf16(tmem + 256u + 128u * h, smem_desc_sw128(dzb + 2048 * s, kHalf / 2, 1024),
                     smem_desc_sw128(acb + 2048 * s, kHalf / 2, 1024), id_w,
                     (k > 0 || s > 0) ? 1u : 0u);
          mma_commit(&edz[st]);
          if (h == 1) mma_commit(&eact[sa]);
        }
        __syncwarp();
      }
    }
    if (lane == 0) mma_commit(dwdone);
    __syncwarp();
  } else if (warp >= 4) {  // -------------------------------------- epilogue
    const int e = warp - 4, q = e & 3, half = e >> 2;
    const int r = 32 * q + lane;  // TMEM lane: dIn column c0 + r; dW row 128 half + r
    const int ci = r;             // this thread's dIn column within the slice
    // mask bytes of column ci in row ro of an h slot (SW128 box ci / 64)
    const uint32_t mcol = (ci >> 6) * (kHalf / 2) + (((ci & 63) >> 3) << 4) + (ci & 7) * 2;
    float cs = 0.f;  // column sum over this thread's rows (64 half .. 64 half + 63 of each tile)
    int64_t k = 0;
    for (int64_t t = grp; t < tiles; t += a.groups, ++k) {
      const int b = (int)(k & 1), sa = (int)(k & 1);
      mbar_wait(&accf[b], (uint32_t)(k >> 1) & 1u);
      mbar_wait(&fact[sa], (uint32_t)(k >> 1) & 1u);  // mask bytes visible to this thread
      tc_fence_after();
      float v[64];
      {
        float v0[32], v1[32];
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + 128u * b + 64u * half;
        tmem_ld32(ta, v0);
        tmem_ld32(ta + 32u, v1);
#pragma unroll
        for (int i = 0; i < 32; ++i) { v[i] = v0[i]; v[32 + i] = v1[i]; }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[b]);
      const unsigned char* slot = actr + sa * kHalf;
      const int64_t m0 = t * 128 + 64 * half;
      __nv_bfloat16* dst = a.dzo + m0 * 256 + c0 + ci;
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int ro = 64 * half + j;  // tile row
        const __nv_bfloat16 mv =
            *reinterpret_cast<const __nv_bfloat16*>(slot + ro * 128 + (mcol ^ ((ro & 7) << 4)));
        const float x = __bfloat162float(mv) > 0.f ? v[j] : 0.f;
        cs += x;  // rows >= M hold zeros (TMA zero fill)
        if (m0 + j < a.M) dst[(int64_t)j * 256] = __float2bfloat16_rn(x);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&eact[sa]);
    }
    a.bpart[((int64_t)grp * 2 + half) * 256 + c0 + ci] = cs;
    // dW slice: TMEM lanes = out features 128 half + r, columns = in c0 ..
    mbar_wait(dwdone, 0);
    tc_fence_after();
    float* wp = a.wpart + ((int64_t)grp * 256 + 128 * half + r) * 256 + c0;
#pragma unroll 1
    for (int cb = 0; cb < 4; ++cb) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 256u + 128u * half + 32u * cb, v);
      float4* d4 = reinterpret_cast<float4*>(wp + 32 * cb);
#pragma unroll
      for (int i = 0; i < 8; ++i) d4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

// ---------------------------------------------------------------------------
// One hidden layer's forward (width 256) in the same shape as the layer
// backward: CTA pairs walk the same 128-row tiles and member m owns output
// columns [128 m, 128 m + 128) — its W slice (128 x 256 bf16, 64 KB) stays
// resident as the K-major A operand, the x tiles stream through a ring of four
// 32 KB halves as the K-major B operand, and the accumulator is transposed
// (TMEM lanes = output columns, double-buffered 2 x 128 columns) so the
// epilogue writes bias + ReLU + bf16 rows into a staging tile (64 B per warp
// row, conflict-free) that one TMA store sends out. The partner's read of the
// same x tile hits L2: HBM sees x once and h once.
struct FwdLayerArgs {
  int64_t M;
  const float* bias;
  int32_t groups;
  CUtensorMap tx, tw, to;
};

__global__ void __launch_bounds__(kBThreads, 1) k_mlp_fwd_layer(const __grid_constant__ FwdLayerArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* Wsl = base;               // 4 boxes [128 out x 64 in] (K chunks)
  unsigned char* ostg = base + 2 * kHalf;  // output staging [128 rows x 128 columns] bf16
  unsigned char* xr = base + 3 * kHalf;    // 4 x 32 KB (two K boxes of one tile each)
  constexpr int kSlots = 4;
  uint64_t* fx = reinterpret_cast<uint64_t*>(xr + kSlots * kHalf);
  uint64_t* ex = fx + kSlots;
  uint64_t* accf = ex + kSlots;
  uint64_t* acce = accf + 2;
  uint64_t* wbar = acce + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(wbar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int member = blockIdx.x & 1, grp = blockIdx.x >> 1;
  const int c0 = 128 * member;
  const int64_t tiles = (a.M + 127) / 128;

  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < kSlots; ++i) { mbar_init(&fx[i], 1); mbar_init(&ex[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&accf[i], 1); mbar_init(&acce[i], kBEpiWarps); }
    mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {  // ------------------------------------------- TMA producer
    if (lane == 0) {
      mbar_expect_tx(wbar, 2 * kHalf);
      for (int c = 0; c < 4; ++c) tma_load_2d(Wsl + c * (kHalf / 2), &a.tw, 64 * c, c0, wbar);
      int64_t k = 0;
      for (int64_t t = grp; t < tiles; t += a.groups, ++k) {
        for (int h = 0; h < 2; ++h) {
          const int64_t q = 2 * k + h;
          const int st = (int)(q % kSlots);
          mbar_wait(&ex[st], ((uint32_t)(q / kSlots) & 1u) ^ 1u);
          mbar_expect_tx(&fx[st], kHalf);
          tma_load_2d(xr + st * kHalf, &a.tx, 128 * h, (int)(t * 128), &fx[st]);
          tma_load_2d(xr + st * kHalf + kHalf / 2, &a.tx, 128 * h + 64, (int)(t * 128), &fx[st]);
        }
      }
    }
  } else if (warp == 1) {  // -------------------------------------- MMA issuer
    const uint32_t id = instr_desc(128, false, false);
    mbar_wait(wbar, 0);
    tc_fence_after();
    const uint32_t wb = smem_u32(Wsl);
    int64_t k = 0;
    for (int64_t t = grp; t < tiles; t += a.groups, ++k) {
      const int b = (int)(k & 1);
      mbar_wait(&acce[b], ((uint32_t)(k >> 1) & 1u) ^ 1u);
      tc_fence_after();
      for (int h = 0; h < 2; ++h) {
        const int64_t q = 2 * k + h;
        const int st = (int)(q % kSlots);
        mbar_wait(&fx[st], (uint32_t)(q / kSlots) & 1u);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t xb = smem_u32(xr + st * kHalf);
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            const int ks = 8 * h + s;  // K16 step over the input features
            mma_bf16(tmem + 128u * b,
                     smem_desc_sw128(wb + (ks >> 2) * (kHalf / 2) + 32 * (ks & 3), 16, 1024),
                     smem_desc_sw128(xb + (s >> 2) * (kHalf / 2) + 32 * (s & 3), 16, 1024), id,
                     ks > 0 ? 1u : 0u);
          }
          mma_commit(&ex[st]);
          if (h == 1) mma_commit(&accf[b]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {  // -------------------------------------- epilogue
    const int e = warp - 4, q = e & 3, half = e >> 2;
    const int cl = 32 * q + lane;  // TMEM lane = output column c0 + cl
    const float bias = a.bias[c0 + cl];
    const bool issuer = e == 0 && lane == 0;
    int64_t k = 0;
    for (int64_t t = grp; t < tiles; t += a.groups, ++k) {
      const int b = (int)(k & 1);
      mbar_wait(&accf[b], (uint32_t)(k >> 1) & 1u);
      tc_fence_after();
      float v[64];
      {
        float v0[32], v1[32];
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + 128u * b + 64u * half;
        tmem_ld32(ta, v0);
        tmem_ld32(ta + 32u, v1);
#pragma unroll
        for (int i = 0; i < 32; ++i) { v[i] = v0[i]; v[32 + i] = v1[i]; }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[b]);
      // stage the tile row-major (lanes = 32 consecutive columns: 64 B per row,
      // conflict-free), then one TMA store (rows >= M are clipped)
      if (issuer) bulk_wait_read();  // the previous tile's store has read the staging
      named_sync(1, 32 * kBEpiWarps);
      __nv_bfloat16* sg = reinterpret_cast<__nv_bfloat16*>(ostg) + (64 * half) * 128 + cl;
#pragma unroll
      for (int j = 0; j < 64; ++j) sg[j * 128] = __float2bfloat16_rn(fmaxf(v[j] + bias, 0.f));
      fence_proxy_async();
      named_sync(1, 32 * kBEpiWarps);
      if (issuer) {
        tma_store_2d(&a.to, c0, (int)(t * 128), ostg);
        bulk_commit();
      }
    }
    if (issuer) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

// ---------------------------------------------------------------------------
// Head backward into the last hidden layer (width 256): dz = (dout Wh) * (h > 0)
// with K = 16 (13 real outputs), i.e. a 300 MB stream with a thin contraction.
// CTA pairs split the 256 columns; per 128-row tile one tcgen05.mma computes the
// transposed product D[c, r] = sum_k Wh[k, c] dout[r, k] (A = the Wh slice,
// MN-major SW128; B = the dout tile, K-major without swizzle: two 8-column TMA
// boxes = the two K core matrices), the mask tile arrives by TMA, and the
// epilogue (lanes = columns) masks, sums columns and stages rows for one TMA
// store, as in the layer kernels.
struct HeadBwdArgs {  // (mask ring of 4 x 32 KB: tiles carry no MMA work to hide loads behind)
  int64_t M;
  float* bpart;
  int32_t groups;
  CUtensorMap tdo, twh, th, tdz;
};

__global__ void __launch_bounds__(kBThreads, 1) k_mlp_head_bwd(const __grid_constant__ HeadBwdArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int kB = 4;                     // dout ring slots (4 KB each)
  constexpr int kH = 4;                     // mask ring slots (32 KB each)
  unsigned char* hr = base;                 // mask ring: kH x 32 KB (SW128 boxes [128 x 64])
  unsigned char* ostg = base + kH * kHalf;  // staging [128 rows x 128 columns] bf16
  unsigned char* wa = ostg + kHalf;         // Wh slice: 2 boxes [16 k x 64 c] (2 KB each)
  unsigned char* br = wa + 4096;            // dout ring: kB x (2 boxes [128 rows x 8 k])
  uint64_t* fb = reinterpret_cast<uint64_t*>(br + kB * 4096);
  uint64_t* eb = fb + kB;
  uint64_t* fh = eb + kB;
  uint64_t* eh = fh + kH;
  uint64_t* accf = eh + kH;
  uint64_t* acce = accf + 2;
  uint64_t* wbar = acce + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(wbar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int member = blockIdx.x & 1, grp = blockIdx.x >> 1;
  const int c0 = 128 * member;
  const int64_t tiles = (a.M + 127) / 128;

  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < kB; ++i) { mbar_init(&fb[i], 1); mbar_init(&eb[i], 1); }
    for (int i = 0; i < kH; ++i) { mbar_init(&fh[i], 1); mbar_init(&eh[i], kBEpiWarps); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&accf[i], 1);
      mbar_init(&acce[i], kBEpiWarps);
    }
    mbar_init(wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {  // ------------------------------------------- TMA producer
    if (lane == 0) {
      mbar_expect_tx(wbar, 4096);
      tma_load_2d(wa, &a.twh, c0, 0, wbar);
      tma_load_2d(wa + 2048, &a.twh, c0 + 64, 0, wbar);
      int64_t k = 0;
      for (int64_t t = grp; t < tiles; t += a.groups, ++k) {
        const int m0 = (int)(t * 128);
        const int st = (int)(k % kB), sa = (int)(k % kH);
        mbar_wait(&eb[st], ((uint32_t)(k / kB) & 1u) ^ 1u);
        mbar_expect_tx(&fb[st], 4096);
        tma_load_2d(br + st * 4096, &a.tdo, 0, m0, &fb[st]);
        tma_load_2d(br + st * 4096 + 2048, &a.tdo, 8, m0, &fb[st]);
        mbar_wait(&eh[sa], ((uint32_t)(k / kH) & 1u) ^ 1u);
        mbar_expect_tx(&fh[sa], kHalf);
        tma_load_2d(hr + sa * kHalf, &a.th, c0, m0, &fh[sa]);
        tma_load_2d(hr + sa * kHalf + kHalf / 2, &a.th, c0 + 64, m0, &fh[sa]);
      }
    }
  } else if (warp == 1) {  // -------------------------------------- MMA issuer
    const uint32_t id = instr_desc(128, true, false);
    mbar_wait(wbar, 0);
    tc_fence_after();
    int64_t k = 0;
    for (int64_t t = grp; t < tiles; t += a.groups, ++k) {
      const int b = (int)(k & 1), st = (int)(k % kB);
      mbar_wait(&acce[b], ((uint32_t)(k >> 1) & 1u) ^ 1u);
      mbar_wait(&fb[st], (uint32_t)(k / kB) & 1u);
      tc_fence_after();
      if (lane == 0) {
        // A: Wh^T (M = columns, two 64-wide SW128 atoms 2 KB apart, K rows 1 KB per 8);
        // B: dout (N = rows; no swizzle: core matrices of 8 rows x 16 B, 128 B apart
        // along N, the second K half 2 KB further)
        mma_bf16(tmem + 128u * b, smem_desc_sw128(smem_u32(wa), 2048, 1024),
                 smem_desc(smem_u32(br + st * 4096), 2048, 128), id, 0u);
        mma_commit(&eb[st]);
        mma_commit(&accf[b]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {  // -------------------------------------- epilogue
    const int e = warp - 4, q = e & 3, half = e >> 2;
    const int ci = 32 * q + lane;  // TMEM lane = column c0 + ci
    const bool issuer = e == 0 && lane == 0;
    const uint32_t mcol = (ci >> 6) * (kHalf / 2) + (((ci & 63) >> 3) << 4) + (ci & 7) * 2;
    float cs = 0.f;
    int64_t k = 0;
    for (int64_t t = grp; t < tiles; t += a.groups, ++k) {
      const int b = (int)(k & 1), sa = (int)(k % kH);
      mbar_wait(&accf[b], (uint32_t)(k >> 1) & 1u);
      mbar_wait(&fh[sa], (uint32_t)(k / kH) & 1u);
      tc_fence_after();
      float v[64];
      {
        float v0[32], v1[32];
        const uint32_t ta = tmem + ((uint32_t)(32 * q) << 16) + 128u * b + 64u * half;
        tmem_ld32(ta, v0);
        tmem_ld32(ta + 32u, v1);
#pragma unroll
        for (int i = 0; i < 32; ++i) { v[i] = v0[i]; v[32 + i] = v1[i]; }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acce[b]);
      if (issuer) bulk_wait_read();  // the previous tile's store has read the staging
      named_sync(1, 32 * kBEpiWarps);
      const unsigned char* slot = hr + sa * kHalf;
      __nv_bfloat16* sg = reinterpret_cast<__nv_bfloat16*>(ostg) + (64 * half) * 128 + ci;
#pragma unroll
      for (int j = 0; j < 64; ++j) {
        const int ro = 64 * half + j;
        const __nv_bfloat16 mv =
            *reinterpret_cast<const __nv_bfloat16*>(slot + ro * 128 + (mcol ^ ((ro & 7) << 4)));
        const float x = __bfloat162float(mv) > 0.f ? v[j] : 0.f;
        cs += x;  // rows >= M: zero-filled mask and dout
        sg[j * 128] = __float2bfloat16_rn(x);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&eh[sa]);
      fence_proxy_async();
      named_sync(1, 32 * kBEpiWarps);
      if (issuer) {
        tma_store_2d(&a.tdz, c0, (int)(t * 128), ostg);
        bulk_commit();
      }
    }
    if (issuer) bulk_wait_all();
    a.bpart[((int64_t)grp * 2 + half) * 256 + c0 + ci] = cs;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
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

// bf16 2-D map: cols x rows (row pitch in elements), box bc x br, 128-byte swizzle
bool map2d(CUtensorMap* m, const void* p, int64_t cols, int64_t rows, int64_t pitch, int bc,
           int br) {
  auto enc = encoder();
  if (!enc || (uintptr_t)p % 16 || (pitch * 2) % 16) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, str[1] = {(cuuint64_t)pitch * 2};
  cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br}, es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, str, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// bf16 2-D map without swizzle (row-major staging tiles for TMA stores)
bool map2d_plain(CUtensorMap* m, const void* p, int64_t cols, int64_t rows, int64_t pitch, int bc,
                 int br) {
  auto enc = encoder();
  if (!enc || (uintptr_t)p % 16 || (pitch * 2) % 16) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, str[1] = {(cuuint64_t)pitch * 2};
  cuuint32_t box[2] = {(cuuint32_t)bc, (cuuint32_t)br}, es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, str, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// Host side of the fused forward; returns false when the shape is outside its
// envelope (the caller then runs the layer-by-layer path).
bool launch_mlp_fused_fwd(const MlpFusedDesc& d, cudaStream_t s, cudaError_t* err) {
  if (d.W % 64 || d.W > 256 || d.D > kFMaxD || d.F > kFMaxFrames || d.E8 > 128 || d.M == 0)
    return false;
  static thread_local FusedArgs a;
  std::memset(&a, 0, sizeof(a));
  a.W = d.W; a.D = d.D; a.skip = d.skip; a.Lx = d.Lx; a.Lt = d.Lt; a.E8 = d.E8;
  a.catw = d.catw; a.train = d.train; a.shc = d.shc; a.N = d.N; a.M = d.M;
  for (int f = 0; f < d.F; ++f) a.t[f] = d.times[f];
  a.theta = d.theta; a.thbh = d.thbh;
  for (int l = 0; l < d.D; ++l) a.thb[l] = d.thb[l];
  a.canon = d.canon; a.frame = d.frame; a.out = d.out;
  bool ok = true;
  for (int l = 0; l < d.D && ok; ++l) {
    if (l == 0) ok = map2d(&a.wl[0], d.wbf[0], d.E8, d.W, d.Kp[0], 64, d.W);
    else if (l == d.skip + 1) {
      ok = map2d(&a.wl[l], d.wbf[l], d.E8, d.W, d.Kp[l], 64, d.W) &&
           map2d(&a.wl[kFMaxD], d.wbf[l] + d.E8, d.W, d.W, d.Kp[l], 64, d.W);
    } else ok = map2d(&a.wl[l], d.wbf[l], d.W, d.W, d.Kp[l], 64, d.W);
  }
  ok = ok && map2d(&a.wh, d.whbf, d.W, 16, d.W, 64, 16);
  if (ok && d.train) {
    for (int l = 0; l < d.D && ok; ++l)
      if (l != d.skip) ok = map2d(&a.hs[l], d.h[l], d.W, d.M, d.W, 64, 128);
    ok = ok && map2d(&a.cate, d.cat, d.E8, d.M, d.catw, 64, 128) &&
         (d.skip < 0 || map2d(&a.cath, d.cat + d.E8, d.W, d.M, d.catw, 64, 128));
  }
  if (!ok) return false;
  const int smem = 6 * (int)kXChunk + kFStages * 256 * 64 * 2 + 1024 + 1024;
  WIPES_SET_SMEM_ONCE(k_mlp_fused_fwd, smem);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (d.M + 127) / 128;
  launch_begin(K_GEMM, s);
  k_mlp_fused_fwd<<<(unsigned)(tiles < sms ? tiles : sms), kFThreads, smem, s>>>(a);
  launch_end(K_GEMM, s);
  *err = cudaGetLastError();
  return true;
}

int launch_mlp_bwd_layer(const MlpBwdDesc& d, cudaStream_t s, cudaError_t* err) {
  if (d.W != 256 || d.M <= 0 || d.M > INT32_MAX - 128) return 0;
  static thread_local BwdArgs a;
  std::memset(&a, 0, sizeof(a));
  a.M = d.M; a.wpart = d.wpart; a.bpart = d.bpart; a.dzo = d.dzo;
  if (!map2d(&a.tdz, d.dz, 256, d.M, 256, 64, 128) ||
      !map2d(&a.tact, d.act, 256, d.M, d.act_ld, 64, 128) ||
      !map2d(&a.tw, d.wl, 256, 256, d.w_ld, 64, 256) || (uintptr_t)d.dzo % 16)
    return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (d.M + 127) / 128;
  int64_t groups = sms / 2;
  if (groups > d.max_groups) groups = d.max_groups;
  if (groups > tiles) groups = tiles;
  if (groups < 1) return 0;
  a.groups = (int32_t)groups;
  const int smem = 7 * (int)kHalf + 1024 + 256;
  WIPES_SET_SMEM_ONCE(k_mlp_bwd_layer, smem);
  launch_begin(K_GEMM, s);
  k_mlp_bwd_layer<<<(unsigned)(2 * groups), kBThreads, smem, s>>>(a);
  launch_end(K_GEMM, s);
  *err = cudaGetLastError();
  return (int)groups;
}

bool launch_mlp_fwd_layer(const MlpFwdLayerDesc& d, cudaStream_t s, cudaError_t* err) {
  if (d.W != 256 || d.M <= 0 || d.M > INT32_MAX - 128) return false;
  static thread_local FwdLayerArgs a;
  std::memset(&a, 0, sizeof(a));
  a.M = d.M; a.bias = d.bias;
  if (!map2d(&a.tx, d.x, 256, d.M, d.x_ld, 64, 128) || !map2d(&a.tw, d.w, 256, 256, 256, 64, 128) ||
      !map2d_plain(&a.to, d.out, 256, d.M, d.out_ld, 128, 128))
    return false;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (d.M + 127) / 128;
  int64_t groups = sms / 2;
  if (groups > tiles) groups = tiles;
  a.groups = (int32_t)groups;
  const int smem = 7 * (int)kHalf + 1024 + 256;
  WIPES_SET_SMEM_ONCE(k_mlp_fwd_layer, smem);
  launch_begin(K_GEMM, s);
  k_mlp_fwd_layer<<<(unsigned)(2 * groups), kBThreads, smem, s>>>(a);
  launch_end(K_GEMM, s);
  *err = cudaGetLastError();
  return true;
}

int launch_mlp_head_bwd(const MlpHeadBwdDesc& d, cudaStream_t s, cudaError_t* err) {
  if (d.W != 256 || d.M <= 0 || d.M > INT32_MAX - 128) return 0;
  static thread_local HeadBwdArgs a;
  std::memset(&a, 0, sizeof(a));
  a.M = d.M; a.bpart = d.bpart;
  if (!map2d_plain(&a.tdo, d.dout, 16, d.M, 16, 8, 128) ||
      !map2d(&a.twh, d.wh, 256, 16, 256, 64, 16) || !map2d(&a.th, d.h, 256, d.M, d.h_ld, 64, 128) ||
      !map2d_plain(&a.tdz, d.dz, 256, d.M, 256, 128, 128))
    return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (d.M + 127) / 128;
  int64_t groups = sms / 2;
  if (groups > d.max_groups) groups = d.max_groups;
  if (groups > tiles) groups = tiles;
  a.groups = (int32_t)groups;
  const int smem = 5 * (int)kHalf + 4096 + 4 * 4096 + 1024 + 256;
  WIPES_SET_SMEM_ONCE(k_mlp_head_bwd, smem);
  launch_begin(K_GEMM, s);
  k_mlp_head_bwd<<<(unsigned)(2 * groups), kBThreads, smem, s>>>(a);
  launch_end(K_GEMM, s);
  *err = cudaGetLastError();
  return (int)groups;
}

}  // namespace wipes
