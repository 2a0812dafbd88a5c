// Per-tile render kernels, FP32 + SFU (MUFU) pipes.
//
//  forward  : PAPER.md:172 (Eq. 4, weighted sum) / PAPER.md:125 (Eq. 3, alpha
//             blending), with the Gaussian G' replaced by the wavelet W'
//             (PAPER.md:215, :272): w = alpha * G * 1/2 [1 + beta cos(f.d + phi)].
//  backward : analytic per-pair gradients ("explicit gradients for all
//             parameters") accumulated as 12 per-record MOMENTS
//              that the FP64 preprocess-backward turns into the
//             record gradients exactly (they are linear in the moments with
//             per-record coefficients). Moments are reduced per warp with a
//             12-slot transpose-reduce of shuffles, then one atomic per (warp,
//             record, moment).
//
// Persistent CTAs (grid = SMs x resident CTAs) pull (view, tile) work items
// from a queue ordered longest-list-first (bin_sort's tile order), so the
// uneven per-tile cost does not leave SMs idle at the end of the launch.
// Each warp owns an 8x8-pixel sub-tile, each lane two pixels (rows y and
// y+4; the second is evaluated incrementally from the first). Records are
// staged in shared memory in batches (structure-of-float4 layout); every staged
// record carries a sub-tile mask from its conservative opacity extent, and each
// warp compacts the batch into its own ordered list of records that can reach
// its pixels (ballot + popc). Branches inside a (warp, record) step are
// warp-uniform (ballots); per-lane decisions are predicated selects. exp is one
// MUFU.EX2 (the -1/2 log2(e) scale and log2(alpha) folded into the record);
// cos / sin are MUFU.COS / MUFU.SIN.
#include <cuda_fp16.h>

#include <mutex>

#include "common.cuh"

namespace wipes {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMom = kMoments;  // 12
enum { Q_FWD = 0, Q_BWD = 1, Q_STATS = 2 };

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float cos_a(float x) {
  float y;
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sin_a(float x) {
  float y;
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_a(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

struct RenderArgs {
  const float4* rec;     // [B*N][4]
  const uint32_t* vals;  // sorted primitive indices
  const int32_t* toff;   // [B*T + 1]
  const int32_t* order;  // [B*T] longest-first tile order
  WsHeader* hdr;         // work queues
  int64_t N, T, BT;
  int32_t W, H, GX, queue;
  float alpha_min, skip_e, alpha_max, T_min;
  float bg0, bg1, bg2;
  float* image;          // [B,3,H,W]
  float* T_final;        // [B,H,W]
  int32_t* n_contrib;    // [B,H,W]
  const float* dLdC;     // [B,3,H,W]
  const float* T_in;
  const int32_t* nc_in;
  float* mom;            // [B*N, 12] gradient moments
  unsigned long long* stats;  // STATS build: {tile-method candidates, in-ellipse, contributing}
};

// Sub-tile mask of a record for tile origin (X0, Y0): bit (sy * NS + sx) set
// when the record's opacity-extent AABB (padded) may touch 8x8 sub-tile (sx, sy).
template <int TS>
__device__ __forceinline__ uint32_t subtile_mask(const float4& r0, const float4& r3, int X0,
                                                 int Y0) {
  constexpr int NS = TS / 8;
  __half2 e2 = *reinterpret_cast<const __half2*>(&r3.w);
  float rx = __low2float(e2) + 0.02f, ry = __high2float(e2) + 0.02f;
  float cx = (r0.x - (float)X0) + r0.z;  // centre relative to the tile origin
  float cy = (r0.y - (float)Y0) + r0.w;
  // sub-tile s covers pixel centres [8 s + 0.5, 8 s + 7.5]
  float fx0 = ceilf((cx - rx - 7.5f) * 0.125f), fx1 = floorf((cx + rx - 0.5f) * 0.125f);
  float fy0 = ceilf((cy - ry - 7.5f) * 0.125f), fy1 = floorf((cy + ry - 0.5f) * 0.125f);
  fx0 = fmaxf(fx0, 0.f); fy0 = fmaxf(fy0, 0.f);
  fx1 = fminf(fx1, (float)(NS - 1)); fy1 = fminf(fy1, (float)(NS - 1));
  if (!(fx0 <= fx1) || !(fy0 <= fy1)) return 0u;
  int sx0 = (int)fx0, sx1 = (int)fx1, sy0 = (int)fy0, sy1 = (int)fy1;
  uint32_t row = ((2u << sx1) - 1u) & ~((1u << sx0) - 1u);
  uint32_t m = 0;
#pragma unroll
  for (int sy = 0; sy < NS; ++sy)
    if (sy >= sy0 && sy <= sy1) m |= row << (sy * NS);
  return m;
}

// Exponents of alpha*G for the lane's two pixels (rows y0 and y0 + 4) — one
// arithmetic shared by every kernel, so all take the same alpha_min decisions
// (and, since 8x8 sub-tiles are 8-aligned for every tile size, every pixel is
// evaluated by the same expression whatever the tiling).
struct PairPos {
  float dx, dy0, e0, e1;
};

__device__ __forceinline__ PairPos pair_exponents(const float4& r0, const float4& r1, float px,
                                                  float py0) {
  PairPos p;
  p.dx = __fsub_rn(__fsub_rn(px, r0.x), r0.z);
  p.dy0 = __fsub_rn(__fsub_rn(py0, r0.y), r0.w);
  const float t = __fmaf_rn(r1.x, p.dx, __fmul_rn(r1.y, p.dy0));  // A dx + B dy
  const float cdy = __fmul_rn(r1.z, p.dy0);                        // C dy
  p.e0 = __fmaf_rn(t, p.dx, __fmaf_rn(cdy, p.dy0, r1.w));
  // dy1 = dy0 + 4: e1 = e0 + 4 (B dx + 2 C dy0 + 4 C)
  const float v = __fmaf_rn(r1.y, p.dx, __fmaf_rn(2.f, cdy, __fmul_rn(4.f, r1.z)));
  p.e1 = __fmaf_rn(4.f, v, p.e0);
  return p;
}

__device__ __forceinline__ float pair_theta(const float4& r2, float dx, float dy) {
  return __fmaf_rn(r2.x, dx, __fmaf_rn(r2.y, dy, r2.z));
}

__device__ __forceinline__ float pair_weight(float ag, float cs, const float4& r2) {
  return __fmul_rn(ag, __fmaf_rn(r2.w, cs, 0.5f));
}

template <int TS>
struct Geo {
  static constexpr int NS = TS / 8;               // sub-tiles per side
  static constexpr int NW = NS * NS;              // warps per CTA
  static constexpr int NT = 32 * NW;              // threads per CTA
  static constexpr int NB = NT < 128 ? 128 : NT;  // records per staged batch
};

template <int TS>
struct Smem {
  float4 rec[4][Geo<TS>::NB];
  uint32_t mask[Geo<TS>::NB];
  uint8_t list[Geo<TS>::NW][Geo<TS>::NB];
  int32_t pid[Geo<TS>::NB];
  int32_t item, maxlast;
};

// Stage records [b0, b0 + nb) of the tile list into shared memory and build
// each warp's compacted list. Returns this warp's list length.
template <int TS>
__device__ __forceinline__ int stage_batch(const RenderArgs& a, const float4* recv, int b0,
                                           int nb, int X0, int Y0, Smem<TS>& sm, int tid,
                                           int lane, int wid) {
  constexpr int NB = Geo<TS>::NB, NT = Geo<TS>::NT;
#pragma unroll
  for (int t = tid; t < NB; t += NT) {
    uint32_t m = 0;
    if (t < nb) {
      const uint32_t pid = a.vals[b0 + t];
      const float4* r = recv + 4 * (int64_t)pid;
      float4 r0 = __ldg(r), r1 = __ldg(r + 1), r2 = __ldg(r + 2), r3 = __ldg(r + 3);
      sm.rec[0][t] = r0; sm.rec[1][t] = r1; sm.rec[2][t] = r2; sm.rec[3][t] = r3;
      sm.pid[t] = (int32_t)pid;
      m = subtile_mask<TS>(r0, r3, X0, Y0);
    }
    sm.mask[t] = m;
  }
  __syncthreads();
  int cnt = 0;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int c = 0; c < NB / 32; ++c) {
    const int j = c * 32 + lane;
    const bool hit = (sm.mask[j] >> wid) & 1u;
    const uint32_t bal = __ballot_sync(kFull, hit);
    if (hit) sm.list[wid][cnt + __popc(bal & lt)] = (uint8_t)j;
    cnt += __popc(bal);
  }
  __syncwarp();
  return cnt;
}

// Persistent work loop helpers: fetch the next (view, tile) item; the last CTA
// to leave resets the queue for the next launch.
template <int TS>
__device__ __forceinline__ int64_t next_item(const RenderArgs& a, Smem<TS>& sm, int tid) {
  __syncthreads();
  if (tid == 0) sm.item = atomicAdd(&a.hdr->work[a.queue], 1);
  __syncthreads();
  const int item = sm.item;
  return item < a.BT ? (int64_t)a.order[item] : -1;
}

__device__ __forceinline__ void leave_queue(const RenderArgs& a, int tid) {
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&a.hdr->done[a.queue], 1) == (int)gridDim.x - 1) {
      a.hdr->work[a.queue] = 0;
      a.hdr->done[a.queue] = 0;
      __threadfence();
    }
  }
}

// Front-to-back alpha compositing step of one pixel (Eq. 3, R9/R10),
// predicated: ok = the pair contributes alpha*W >= alpha_min.
__device__ __forceinline__ void alpha_step(bool ok, float w, const float4& r3, int pos,
                                           float amax, float tmin, float& T, float& C0,
                                           float& C1, float& C2, int& last, bool& done,
                                           int& stop) {
  const float al = fminf(amax, w);
  const float Tn = __fmul_rn(T, __fsub_rn(1.f, al));
  const bool stp = ok && Tn < tmin;
  const bool comp = ok && !stp;
  const float aT = comp ? __fmul_rn(al, T) : 0.f;
  C0 = __fmaf_rn(r3.x, aT, C0);
  C1 = __fmaf_rn(r3.y, aT, C1);
  C2 = __fmaf_rn(r3.z, aT, C2);
  T = comp ? Tn : T;
  last = comp ? pos : last;
  done = done || stp;
  stop = stp ? pos : stop;
}

template <int TS, bool ALPHA, bool STATS>
__global__ void __launch_bounds__(Geo<TS>::NT) k_render_fwd(RenderArgs a) {
  using G = Geo<TS>;
  constexpr int NB = G::NB;
  __shared__ Smem<TS> sm;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ox = (wid % G::NS) * 8 + (lane & 7), oy = (wid / G::NS) * 8 + (lane >> 3);
  unsigned long long st_cand = 0, st_ell = 0, st_con = 0;  // STATS only
  for (;;) {
    const int64_t tile = next_item<TS>(a, sm, tid);
    if (tile < 0) break;
    const int64_t v = tile / a.T;
    const int64_t t_in_v = tile - v * a.T;
    const int ty = (int)(t_in_v / a.GX), tx = (int)(t_in_v - (int64_t)ty * a.GX);
    const int X0 = tx * TS, Y0 = ty * TS;
    const int x = X0 + ox, y0 = Y0 + oy, y1 = y0 + 4;
    const bool in0 = x < a.W && y0 < a.H, in1 = x < a.W && y1 < a.H;
    const float px = (float)x + 0.5f, py0 = (float)y0 + 0.5f;
    const int start = a.toff[tile], end = a.toff[tile + 1];
    const float4* recv = a.rec + 4 * (v * a.N);
    float C00 = 0.f, C01 = 0.f, C02 = 0.f, C10 = 0.f, C11 = 0.f, C12 = 0.f;
    float T0 = 1.f, T1 = 1.f;
    int last0 = 0, last1 = 0, stop0 = end - start, stop1 = end - start;
    bool done0 = ALPHA ? !in0 : false, done1 = ALPHA ? !in1 : false;
    for (int b0 = start; b0 < end; b0 += NB) {
      const int nb = min(NB, end - b0);
      __syncthreads();
      const int cnt = stage_batch<TS>(a, recv, b0, nb, X0, Y0, sm, tid, lane, wid);
      if (!ALPHA || !__all_sync(kFull, done0 && done1)) {
        for (int i = 0; i < cnt; ++i) {
          const int j = sm.list[wid][i];
          const float4 r0 = sm.rec[0][j], r1 = sm.rec[1][j];
          const PairPos pp = pair_exponents(r0, r1, px, py0);
          const bool h0 = pp.e0 >= a.skip_e && !done0, h1 = pp.e1 >= a.skip_e && !done1;
          if (STATS) st_ell += (h0 && in0) + (h1 && in1);
          const uint32_t b0m = __ballot_sync(kFull, h0), b1m = __ballot_sync(kFull, h1);
          if (!(b0m | b1m)) continue;
          const float4 r2 = sm.rec[2][j], r3 = sm.rec[3][j];
          const int pos = b0 + j - start + 1;
          if (b0m) {
            const float w = pair_weight(ex2(pp.e0), cos_a(pair_theta(r2, pp.dx, pp.dy0)), r2);
            const bool ok = h0 && w >= a.alpha_min;
            if (!ALPHA) {
              const float we = ok ? w : 0.f;
              if (STATS) st_con += ok && in0;
              C00 = __fmaf_rn(r3.x, we, C00);
              C01 = __fmaf_rn(r3.y, we, C01);
              C02 = __fmaf_rn(r3.z, we, C02);
            } else {
              if (STATS) st_con += ok;
              alpha_step(ok, w, r3, pos, a.alpha_max, a.T_min, T0, C00, C01, C02, last0,
                         done0, stop0);
              if (STATS) st_con -= ok && done0 && stop0 == pos;
            }
          }
          if (b1m) {
            const float dy1 = __fadd_rn(pp.dy0, 4.f);
            const float w = pair_weight(ex2(pp.e1), cos_a(pair_theta(r2, pp.dx, dy1)), r2);
            const bool ok = h1 && w >= a.alpha_min;
            if (!ALPHA) {
              const float we = ok ? w : 0.f;
              if (STATS) st_con += ok && in1;
              C10 = __fmaf_rn(r3.x, we, C10);
              C11 = __fmaf_rn(r3.y, we, C11);
              C12 = __fmaf_rn(r3.z, we, C12);
            } else {
              if (STATS) st_con += ok;
              alpha_step(ok, w, r3, pos, a.alpha_max, a.T_min, T1, C10, C11, C12, last1,
                         done1, stop1);
              if (STATS) st_con -= ok && done1 && stop1 == pos;
            }
          }
          if (ALPHA && __all_sync(kFull, done0 && done1)) break;
        }
      }
      if (ALPHA) {
        if (__syncthreads_count(!(done0 && done1)) == 0) break;
      }
    }
    if (STATS) {
      st_cand += (in0 ? (unsigned long long)stop0 : 0ull) + (in1 ? (unsigned long long)stop1 : 0ull);
      continue;
    }
    const int64_t HW = (int64_t)a.H * a.W;
    float* img = a.image + v * 3 * HW;
    if (in0) {
      const int64_t p = (int64_t)y0 * a.W + x;
      if (ALPHA) {
        C00 = __fmaf_rn(T0, a.bg0, C00);
        C01 = __fmaf_rn(T0, a.bg1, C01);
        C02 = __fmaf_rn(T0, a.bg2, C02);
        a.T_final[v * HW + p] = T0;
        a.n_contrib[v * HW + p] = last0;
      }
      img[p] = C00; img[HW + p] = C01; img[2 * HW + p] = C02;
    }
    if (in1) {
      const int64_t p = (int64_t)y1 * a.W + x;
      if (ALPHA) {
        C10 = __fmaf_rn(T1, a.bg0, C10);
        C11 = __fmaf_rn(T1, a.bg1, C11);
        C12 = __fmaf_rn(T1, a.bg2, C12);
        a.T_final[v * HW + p] = T1;
        a.n_contrib[v * HW + p] = last1;
      }
      img[p] = C10; img[HW + p] = C11; img[2 * HW + p] = C12;
    }
  }
  if (STATS) {
    unsigned long long c3[3] = {st_cand, st_ell, st_con};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      unsigned long long s = c3[k];
#pragma unroll
      for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
      if (lane == 0 && s) atomicAdd(a.stats + k, s);
    }
  }
  leave_queue(a, tid);
}

// 12-slot warp transpose-reduce. On return lane L holds the warp-wide sum of
// moment index 6*b4 + 3*b3 + q (b_k = bit k of L, q = (L >> 1) & 3) when q < 3.
__device__ __forceinline__ float transpose_reduce12(float (&v)[kMom], int lane) {
  {
    const bool up = lane & 16;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      float send = up ? v[k] : v[k + 6];
      float keep = up ? v[k + 6] : v[k];
      v[k] = keep + __shfl_xor_sync(kFull, send, 16);
    }
  }
  {
    const bool up = lane & 8;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      float send = up ? v[k] : v[k + 3];
      float keep = up ? v[k + 3] : v[k];
      v[k] = keep + __shfl_xor_sync(kFull, send, 8);
    }
  }
  {
    const bool up = lane & 4;  // pairs (0, 2) and (1, pad)
    float s0 = up ? v[0] : v[2], k0 = up ? v[2] : v[0];
    float s1 = up ? v[1] : 0.f, k1 = up ? 0.f : v[1];
    v[0] = k0 + __shfl_xor_sync(kFull, s0, 4);
    v[1] = k1 + __shfl_xor_sync(kFull, s1, 4);
  }
  {
    const bool up = lane & 2;
    float s = up ? v[0] : v[1], k = up ? v[1] : v[0];
    v[0] = k + __shfl_xor_sync(kFull, s, 2);
  }
  return v[0] + __shfl_xor_sync(kFull, v[0], 1);
}

// Moments of one pair, gw = dL/dw and w already zeroed when the
// pair does not contribute: M0 = gw w, M1 = gw w dx, M2 = gw w dy,
// M3 = gw w dx^2, M4 = gw w dx dy, M5 = gw w dy^2, M6 = gw ag sin, M7 = M6 dx,
// M8 = M6 dy, M9..11 = dL/dc terms.
__device__ __forceinline__ void add_moments(float (&m)[kMom], float gw, float w, float ag,
                                            float sn, float dx, float dy, float c0, float c1,
                                            float c2) {
  const float gww = gw * w;
  const float m1 = gww * dx, m2 = gww * dy;
  const float m6 = gw * ag * sn;
  m[0] += gww;
  m[1] += m1;
  m[2] += m2;
  m[3] = __fmaf_rn(m1, dx, m[3]);
  m[4] = __fmaf_rn(m1, dy, m[4]);
  m[5] = __fmaf_rn(m2, dy, m[5]);
  m[6] += m6;
  m[7] = __fmaf_rn(m6, dx, m[7]);
  m[8] = __fmaf_rn(m6, dy, m[8]);
  m[9] += c0;
  m[10] += c1;
  m[11] += c2;
}

// Backward of one pixel for one record (predicated on `h`).
template <bool ALPHA>
__device__ __forceinline__ void bwd_pixel(bool h, float e, float dx, float dy, const float4& r2,
                                          const float4& r3, float g0, float g1, float g2,
                                          float amin, float amax, float& T, float& S0,
                                          float& S1, float& S2, float (&m)[kMom], bool& any) {
  const float ag = ex2(e);
  const float th = pair_theta(r2, dx, dy);
  const float cs = cos_a(th), sn = sin_a(th);
  const float w = pair_weight(ag, cs, r2);
  const bool ok = h && w >= amin;
  any = any || ok;
  const float gdc = __fmaf_rn(r3.x, g0, __fmaf_rn(r3.y, g1, __fmul_rn(r3.z, g2)));
  if (!ALPHA) {
    const float we = ok ? w : 0.f;
    add_moments(m, ok ? gdc : 0.f, we, ag, sn, dx, dy, we * g0, we * g1, we * g2);
  } else {
    const float al = fminf(amax, w);
    const float ri = rcp_a(1.f - al);
    const float Tk = T * ri;
    const float sdg = __fmaf_rn(S0, g0, __fmaf_rn(S1, g1, __fmul_rn(S2, g2)));
    const float dLda = __fmaf_rn(Tk, gdc, -sdg * ri);
    const float aT = ok ? al * Tk : 0.f;
    S0 = __fmaf_rn(r3.x, aT, S0);
    S1 = __fmaf_rn(r3.y, aT, S1);
    S2 = __fmaf_rn(r3.z, aT, S2);
    T = ok ? Tk : T;
    add_moments(m, (ok && w < amax) ? dLda : 0.f, ok ? w : 0.f, ag, sn, dx, dy, aT * g0,
                aT * g1, aT * g2);
  }
}

template <int TS, bool ALPHA>
__global__ void __launch_bounds__(Geo<TS>::NT) k_render_bwd(RenderArgs a) {
  using G = Geo<TS>;
  constexpr int NB = G::NB;
  __shared__ Smem<TS> sm;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ox = (wid % G::NS) * 8 + (lane & 7), oy = (wid / G::NS) * 8 + (lane >> 3);
  const int q3 = (lane >> 1) & 3;
  const int my_m = 6 * ((lane >> 4) & 1) + 3 * ((lane >> 3) & 1) + q3;
  const bool writer = !(lane & 1) && q3 < 3;
  for (;;) {
    const int64_t tile = next_item<TS>(a, sm, tid);
    if (tile < 0) break;
    const int64_t v = tile / a.T;
    const int64_t t_in_v = tile - v * a.T;
    const int ty = (int)(t_in_v / a.GX), tx = (int)(t_in_v - (int64_t)ty * a.GX);
    const int X0 = tx * TS, Y0 = ty * TS;
    const int x = X0 + ox, y0 = Y0 + oy, y1 = y0 + 4;
    const bool in0 = x < a.W && y0 < a.H, in1 = x < a.W && y1 < a.H;
    const float px = (float)x + 0.5f, py0 = (float)y0 + 0.5f;
    const int start = a.toff[tile];
    int end = a.toff[tile + 1];
    const int64_t HW = (int64_t)a.H * a.W;
    const int64_t p0 = v * HW + (int64_t)y0 * a.W + x, p1 = v * HW + (int64_t)y1 * a.W + x;
    float g00 = 0.f, g01 = 0.f, g02 = 0.f, g10 = 0.f, g11 = 0.f, g12 = 0.f;
    float T0 = 1.f, T1 = 1.f, S00 = 0.f, S01 = 0.f, S02 = 0.f, S10 = 0.f, S11 = 0.f, S12 = 0.f;
    int last0 = 0, last1 = 0;
    const float* gp = a.dLdC + v * 3 * HW;
    if (in0) {
      const int64_t q = (int64_t)y0 * a.W + x;
      g00 = gp[q]; g01 = gp[HW + q]; g02 = gp[2 * HW + q];
      if (ALPHA) {
        T0 = a.T_in[p0]; last0 = a.nc_in[p0];
        S00 = T0 * a.bg0; S01 = T0 * a.bg1; S02 = T0 * a.bg2;
      }
    }
    if (in1) {
      const int64_t q = (int64_t)y1 * a.W + x;
      g10 = gp[q]; g11 = gp[HW + q]; g12 = gp[2 * HW + q];
      if (ALPHA) {
        T1 = a.T_in[p1]; last1 = a.nc_in[p1];
        S10 = T1 * a.bg0; S11 = T1 * a.bg1; S12 = T1 * a.bg2;
      }
    }
    if (ALPHA) {
      if (tid == 0) sm.maxlast = 0;
      __syncthreads();
      const int ml = max(last0, last1);
      if (ml > 0) atomicMax(&sm.maxlast, ml);
      __syncthreads();
      end = start + sm.maxlast;
    }
    const float4* recv = a.rec + 4 * (v * a.N);
    const int64_t vN = v * a.N;
    const int nbatch = (end - start + NB - 1) / NB;
    for (int bi = 0; bi < nbatch; ++bi) {
      // ALPHA walks batches back to front; SUM front to back (order-free).
      const int b0 = ALPHA ? max(start, end - (bi + 1) * NB) : start + bi * NB;
      const int nb = ALPHA ? (end - bi * NB) - b0 : min(NB, end - b0);
      __syncthreads();
      const int cnt = stage_batch<TS>(a, recv, b0, nb, X0, Y0, sm, tid, lane, wid);
      for (int ii = 0; ii < cnt; ++ii) {
        const int j = sm.list[wid][ALPHA ? cnt - 1 - ii : ii];
        const int pos = b0 + j - start;  // index within the tile list
        const float4 r0 = sm.rec[0][j], r1 = sm.rec[1][j];
        const PairPos pp = pair_exponents(r0, r1, px, py0);
        const bool h0 = in0 && pp.e0 >= a.skip_e && (!ALPHA || pos < last0);
        const bool h1 = in1 && pp.e1 >= a.skip_e && (!ALPHA || pos < last1);
        const uint32_t b0m = __ballot_sync(kFull, h0), b1m = __ballot_sync(kFull, h1);
        if (!(b0m | b1m)) continue;
        const float4 r2 = sm.rec[2][j], r3 = sm.rec[3][j];
        float m[kMom];
#pragma unroll
        for (int k = 0; k < kMom; ++k) m[k] = 0.f;
        bool any = false;
        if (b0m)
          bwd_pixel<ALPHA>(h0, pp.e0, pp.dx, pp.dy0, r2, r3, g00, g01, g02, a.alpha_min,
                           a.alpha_max, T0, S00, S01, S02, m, any);
        if (b1m)
          bwd_pixel<ALPHA>(h1, pp.e1, pp.dx, __fadd_rn(pp.dy0, 4.f), r2, r3, g10, g11, g12,
                           a.alpha_min, a.alpha_max, T1, S10, S11, S12, m, any);
        if (!__any_sync(kFull, any)) continue;
        const float red = transpose_reduce12(m, lane);
        if (writer) atomicAdd(a.mom + (vN + sm.pid[j]) * kMom + my_m, red);
      }
    }
  }
  leave_queue(a, tid);
}

// Persistent grid: SMs x resident CTAs of this kernel (cached per kernel).
unsigned persistent_grid(void (*kernel)(RenderArgs), int threads, int64_t items) {
  struct Entry { const void* k; int dev, ctas; };
  static std::mutex mu;
  static Entry cache[64];
  static int n = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  int ctas = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < n; ++i)
      if (cache[i].k == (const void*)kernel && cache[i].dev == dev) ctas = cache[i].ctas;
    if (!ctas) {
      int sms = 0, per_sm = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0);
      ctas = sms * (per_sm < 1 ? 1 : per_sm);
      if (n < 64) cache[n++] = {(const void*)kernel, dev, ctas};
    }
  }
  return (unsigned)(ctas < items ? ctas : (items > 0 ? items : 1));
}

template <int TS>
cudaError_t launch_fwd_ts(bool alpha, RenderArgs ra, cudaStream_t s) {
  constexpr int NT = Geo<TS>::NT;
  if (ra.stats) {
    ra.queue = Q_STATS;
    if (alpha) {
      auto k = k_render_fwd<TS, true, true>;
      k<<<persistent_grid(k, NT, ra.BT), NT, 0, s>>>(ra);
    } else {
      auto k = k_render_fwd<TS, false, true>;
      k<<<persistent_grid(k, NT, ra.BT), NT, 0, s>>>(ra);
    }
    return cudaGetLastError();
  }
  ra.queue = Q_FWD;
  launch_begin(K_RENDER_FWD, s);
  if (alpha) {
    auto k = k_render_fwd<TS, true, false>;
    k<<<persistent_grid(k, NT, ra.BT), NT, 0, s>>>(ra);
  } else {
    auto k = k_render_fwd<TS, false, false>;
    k<<<persistent_grid(k, NT, ra.BT), NT, 0, s>>>(ra);
  }
  launch_end(K_RENDER_FWD, s);
  return cudaGetLastError();
}

template <int TS>
cudaError_t launch_bwd_ts(bool alpha, RenderArgs ra, cudaStream_t s) {
  constexpr int NT = Geo<TS>::NT;
  ra.queue = Q_BWD;
  launch_begin(K_RENDER_BWD, s);
  if (alpha) {
    auto k = k_render_bwd<TS, true>;
    k<<<persistent_grid(k, NT, ra.BT), NT, 0, s>>>(ra);
  } else {
    auto k = k_render_bwd<TS, false>;
    k<<<persistent_grid(k, NT, ra.BT), NT, 0, s>>>(ra);
  }
  launch_end(K_RENDER_BWD, s);
  return cudaGetLastError();
}

RenderArgs make_args(const wipes_config& c, const Layout& L, char* ws, int final_in_b) {
  RenderArgs ra;
  ra.rec = (const float4*)(ws + L.rec);
  ra.vals = (const uint32_t*)(ws + (final_in_b ? L.valsB : L.valsA));
  ra.toff = (const int32_t*)(ws + L.toff);
  ra.order = (const int32_t*)(ws + L.order);
  ra.hdr = (WsHeader*)(ws + L.hdr);
  ra.N = L.N;
  ra.T = L.T;
  ra.BT = L.BT;
  ra.W = c.width; ra.H = c.height; ra.GX = L.GX;
  ra.queue = 0;
  ra.alpha_min = c.alpha_min;
  // conservative early-out on the exponent: e < log2(alpha_min) - 1e-4 implies
  // alpha*W < alpha_min after the MUFU roundings
  ra.skip_e = c.alpha_min > 0.f ? (float)(log2((double)c.alpha_min) - 1e-4) : -INFINITY;
  ra.alpha_max = c.alpha_max;
  ra.T_min = c.T_min;
  ra.bg0 = c.background[0]; ra.bg1 = c.background[1]; ra.bg2 = c.background[2];
  ra.image = nullptr; ra.T_final = nullptr; ra.n_contrib = nullptr;
  ra.dLdC = nullptr; ra.T_in = nullptr; ra.nc_in = nullptr;
  ra.mom = (float*)(ws + L.rgrad);
  ra.stats = nullptr;
  return ra;
}

}  // namespace

cudaError_t launch_render_fwd(const wipes_config& c, const Layout& L, char* ws, int final_in_b,
                              float* image, float* T_final, int32_t* n_contrib,
                              cudaStream_t s, unsigned long long* stats) {
  if (L.BT == 0) return cudaSuccess;
  RenderArgs ra = make_args(c, L, ws, final_in_b);
  ra.image = image; ra.T_final = T_final; ra.n_contrib = n_contrib;
  ra.stats = stats;
  const bool alpha = c.blend == WIPES_BLEND_ALPHA;
  switch (c.tile) {
    case 8: return launch_fwd_ts<8>(alpha, ra, s);
    case 16: return launch_fwd_ts<16>(alpha, ra, s);
    default: return launch_fwd_ts<32>(alpha, ra, s);
  }
}

cudaError_t launch_render_bwd(const wipes_config& c, const Layout& L, char* ws, int final_in_b,
                              const float* dLdC, const float* T_final,
                              const int32_t* n_contrib, cudaStream_t s) {
  if (L.BT == 0) return cudaSuccess;
  RenderArgs ra = make_args(c, L, ws, final_in_b);
  ra.dLdC = dLdC; ra.T_in = T_final; ra.nc_in = n_contrib;
  const bool alpha = c.blend == WIPES_BLEND_ALPHA;
  switch (c.tile) {
    case 8: return launch_bwd_ts<8>(alpha, ra, s);
    case 16: return launch_bwd_ts<16>(alpha, ra, s);
    default: return launch_bwd_ts<32>(alpha, ra, s);
  }
}

}  // namespace wipes
