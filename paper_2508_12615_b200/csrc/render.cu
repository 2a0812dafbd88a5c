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
// Every WARP is an independent persistent worker (no CTA barriers): it pulls
// work items (view, tile, warp footprint [, record chunk]) from a queue ordered
// longest-tile-list first, walks the tile's sorted record list 32 records at a
// time — each lane loads one 64-byte record, tests it against the warp's
// footprint with the record's conservative opacity extent, and the hits are
// compacted in order (ballot + popc) into warp-private shared memory. A warp
// footprint is G stacked 8x8 blocks (G = 2 for 16/32-pixel tiles, 1 for 8);
// each lane owns 2G pixels: rows y + 8g and y + 8g + 4 of every block g (the
// +4 row evaluated incrementally — the same arithmetic for a given pixel
// whatever the tile size). Branches inside a (warp, record) step are
// warp-uniform (ballots); per-lane decisions are predicated selects. exp is one
// MUFU.EX2 (the -1/2 log2(e) scale and log2(alpha) folded into the record);
// cos / sin are MUFU.COS / MUFU.SIN.
#include <cuda_fp16.h>

#include <mutex>
#include <type_traits>

#include "common.cuh"

namespace wipes {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMom = kMoments;  // 12
#ifndef WIPES_MINB_FWD
#define WIPES_MINB_FWD 8  // __launch_bounds__ min CTAs per SM (register cap), forward
#endif
#ifndef WIPES_MINB_FWD_ALPHA
#define WIPES_MINB_FWD_ALPHA 8  // ... forward, ALPHA
#endif
#ifndef WIPES_MINB_BWD
#define WIPES_MINB_BWD 7  // ... backward, SUM (72 registers with dL/dC in shared memory)
#endif
#ifndef WIPES_MINB_BWD_ALPHA
#define WIPES_MINB_BWD_ALPHA 7  // ... backward, ALPHA (72 registers: C3 -6% against 6)
#endif
#ifndef WIPES_MINB_BWD_F64
#define WIPES_MINB_BWD_F64 6  // ... backward with FP64 moments (SUM and ALPHA)
#endif
constexpr int kWarpsPerCta = 4;
#ifdef WIPES_BWD_COUNT
__device__ unsigned long long g_bwd_cnt[8];
#define BCNT(i, v) do { if (lane == 0) atomicAdd(&g_bwd_cnt[i], (unsigned long long)(v)); } while (0)
#else
#define BCNT(i, v) do { } while (0)
#endif
constexpr int kCta = 32 * kWarpsPerCta;
// Moment accumulation precision (R37): a lane's per-pair moment sums,
// the per-record finish and the warp reduction run in MomT<F64>::T; the
// colour moments M9..M11 (well conditioned) are always summed in FP32.
template <bool F64> struct MomT { typedef float T; };
template <> struct MomT<true> { typedef double T; };
enum { Q_FWD = 0, Q_BWD = 1, Q_STATS = 2 };

#ifndef WIPES_FWD_UNROLL
#define WIPES_FWD_UNROLL 1  // record-loop unroll of the SUM forward (A/B knob)
#endif
#ifndef WIPES_FWD_UNROLL_ALPHA
#define WIPES_FWD_UNROLL_ALPHA 1  // ALPHA forward (packed pairs): 1 and 2 measure the same (C3 2.51 ms)
#endif
#ifndef WIPES_BWD_UNROLL
#define WIPES_BWD_UNROLL 1  // record-loop unroll of the backward (A/B knob)
#endif
constexpr int kBwdUnroll = WIPES_BWD_UNROLL;
// SUM backward: record chunks per (tile, footprint) work item. 0 = by grid size:
// 4 on small frames (items to fill 148 SMs), 2 from 16384 tiles up (fewer partial
// sums / atomics per primitive). A/B on B200 (variants/ab_cfg.sh, gpurun_out/ch_ab.txt):
// C2 bwd 0.119 ms at 4 vs 0.129 at 2; C5 bwd 2.99 ms at 4 vs 2.91 at 2; 6 and 8 slower on both.
#ifndef WIPES_BWD_CHUNKS
#define WIPES_BWD_CHUNKS 0
#endif

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
// Fire-and-forget float add (RED, no return): atomicAdd here compiled to an
// ATOMG whose completion the loop then waited on (long-scoreboard stall at the
// next record's branch: 16% of the C2 backward's stall samples).
__device__ __forceinline__ void red_add(float* p, float v) {
  asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ float4 ldg_nc(const float4* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::evict_last.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
  return v;
}

struct RenderArgs {
  const float4* rec;     // [B*N][4]
  const uint32_t* vals;  // sorted primitive indices
  const int32_t* toff;   // [B*T + 1]
  const int32_t* order;  // [B*T] longest-first tile order
  WsHeader* hdr;         // work queues
  int64_t N, T, BT;
  int32_t W, H, GX, queue;
  int32_t chunks;        // SUM backward: each footprint's list is split into this many items
  float alpha_min, skip_e, alpha_max, T_min;
  float bg0, bg1, bg2;
  float* image;          // [B,3,H,W]
  float* T_final;        // [B,H,W]
  int32_t* n_contrib;    // [B,H,W]
  const float* dLdC;     // [B,3,H,W]
  const float* T_in;
  const int32_t* nc_in;
  float* mom;            // [B*N, 12] gradient moments
  float* mom_beta;       // [B*N] exact mode: M12 = sum gw alpha G cos(theta) (dbeta = M12/2)
  const uint32_t* prevals;  // deterministic mode: sorted vals are dup indices j -> primitive
  float* slots;             // deterministic mode: [cap, fps, slotw] per-(dup, footprint) moments
  uint8_t* slotmask;        // deterministic mode: byte (dup * fps + footprint) = slot written
  int32_t fps, slotw;
  int32_t f64;              // backward: FP64 moment accumulation (R37)
  unsigned long long* stats;  // STATS build: {tile-method candidates, in-ellipse, contributing}
};

#ifndef WIPES_FWD_PACK
#define WIPES_FWD_PACK 1  // SUM forward: a lane's two pixels in packed FP32 (FFMA2/FMUL2)
#endif
#ifndef WIPES_FWD_G
#define WIPES_FWD_G 1  // forward footprint: 8 x 8 (the backward keeps 8 x 16 for TS >= 16)
#endif
template <int TS, int GG = (TS >= 16 ? 2 : 1)>
struct Geo {
  static constexpr int G = GG;                 // 8x8 blocks per warp footprint (stacked)
  static constexpr int P = 2 * G;             // pixels per lane
  static constexpr int FX = TS / 8;           // footprints per tile row
  static constexpr int FY = TS / (8 * G);     // footprints per tile column
  static constexpr int S = FX * FY;           // footprints (work items) per tile
};

// Conservative test: can the record's opacity-extent AABB (padded) touch the
// footprint whose pixel centres span [sx0 + 0.5, sx0 + 7.5] x [sy0 + 0.5, sy0 + h - 0.5]?
// Exact (up to a small margin) test of the record's ellipse {e >= thr} against
// the footprint's pixel-centre rectangle: the exponent e = A dx^2 + B dx dy +
// C dy^2 + log2(alpha) is concave (A, C < 0); if its maximiser (the centre) is
// outside the rectangle, the constrained maximum lies on an edge facing the
// centre (KKT: the active constraint's normal has a positive product with
// centre - argmax), where e is a 1-D concave quadratic maximised in closed form.
__device__ __forceinline__ bool ellipse_hits_rect(const float4& r0, const float4& r1, float sx0,
                                                  float sy0, float h, float thr) {
  const float x0 = (sx0 + 0.5f - r0.x) - r0.z, x1 = x0 + 7.f;
  const float y0 = (sy0 + 0.5f - r0.y) - r0.w, y1 = y0 + (h - 1.f);
  const bool inx = x0 <= 0.f && 0.f <= x1, iny = y0 <= 0.f && 0.f <= y1;
  if (inx && iny) return true;
  const float A = r1.x, B = r1.y, C = r1.z, L = r1.w;
  float best = -INFINITY;
  if (!inx) {  // facing vertical edge x = xe, maximise over y
    const float xe = x0 > 0.f ? x0 : x1;
    const float y = fminf(fmaxf(-B * xe / (2.f * C), y0), y1);
    best = fmaxf(best, fmaf(fmaf(A, xe, B * y), xe, fmaf(C * y, y, L)));
  }
  if (!iny) {  // facing horizontal edge y = ye, maximise over x
    const float ye = y0 > 0.f ? y0 : y1;
    const float x = fminf(fmaxf(-B * ye / (2.f * A), x0), x1);
    best = fmaxf(best, fmaf(fmaf(A, x, B * ye), x, fmaf(C * ye, ye, L)));
  }
  return best >= thr;
}

__device__ __forceinline__ bool hits_footprint(const float4& r0, const float4& r3, float sx0,
                                               float sy0, float h) {
  __half2 e2 = *reinterpret_cast<const __half2*>(&r3.w);
  const float rx = __low2float(e2) + 0.02f, ry = __high2float(e2) + 0.02f;
  const float cx = (r0.x - sx0) + r0.z, cy = (r0.y - sy0) + r0.w;
  return cx + rx >= 0.5f && cx - rx <= 7.5f && cy + ry >= 0.5f && cy - ry <= h - 0.5f;
}

__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }

// Exponents of alpha*G for a lane's pixel pair (rows y0 and y0 + 4) — one
// arithmetic shared by every kernel, so all take the same alpha_min decisions
// (and, since 8x8 blocks are 8-aligned for every tile size, every pixel is
// evaluated by the same expression whatever the tiling).
struct PairPos {
  float dy0, e0, e1;
};

__device__ __forceinline__ float pair_dx(const float4& r0, float px) {
  return __fsub_rn(__fsub_rn(px, r0.x), r0.z);
}

__device__ __forceinline__ PairPos pair_exponents(const float4& r0, const float4& r1, float dx,
                                                  float py0) {
  PairPos p;
  p.dy0 = __fsub_rn(__fsub_rn(py0, r0.y), r0.w);
  const float t = __fmaf_rn(r1.x, dx, __fmul_rn(r1.y, p.dy0));  // A dx + B dy
  const float cdy = __fmul_rn(r1.z, p.dy0);                      // C dy
  p.e0 = __fmaf_rn(t, dx, __fmaf_rn(cdy, p.dy0, r1.w));
  // dy1 = dy0 + 4: e1 = e0 + 4 (B dx + 2 C dy0 + 4 C)
  const float v = __fmaf_rn(r1.y, dx, __fmaf_rn(2.f, cdy, __fmul_rn(4.f, r1.z)));
  p.e1 = __fmaf_rn(4.f, v, p.e0);
  return p;
}

__device__ __forceinline__ float pair_theta(const float4& r2, float dx, float dy) {
  return __fmaf_rn(r2.x, dx, __fmaf_rn(r2.y, dy, r2.z));
}

__device__ __forceinline__ float pair_weight(float ag, float cs, const float4& r2) {
  return __fmul_rn(ag, __fmaf_rn(r2.w, cs, 0.5f));
}

// Warp-private staging area: the compacted hits of the current 32-record chunk.
struct WarpSmem {
  float4 rec[4][32];
  int32_t pid[32];
  int32_t pos[32];
  int32_t dj[32];  // deterministic mode: dup index of the staged record
};

// Backward: the staging area plus the warp's moment-reduction buffer.
struct WarpSmemB : WarpSmem {
  float4 red4[12 * 32 / 4];  // [moment][lane] (16-byte aligned for LDS.128)
};
// SUM backward: each lane's dL/dC values live in warp-private shared memory
// (lane-private slots: written and read by the same lane, no barrier) instead
// of 12 registers, which lets the kernel run 7 CTAs/SM without spills (C2 bwd
// 0.1037 -> 0.1028 ms, C5 2.268 -> 2.205 ms); the ALPHA backward measured
// slower this way (C3 4.61 -> 4.77 ms, also at 8 CTAs/SM) and keeps registers.
#ifndef WIPES_BWD_GSMEM
#define WIPES_BWD_GSMEM 1
#endif
struct WarpSmemBG : WarpSmemB {
  float4 g4[4][32];  // [pixel][lane] (dL/dC r, g, b, -)
};

// One work item of a warp.
struct Item {
  int64_t v, tile;
  int x, y0;       // the lane's column and first row
  float sx0, sy0;  // footprint origin (pixels)
  int start, end;  // record range in the tile list
  int lstart;      // start of the whole tile list (for list positions)
  int sub;         // footprint index within the tile
};

// Work items: lane 0 claims the next index from the queue. With
// WIPES_ITEM_PREFETCH the claim runs one item ahead (`pf` holds the index for
// the NEXT item, so the atomic's round trip overlaps the current item); on small
// frames (C2 forward: 1.3 items per warp) claiming ahead unbalances the warps
// (fwd 60 -> 76 us), so it is off by default. A claimed index >= the item
// count is dropped (nothing behind it).
#ifndef WIPES_STAGE_ALL
#define WIPES_STAGE_ALL 0  // staging: load all four record quads before the footprint tests
#endif
#ifndef WIPES_ITEM_PREFETCH
#define WIPES_ITEM_PREFETCH 0  // claim items one ahead (A/B knob; see next_item)
#endif
template <int TS, int GG = (TS >= 16 ? 2 : 1)>
__device__ __forceinline__ bool next_item(const RenderArgs& a, int lane, int chunks, Item& it,
                                          int& pf) {
  using Gm = Geo<TS, GG>;
  int item = 0;
  if (lane == 0) {
    if (WIPES_ITEM_PREFETCH) {
      item = pf;
      pf = atomicAdd(&a.hdr->work[a.queue], 1);
    } else {
      item = atomicAdd(&a.hdr->work[a.queue], 1);
    }
  }
  item = __shfl_sync(kFull, item, 0);
  if ((int64_t)item >= a.BT * Gm::S * chunks) return false;
  const int chunk = item % chunks;
  const int sub = (item / chunks) % Gm::S;
  it.sub = sub;
  it.tile = a.order[item / (chunks * Gm::S)];
  WCHECK(it.tile >= 0 && it.tile < a.BT);
  it.v = it.tile / a.T;
  const int64_t t_in_v = it.tile - it.v * a.T;
  const int ty = (int)(t_in_v / a.GX), tx = (int)(t_in_v - (int64_t)ty * a.GX);
  const int X0 = tx * TS + (sub % Gm::FX) * 8, Y0 = ty * TS + (sub / Gm::FX) * (8 * Gm::G);
  it.sx0 = (float)X0;
  it.sy0 = (float)Y0;
  it.x = X0 + (lane & 7);
  it.y0 = Y0 + (lane >> 3);
  it.lstart = a.toff[it.tile];
  int end = a.toff[it.tile + 1];
  if (chunks > 1) {
    const int per = (end - it.lstart + chunks - 1) / chunks;
    const int s0 = it.lstart + chunk * per;
    it.end = min(end, s0 + per);
    it.start = min(s0, it.end);
  } else {
    it.start = it.lstart;
    it.end = end;
  }
  return true;
}

__device__ __forceinline__ void leave_queue(const RenderArgs& a, int tid) {
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&a.hdr->done[a.queue], 1) == (int)gridDim.x - 1) {
      a.hdr->work[a.queue] = 0;
      a.hdr->done[a.queue] = 0;
      __threadfence();
    }
  }
}

// Load list entry `idx` (one per lane), test it against the footprint and
// compact the hits into `ws` in list order; returns their count.
template <int G>
__device__ __forceinline__ int stage_chunk(const RenderArgs& a, const float4* recv, int idx,
                                           bool valid, int pos, const Item& it, WarpSmem& ws,
                                           int lane) {
  float4 r0, r1, r2, r3;
  int32_t pid = 0, dj = 0;
  bool hit = false;
  if (valid) {
    pid = (int32_t)a.vals[idx];
    if (a.prevals) {  // deterministic mode: the sorted value is the dup index
      dj = pid;
      pid = (int32_t)a.prevals[dj];
    }
    WCHECK(pid >= 0 && pid < a.N);
    const float4* r = recv + 4 * (int64_t)pid;
    if (WIPES_STAGE_ALL) {  // the whole record at once: one dependent round trip, not three
      r0 = ldg_nc(r); r1 = ldg_nc(r + 1); r2 = ldg_nc(r + 2); r3 = ldg_nc(r + 3);
      hit = hits_footprint(r0, r3, it.sx0, it.sy0, 8.f * G) &&
            ellipse_hits_rect(r0, r1, it.sx0, it.sy0, 8.f * G, a.skip_e - 0.01f);
    } else {
      r0 = ldg_nc(r); r3 = ldg_nc(r + 3);
      hit = hits_footprint(r0, r3, it.sx0, it.sy0, 8.f * G);
      if (hit) {
        r1 = ldg_nc(r + 1);
        hit = ellipse_hits_rect(r0, r1, it.sx0, it.sy0, 8.f * G, a.skip_e - 0.01f);
        if (hit) r2 = ldg_nc(r + 2);
      }
    }
  }
  const uint32_t bal = __ballot_sync(kFull, hit);
  if (hit) {
    const int k = __popc(bal & ((1u << lane) - 1u));
    ws.rec[0][k] = r0; ws.rec[1][k] = r1; ws.rec[2][k] = r2; ws.rec[3][k] = r3;
    ws.pid[k] = pid;
    ws.pos[k] = pos;
    ws.dj[k] = dj;
  }
  __syncwarp();
  return __popc(bal);
}

// Front-to-back alpha compositing step of one pixel (Eq. 3, R9/R10),
// predicated: ok = the pair contributes alpha*W >= alpha_min.
__device__ __forceinline__ void alpha_step(bool ok, float w, const float4& r3, int pos,
                                           float amax, float tmin, float& T, float (&C)[3],
                                           int& last, bool& done, int& stop) {
  const float al = fminf(amax, w);
  const float Tn = __fmul_rn(T, __fsub_rn(1.f, al));
  const bool stp = ok && Tn < tmin;
  const bool comp = ok && !stp;
  const float aT = comp ? __fmul_rn(al, T) : 0.f;
  C[0] = __fmaf_rn(r3.x, aT, C[0]);
  C[1] = __fmaf_rn(r3.y, aT, C[1]);
  C[2] = __fmaf_rn(r3.z, aT, C[2]);
  T = comp ? Tn : T;
  last = comp ? pos : last;
  done = done || stp;
  stop = stp ? pos : stop;
}

template <int TS, bool ALPHA, bool STATS>
__global__ void __launch_bounds__(kCta, ALPHA ? WIPES_MINB_FWD_ALPHA : WIPES_MINB_FWD) k_render_fwd(RenderArgs a) {
  constexpr int GF = (TS >= 16 ? WIPES_FWD_G : 1);
  constexpr int kFwdUnroll = ALPHA ? WIPES_FWD_UNROLL_ALPHA : WIPES_FWD_UNROLL;
  using Gm = Geo<TS, GF>;
  constexpr int G = Gm::G, P = Gm::P;
  __shared__ WarpSmem sm_all[kWarpsPerCta];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  WarpSmem& ws = sm_all[wid];
  unsigned long long st_cand = 0, st_ell = 0, st_con = 0;  // STATS only
  Item it;
  // SUM with two pixels per lane: the pair's colour sums are packed float2
  // accumulators updated by FFMA2 (elementwise identical to two FFMAs)
  constexpr bool PACK = !ALPHA && !STATS && P == 2 && WIPES_FWD_PACK;
  // ALPHA likewise: the pair's transmittances and colour sums packed; the
  // per-pixel decisions (skip, clamp, stop) stay scalar
  constexpr bool PACKA = ALPHA && !STATS && P == 2 && WIPES_FWD_PACK;
  int pf = (WIPES_ITEM_PREFETCH && lane == 0) ? atomicAdd(&a.hdr->work[a.queue], 1) : 0;
  while (next_item<TS, GF>(a, lane, 1, it, pf)) {
    bool in[P], done[P];
    float C[P][3], T[P];
    float2 Cp[3] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    float2 Tp = make_float2(1.f, 1.f);
    int last[P], stop[P];
    const int len = it.end - it.start;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int y = it.y0 + 8 * (p >> 1) + 4 * (p & 1);
      in[p] = it.x < a.W && y < a.H;
      done[p] = ALPHA ? !in[p] : false;
      C[p][0] = C[p][1] = C[p][2] = 0.f;
      T[p] = 1.f;
      last[p] = 0;
      stop[p] = len;
    }
    const float px = (float)it.x + 0.5f, py0 = (float)it.y0 + 0.5f;
    const float4* recv = a.rec + 4 * (it.v * a.N);
    for (int b0 = it.start; b0 < it.end; b0 += 32) {
      if (ALPHA) {
        bool all = true;
#pragma unroll
        for (int p = 0; p < P; ++p) all = all && done[p];
        if (__all_sync(kFull, all)) break;
      }
      const bool valid = b0 + lane < it.end;
      const int cnt = stage_chunk<G>(a, recv, b0 + lane, valid, b0 - it.start + lane + 1, it, ws,
                                     lane);
#pragma unroll kFwdUnroll
      for (int i = 0; i < cnt; ++i) {
        const float4 r0 = ws.rec[0][i], r1 = ws.rec[1][i];
        const float dx = pair_dx(r0, px);
        float e[P], dy[P];
        bool h[P];
        uint32_t any = 0, bm[P];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const PairPos pp = pair_exponents(r0, r1, dx, py0 + 8.f * g);
          e[2 * g] = pp.e0; e[2 * g + 1] = pp.e1;
          dy[2 * g] = pp.dy0; dy[2 * g + 1] = pp.dy0 + 4.f;
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
          h[p] = e[p] >= a.skip_e && !done[p];
          if (STATS) st_ell += h[p] && in[p];
          bm[p] = __ballot_sync(kFull, h[p]);
          any |= bm[p];
        }
        if (!any) continue;
        const float4 r2 = ws.rec[2][i], r3 = ws.rec[3][i];
        const int pos = ws.pos[i];
        if constexpr (PACK) {
          // theta = fx dx + (fy dy + phi) and w = ag (1/2 + beta/2 cos theta) in the
          // same expression order as the scalar pair_theta / pair_weight
          const float2 th = __ffma2_rn(make_float2(r2.x, r2.x), make_float2(dx, dx),
                                       __ffma2_rn(make_float2(r2.y, r2.y),
                                                  make_float2(dy[0], dy[1]),
                                                  make_float2(r2.z, r2.z)));
          const float2 ag = make_float2(ex2(e[0]), ex2(e[1]));
          const float2 hw = __ffma2_rn(make_float2(r2.w, r2.w),
                                       make_float2(cos_a(th.x), cos_a(th.y)),
                                       make_float2(0.5f, 0.5f));
          const float2 w = __fmul2_rn(ag, hw);
          // h (e >= skip_e) is implied by w >= alpha_min here: skip_e sits 1e-4 below
          // log2(alpha_min) and w <= ag (beta <= 1), so the gate is the w test alone
          const float2 we = make_float2(w.x >= a.alpha_min ? w.x : 0.f,
                                        w.y >= a.alpha_min ? w.y : 0.f);
          Cp[0] = __ffma2_rn(make_float2(r3.x, r3.x), we, Cp[0]);
          Cp[1] = __ffma2_rn(make_float2(r3.y, r3.y), we, Cp[1]);
          Cp[2] = __ffma2_rn(make_float2(r3.z, r3.z), we, Cp[2]);
          continue;
        }
        if constexpr (PACKA) {
          const float2 th = __ffma2_rn(f2(r2.x), f2(dx),
                                       __ffma2_rn(f2(r2.y), make_float2(dy[0], dy[1]), f2(r2.z)));
          const float2 ag = make_float2(ex2(e[0]), ex2(e[1]));
          const float2 w = __fmul2_rn(ag, __ffma2_rn(f2(r2.w), make_float2(cos_a(th.x), cos_a(th.y)),
                                                     f2(0.5f)));
          const bool ok0 = h[0] && w.x >= a.alpha_min, ok1 = h[1] && w.y >= a.alpha_min;
          // alpha_step on both pixels: al = min(amax, w), T' = T (1 - al), stop if
          // T' < T_min (not composited), else C += c al T, T = T'
          const float2 al = make_float2(fminf(a.alpha_max, w.x), fminf(a.alpha_max, w.y));
          const float2 Tn = __fmul2_rn(Tp, __fadd2_rn(f2(1.f), make_float2(-al.x, -al.y)));
          const bool stp0 = ok0 && Tn.x < a.T_min, stp1 = ok1 && Tn.y < a.T_min;
          const bool cmp0 = ok0 && !stp0, cmp1 = ok1 && !stp1;
          const float2 aT = __fmul2_rn(al, Tp);
          const float2 aTs = make_float2(cmp0 ? aT.x : 0.f, cmp1 ? aT.y : 0.f);
          Cp[0] = __ffma2_rn(f2(r3.x), aTs, Cp[0]);
          Cp[1] = __ffma2_rn(f2(r3.y), aTs, Cp[1]);
          Cp[2] = __ffma2_rn(f2(r3.z), aTs, Cp[2]);
          Tp = make_float2(cmp0 ? Tn.x : Tp.x, cmp1 ? Tn.y : Tp.y);
          last[0] = cmp0 ? pos : last[0];
          last[1] = cmp1 ? pos : last[1];
          done[0] = done[0] || stp0;
          done[1] = done[1] || stp1;
          stop[0] = stp0 ? pos : stop[0];
          stop[1] = stp1 ? pos : stop[1];
          if (__all_sync(kFull, done[0] && done[1])) break;
          continue;
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
          if (!bm[p]) continue;
          const float w = pair_weight(ex2(e[p]), cos_a(pair_theta(r2, dx, dy[p])), r2);
          const bool ok = h[p] && w >= a.alpha_min;
          if (!ALPHA) {
            const float we = ok ? w : 0.f;
            if (STATS) st_con += ok && in[p];
            C[p][0] = __fmaf_rn(r3.x, we, C[p][0]);
            C[p][1] = __fmaf_rn(r3.y, we, C[p][1]);
            C[p][2] = __fmaf_rn(r3.z, we, C[p][2]);
          } else {
            alpha_step(ok, w, r3, pos, a.alpha_max, a.T_min, T[p], C[p], last[p], done[p],
                       stop[p]);
            if (STATS) st_con += ok && !(done[p] && stop[p] == pos);
          }
        }
        if (ALPHA) {
          bool all = true;
#pragma unroll
          for (int p = 0; p < P; ++p) all = all && done[p];
          if (__all_sync(kFull, all)) break;
        }
      }
      __syncwarp();
    }
    if (STATS) {
#pragma unroll
      for (int p = 0; p < P; ++p) st_cand += in[p] ? (unsigned long long)stop[p] : 0ull;
      continue;
    }
    const int64_t HW = (int64_t)a.H * a.W;
    float* img = a.image + it.v * 3 * HW;
    if constexpr (PACK || PACKA) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        C[0][c] = Cp[c].x;
        C[1][c] = Cp[c].y;
      }
      if (PACKA) {
        T[0] = Tp.x;
        T[1] = Tp.y;
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (!in[p]) continue;
      const int64_t q = (int64_t)(it.y0 + 8 * (p >> 1) + 4 * (p & 1)) * a.W + it.x;
      if (ALPHA) {
        C[p][0] = __fmaf_rn(T[p], a.bg0, C[p][0]);
        C[p][1] = __fmaf_rn(T[p], a.bg1, C[p][1]);
        C[p][2] = __fmaf_rn(T[p], a.bg2, C[p][2]);
        a.T_final[it.v * HW + q] = T[p];
        a.n_contrib[it.v * HW + q] = last[p];
      }
      WCHECK(q >= 0 && q < HW);
      img[q] = C[p][0]; img[HW + q] = C[p][1]; img[2 * HW + q] = C[p][2];
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
template <typename mom_t>
__device__ __forceinline__ mom_t transpose_reduce12(mom_t (&v)[kMom], int lane) {
  {
    const bool up = lane & 16;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      mom_t send = up ? v[k] : v[k + 6];
      mom_t keep = up ? v[k + 6] : v[k];
      v[k] = keep + __shfl_xor_sync(kFull, send, 16);
    }
  }
  {
    const bool up = lane & 8;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      mom_t send = up ? v[k] : v[k + 3];
      mom_t keep = up ? v[k + 3] : v[k];
      v[k] = keep + __shfl_xor_sync(kFull, send, 8);
    }
  }
  {
    const bool up = lane & 4;  // pairs (0, 2) and (1, pad)
    mom_t s0 = up ? v[0] : v[2], k0 = up ? v[2] : v[0];
    mom_t s1 = up ? v[1] : (mom_t)0, k1 = up ? (mom_t)0 : v[1];
    v[0] = k0 + __shfl_xor_sync(kFull, s0, 4);
    v[1] = k1 + __shfl_xor_sync(kFull, s1, 4);
  }
  {
    const bool up = lane & 2;
    mom_t s = up ? v[0] : v[1], k = up ? v[1] : v[0];
    v[0] = k + __shfl_xor_sync(kFull, s, 2);
  }
  return v[0] + __shfl_xor_sync(kFull, v[0], 1);
}

// Column-first reduction of a lane's 8 dx-free moment sums (m0, m2, m5, m6, m8,
// c0, c1, c2): lanes l ^ 8 and l ^ 16 hold the same pixel column (lane & 7, one
// dx), so the first two transposing levels sum each column's 8 values over its 4
// lanes, the dx products are formed once per column on the column sums
// (M1 = M0 dx, M3 = M1 dx, M4 = M2 dx, M7 = M6 dx: exact factorisations, as in
// finish_moments), and three more levels sum the 8 columns. 10 SHFL, 18 FSEL,
// 10 FADD and 2 FMUL per record instead of finish_moments + transpose_reduce12's
// 4 FMUL, 13 SHFL, 24 FSEL and 13 FADD. After the reduction lane l holds the
// moment col_first_moment(l) (kMom for a pad slot).
__device__ __forceinline__ int col_first_moment(int lane) {
  // group (b4, b3) -> its four outputs o0..o3 (o = 2 b2 + b1), one nibble each:
  // (0,0): M0 M9 M1 M3 | (0,1): M2 M5 M4 - | (1,0): M6 M8 M7 - | (1,1): M10 M11 - -
  static_assert(kMoments == 12, "nibble table");
  const int idx = ((lane >> 3) & 3) * 4 + ((lane >> 1) & 3);
  return (int)((0xccbac786c4523190ull >> (4 * idx)) & 0xfull);
}
template <typename mom_t>
__device__ __forceinline__ mom_t col_first_reduce(const mom_t (&m)[9], const mom_t (&mc)[3],
                                                  float dx, int lane) {
  // level A (xor 16): b4 = 0 keeps {m0, c0, m2, m5}, b4 = 1 keeps {m6, m8, c1, c2}
  const mom_t s0[4] = {m[0], mc[0], m[2], m[5]};
  const mom_t s1[4] = {m[6], m[8], mc[1], mc[2]};
  mom_t t[4];
  {
    const bool up = lane & 16;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const mom_t send = up ? s0[j] : s1[j];
      const mom_t keep = up ? s1[j] : s0[j];
      t[j] = keep + __shfl_xor_sync(kFull, send, 16);
    }
  }
  // level B (xor 8): b3 = 0 keeps t0, t1; b3 = 1 keeps t2, t3 -> column sums
  // (0,0): (M0, M9), (0,1): (M2, M5), (1,0): (M6, M8), (1,1): (M10, M11)
  mom_t o[4];
  {
    const bool up = lane & 8;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const mom_t send = up ? t[j] : t[j + 2];
      const mom_t keep = up ? t[j + 2] : t[j];
      o[j] = keep + __shfl_xor_sync(kFull, send, 8);
    }
  }
  const mom_t d = (mom_t)dx;
  o[2] = o[0] * d;  // M1 | M4 | M7 | pad
  o[3] = o[2] * d;  // M3 | pad ...
  {  // level C (xor 4): b2 = 0 keeps o0, o1; b2 = 1 keeps o2, o3
    const bool up = lane & 4;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const mom_t send = up ? o[j] : o[j + 2];
      const mom_t keep = up ? o[j + 2] : o[j];
      o[j] = keep + __shfl_xor_sync(kFull, send, 4);
    }
  }
  {  // level D (xor 2)
    const bool up = lane & 2;
    const mom_t send = up ? o[0] : o[1];
    const mom_t keep = up ? o[1] : o[0];
    o[0] = keep + __shfl_xor_sync(kFull, send, 2);
  }
  return o[0] + __shfl_xor_sync(kFull, o[0], 1);
}

#ifndef WIPES_COLFIRST
#define WIPES_COLFIRST 1  // column-first moment reduction (0: finish_moments + transpose_reduce12)
#endif
#ifndef WIPES_SMEM_REDUCE
#define WIPES_SMEM_REDUCE 0  // A/B knob: measured slower (C2 bwd 0.126 vs 0.114 ms, C5 3.07 vs 2.55)
#endif
// 12-moment warp reduction through the warp's shared buffer: every lane stores
// its 12 partial moments moment-major (12 conflict-free STS), then lane 2k + h
// (k < 12) sums the 16 values of moment k from lanes 16h..16h + 15 (four
// LDS.128, fixed order) and the pair combines with one shuffle: lane 2k holds
// moment k. ~35 instructions instead of the transpose-reduce's ~60 (13 SHFL,
// 24 FSEL, 13 FADD); deterministic order.
__device__ __forceinline__ float smem_reduce12(const float (&v)[kMom], float4* buf4, int lane) {
  float* buf = reinterpret_cast<float*>(buf4);
#pragma unroll
  for (int k = 0; k < kMom; ++k) buf[k * 32 + lane] = v[k];
  __syncwarp();
  float s = 0.f;
  if (lane < 2 * kMom) {
    const float4* q = buf4 + (lane >> 1) * 8 + (lane & 1) * 4;
    const float4 a = q[0], b = q[1], c = q[2], d = q[3];
    s = (((a.x + a.y) + (a.z + a.w)) + ((b.x + b.y) + (b.z + b.w))) +
        (((c.x + c.y) + (c.z + c.w)) + ((d.x + d.y) + (d.z + d.w)));
  }
  s += __shfl_xor_sync(kFull, s, 1);
  __syncwarp();  // the buffer is rewritten by the next record
  return s;
}

// Moments of one pair, gw = dL/dw and w already zeroed when the
// pair does not contribute: M0 = gw w, M1 = gw w dx, M2 = gw w dy,
// M3 = gw w dx^2, M4 = gw w dx dy, M5 = gw w dy^2, M6 = gw ag sin, M7 = M6 dx,
// M8 = M6 dy, M9..11 = dL/dc terms. A lane's pixels share dx (one column), so
// the lane sums M0, M2, M5, M6, M8 (each pixel with its own dy) and
// finish_moments applies dx once per record (M1 = M0 dx, M3 = M0 dx^2,
// M4 = M2 dx, M7 = M6 dx: exact factorisations, no cancellation). An earlier
// expansion of the dy sums about the lane's first row (dy0^2 M0 + 2 dy0 S_ky +
// S_ky2) cancelled when dy0 ~ -ky and is gone (R37).
template <bool F64>
__device__ __forceinline__ void add_moments(typename MomT<F64>::T (&m)[9], float (&mc)[3],
                                            float gw, float w, float ag, float sn,
                                            typename MomT<F64>::T dy, float c0, float c1,
                                            float c2) {
  typedef typename MomT<F64>::T T;
#ifdef WIPES_EXP_FPROD  // experiment: FP32 products widened (FP64 path)
  const T gww = (T)(gw * w);
  const T m6 = (T)(gw * (ag * sn));
#else
  // FP64: the products are exact (a product of two floats fits a double) or
  // rounded once at 2^-53; FP32: one rounding each
  const T gwT = (T)gw;
  const T gww = gwT * (T)w;
  const T m6 = (gwT * (T)ag) * (T)sn;
#endif
  const T gwy = gww * dy;
  m[0] += gww;
  m[2] += gwy;
  m[5] = fma(gwy, dy, m[5]);
  m[6] += m6;
  m[8] = fma(m6, dy, m[8]);
  mc[0] += c0;
  mc[1] += c1;
  mc[2] += c2;
}

template <bool F64>
__device__ __forceinline__ void finish_moments(typename MomT<F64>::T (&r)[kMom],
                                               const typename MomT<F64>::T (&m)[9],
                                               const float (&mc)[3], float dx) {
  typedef typename MomT<F64>::T T;
  const T d = (T)dx;
  r[0] = m[0];
  r[2] = m[2];
  r[5] = m[5];
  r[6] = m[6];
  r[8] = m[8];
  r[1] = m[0] * d;
  r[3] = r[1] * d;
  r[4] = m[2] * d;
  r[7] = m[6] * d;
  r[9] = (T)mc[0];
  r[10] = (T)mc[1];
  r[11] = (T)mc[2];
}

// ALPHA: T is the transmittance in front of the pixel's current record, sdg =
// S.g with S the colour accumulated behind it (incl. T_final bg); since
// S' = S + c aT, sdg is carried directly: sdg' = sdg + (c.g) aT. A
// non-contributing pair gets al = 0, so rcp(1) = 1 leaves T, sdg unchanged and
// aT = 0 without selects; only dL/dw needs the gate.
template <bool ALPHA, bool EXACT, bool F64>
__device__ __forceinline__ void bwd_pixel(bool h, float e, float dx, float dy,
                                          typename MomT<F64>::T dym, const float4& r2,
                                          const float4& r3, const float (&g)[3], float amin,
                                          float amax, float& T, float& sdg,
                                          typename MomT<F64>::T (&m)[9], float (&mc)[3],
                                          float& mb, float& any) {
  const float ag = ex2(e);
  const float th = pair_theta(r2, dx, dy);
  const float cs = cos_a(th), sn = sin_a(th);
  const float w = pair_weight(ag, cs, r2);
  const bool ok = h && w >= amin;
  const float gdc = __fmaf_rn(r3.x, g[0], __fmaf_rn(r3.y, g[1], __fmul_rn(r3.z, g[2])));
  if (!ALPHA) {
    const float we = ok ? w : 0.f;
    any += we;  // > 0 iff some pair contributed (w >= alpha_min > 0): one FADD, no bool
    add_moments<F64>(m, mc, ok ? gdc : 0.f, we, ag, sn, dym, we * g[0], we * g[1], we * g[2]);
    if (EXACT) mb = __fmaf_rn(ok ? gdc * ag : 0.f, cs, mb);
  } else {
    const float al = ok ? fminf(amax, w) : 0.f;
    any += al;
    const float ri = rcp_a(1.f - al);  // exactly 1 when al = 0
    const float Tk = T * ri;
    const float dLda = __fmaf_rn(Tk, gdc, -sdg * ri);
    const float aT = al * Tk;
    sdg = __fmaf_rn(gdc, aT, sdg);
    T = Tk;
    const float gw = (ok && w < amax) ? dLda : 0.f;
    add_moments<F64>(m, mc, gw, w, ag, sn, dym, aT * g[0], aT * g[1], aT * g[2]);
    if (EXACT) mb = __fmaf_rn(gw * ag, cs, mb);
  }
}

#ifndef WIPES_BWD_PACK
#define WIPES_BWD_PACK 0  // FP32 backward in FFMA2 pairs: A/B knob, measured slower (register spills), off
#endif

// Packed moment sums of a lane (FP32 path): .x collects the pairs' first
// pixels (rows y0, y0 + 8), .y the second (y0 + 4, y0 + 12); the two halves
// are added once per record. Same moments as add_moments (M0, M2, M5, M6, M8,
// M9..11).
struct MomPack {
  float2 m0, m2, m5, m6, m8, c0, c1, c2;
};

// bwd_pixel for the two pixels of a lane's pair (same column, rows dy and
// dy + 4), every FP32 operation packed where both pixels take the same one
// (elementwise the scalar expressions, in the same order).
template <bool ALPHA, bool EXACT>
__device__ __forceinline__ void bwd_pair(bool h0, bool h1, float e0, float e1, float dx,
                                         float2 dy, const float4& r2, const float4& r3,
                                         const float2 (&g)[3], float amin, float amax,
                                         float2& T, float2& sdg, MomPack& m, float& mb,
                                         float& any) {
  const float2 ag = make_float2(ex2(e0), ex2(e1));
  const float2 th = __ffma2_rn(f2(r2.x), f2(dx), __ffma2_rn(f2(r2.y), dy, f2(r2.z)));
  const float2 cs = make_float2(cos_a(th.x), cos_a(th.y));
  const float2 sn = make_float2(sin_a(th.x), sin_a(th.y));
  const float2 w = __fmul2_rn(ag, __ffma2_rn(f2(r2.w), cs, f2(0.5f)));
  const bool ok0 = h0 && w.x >= amin, ok1 = h1 && w.y >= amin;
  const float2 gdc = __ffma2_rn(f2(r3.x), g[0], __ffma2_rn(f2(r3.y), g[1], __fmul2_rn(f2(r3.z), g[2])));
  float2 gw, wm, cw;
  if (!ALPHA) {
    wm = make_float2(ok0 ? w.x : 0.f, ok1 ? w.y : 0.f);
    gw = make_float2(ok0 ? gdc.x : 0.f, ok1 ? gdc.y : 0.f);
    cw = wm;
    any += wm.x + wm.y;
    if (EXACT) {
      mb = __fmaf_rn(gw.x * ag.x, cs.x, mb);
      mb = __fmaf_rn(gw.y * ag.y, cs.y, mb);
    }
  } else {
    const float2 al = make_float2(ok0 ? fminf(amax, w.x) : 0.f, ok1 ? fminf(amax, w.y) : 0.f);
    any += al.x + al.y;
    const float2 ri = make_float2(rcp_a(1.f - al.x), rcp_a(1.f - al.y));  // 1 when al = 0
    const float2 Tk = __fmul2_rn(T, ri);
    const float2 dLda = __ffma2_rn(Tk, gdc, __fmul2_rn(make_float2(-sdg.x, -sdg.y), ri));
    const float2 aT = __fmul2_rn(al, Tk);
    sdg = __ffma2_rn(gdc, aT, sdg);
    T = Tk;
    gw = make_float2((ok0 && w.x < amax) ? dLda.x : 0.f, (ok1 && w.y < amax) ? dLda.y : 0.f);
    wm = w;
    cw = aT;
    if (EXACT) {
      mb = __fmaf_rn(gw.x * ag.x, cs.x, mb);
      mb = __fmaf_rn(gw.y * ag.y, cs.y, mb);
    }
  }
  const float2 gww = __fmul2_rn(gw, wm);
  const float2 m6 = __fmul2_rn(gw, __fmul2_rn(ag, sn));
  const float2 gwy = __fmul2_rn(gww, dy);
  m.m0 = __fadd2_rn(m.m0, gww);
  m.m2 = __fadd2_rn(m.m2, gwy);
  m.m5 = __ffma2_rn(gwy, dy, m.m5);
  m.m6 = __fadd2_rn(m.m6, m6);
  m.m8 = __ffma2_rn(m6, dy, m.m8);
  m.c0 = __ffma2_rn(cw, g[0], m.c0);
  m.c1 = __ffma2_rn(cw, g[1], m.c1);
  m.c2 = __ffma2_rn(cw, g[2], m.c2);
}

template <int TS, bool ALPHA, bool EXACT, bool F64, bool DET>
__global__ void __launch_bounds__(kCta, F64 ? WIPES_MINB_BWD_F64
                                            : (ALPHA ? WIPES_MINB_BWD_ALPHA : WIPES_MINB_BWD))
    k_render_bwd(RenderArgs a) {
  typedef typename MomT<F64>::T MT;
  using Gm = Geo<TS>;
  constexpr int G = Gm::G, P = Gm::P;
  constexpr bool PACKB = !F64 && WIPES_BWD_PACK;
  constexpr bool GSM = !ALPHA && WIPES_BWD_GSMEM;
  using WS = std::conditional_t<GSM, WarpSmemBG, WarpSmemB>;
  __shared__ WS sm_all[kWarpsPerCta];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  WS& ws = sm_all[wid];
  // which moment this lane holds after the warp reduction (and writes out)
  constexpr bool SMRED = !F64 && WIPES_SMEM_REDUCE;
  constexpr bool COLF = !SMRED && WIPES_COLFIRST;
  const int q3 = (lane >> 1) & 3;
  const int my_m = SMRED ? (lane >> 1)
                         : (COLF ? col_first_moment(lane)
                                 : 6 * ((lane >> 4) & 1) + 3 * ((lane >> 3) & 1) + q3);
  const bool writer = SMRED ? (!(lane & 1) && lane < 2 * kMom)
                            : (COLF ? (!(lane & 1) && my_m < kMom) : (!(lane & 1) && q3 < 3));
  // the moment this lane writes, kMom if none, held in a register the compiler
  // cannot rematerialise (it recomputed the lane arithmetic for every record)
  int wm;
  asm volatile("mov.b32 %0, %1;" : "=r"(wm) : "r"(writer ? my_m : kMom));
  Item it;
  int pf = (WIPES_ITEM_PREFETCH && lane == 0) ? atomicAdd(&a.hdr->work[a.queue], 1) : 0;
  while (next_item<TS>(a, lane, ALPHA ? 1 : a.chunks, it, pf)) {
    const int64_t HW = (int64_t)a.H * a.W;
    const float* gp = a.dLdC + it.v * 3 * HW;
    bool in[P];
    float g[P][3], T[P], sdg[P];
    int last[P];
    int ml = 0;
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int y = it.y0 + 8 * (p >> 1) + 4 * (p & 1);
      in[p] = it.x < a.W && y < a.H;
      g[p][0] = g[p][1] = g[p][2] = 0.f;
      T[p] = 1.f;
      sdg[p] = 0.f;
      last[p] = 0;
      if (in[p]) {
        const int64_t q = (int64_t)y * a.W + it.x;
        g[p][0] = gp[q]; g[p][1] = gp[HW + q]; g[p][2] = gp[2 * HW + q];
        if (ALPHA) {
          T[p] = a.T_in[it.v * HW + q];
          last[p] = a.nc_in[it.v * HW + q];
          sdg[p] = T[p] * __fmaf_rn(a.bg0, g[p][0], __fmaf_rn(a.bg1, g[p][1], a.bg2 * g[p][2]));
          ml = max(ml, last[p]);
        }
      }
      if constexpr (GSM) ws.g4[p][lane] = make_float4(g[p][0], g[p][1], g[p][2], 0.f);
    }
    // packed per-pair state of the FP32 path (pair gg = pixels 2gg, 2gg + 1)
    float2 g2[G][3], T2[G], sdg2[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
#pragma unroll
      for (int c = 0; c < 3; ++c) g2[gg][c] = make_float2(g[2 * gg][c], g[2 * gg + 1][c]);
      T2[gg] = make_float2(T[2 * gg], T[2 * gg + 1]);
      sdg2[gg] = make_float2(sdg[2 * gg], sdg[2 * gg + 1]);
    }
    int start = it.start, end = it.end;
    if (ALPHA) {  // only entries before this warp's last composited one matter
#pragma unroll
      for (int off = 16; off; off >>= 1) ml = max(ml, __shfl_xor_sync(kFull, ml, off));
      end = it.lstart + ml;
    }
    const float px = (float)it.x + 0.5f, py0 = (float)it.y0 + 0.5f;
    const float4* recv = a.rec + 4 * (it.v * a.N);
    const int64_t vN = it.v * a.N;
    // ALPHA walks 32-record chunks back to front; SUM front to back.
    const int nchunk = (end - start + 31) / 32;
    for (int ci = 0; ci < nchunk; ++ci) {
      const int b0 = ALPHA ? end - 32 * (ci + 1) : start + 32 * ci;
      const bool valid = b0 + lane >= start && b0 + lane < end;
      const int cnt = stage_chunk<G>(a, recv, b0 + lane, valid, b0 + lane - it.lstart, it, ws,
                                     lane);
      BCNT(0, cnt);
      BCNT(5, 1);
#pragma unroll kBwdUnroll
      for (int ii = 0; ii < cnt; ++ii) {
        const int i = ALPHA ? cnt - 1 - ii : ii;
        const int pos = ws.pos[i];  // index within the tile list
        const float4 r0 = ws.rec[0][i], r1 = ws.rec[1][i];
        const float dx = pair_dx(r0, px);
        float e[P], dy[P];
        bool h[P];
        uint32_t any_h = 0, bm[P];
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          const PairPos pp = pair_exponents(r0, r1, dx, py0 + 8.f * gg);
          e[2 * gg] = pp.e0; e[2 * gg + 1] = pp.e1;
          dy[2 * gg] = pp.dy0; dy[2 * gg + 1] = pp.dy0 + 4.f;
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
          h[p] = in[p] && e[p] >= a.skip_e && (!ALPHA || pos < last[p]);
          bm[p] = __ballot_sync(kFull, h[p]);
          any_h |= bm[p];
        }
        if (!any_h) continue;
#ifdef WIPES_BWD_COUNT
        {
          int ns = 0, nl = 0;
#pragma unroll
          for (int p = 0; p < P; ++p) { ns += bm[p] != 0; nl += __popc(bm[p]); }
          BCNT(1, 1); BCNT(2, ns); BCNT(4, nl);
        }
#endif
        const float4 r2 = ws.rec[2][i], r3 = ws.rec[3][i];
        MT m[9];
        float mc[3] = {0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < 9; ++k) m[k] = 0;
        float any = 0.f;  // sum of the contributing pairs' weights (> 0 iff any)
        float mb = 0.f;
        if constexpr (PACKB) {
          MomPack mp;
          mp.m0 = mp.m2 = mp.m5 = mp.m6 = mp.m8 = mp.c0 = mp.c1 = mp.c2 = f2(0.f);
#pragma unroll
          for (int gg = 0; gg < G; ++gg)
            if (bm[2 * gg] | bm[2 * gg + 1])
              bwd_pair<ALPHA, EXACT>(h[2 * gg], h[2 * gg + 1], e[2 * gg], e[2 * gg + 1], dx,
                                     make_float2(dy[2 * gg], dy[2 * gg + 1]), r2, r3, g2[gg],
                                     a.alpha_min, a.alpha_max, T2[gg], sdg2[gg], mp, mb, any);
          m[0] = mp.m0.x + mp.m0.y;
          m[2] = mp.m2.x + mp.m2.y;
          m[5] = mp.m5.x + mp.m5.y;
          m[6] = mp.m6.x + mp.m6.y;
          m[8] = mp.m8.x + mp.m8.y;
          mc[0] = mp.c0.x + mp.c0.y;
          mc[1] = mp.c1.x + mp.c1.y;
          mc[2] = mp.c2.x + mp.c2.y;
        } else {
          // FP64: each pixel's dy exactly as dy0 + ky (dy0 converted once per record)
          const MT dy0m = (MT)dy[0];
#pragma unroll
          for (int p = 0; p < P; ++p)
            if (bm[p]) {
              float gl[3];
              if constexpr (GSM) {
                const float4 gv = ws.g4[p][lane];
                gl[0] = gv.x; gl[1] = gv.y; gl[2] = gv.z;
              } else {
                gl[0] = g[p][0]; gl[1] = g[p][1]; gl[2] = g[p][2];
              }
              bwd_pixel<ALPHA, EXACT, F64>(h[p], e[p], dx, dy[p],
                                           F64 ? dy0m + (MT)(8 * (p >> 1) + 4 * (p & 1))
                                               : (MT)dy[p],
                                           r2, r3, gl, a.alpha_min, a.alpha_max, T[p], sdg[p],
                                           m, mc, mb, any);
            }
        }
        if (!__any_sync(kFull, any > 0.f)) continue;
        BCNT(3, 1);
        float red;
        if constexpr (COLF) {
          const MT mcm[3] = {(MT)mc[0], (MT)mc[1], (MT)mc[2]};
          red = (float)col_first_reduce<MT>(m, mcm, dx, lane);
        } else {
          MT mr[kMom];
          finish_moments<F64>(mr, m, mc, dx);
          if constexpr (SMRED) {
            red = smem_reduce12(mr, ws.red4, lane);
          } else {
            red = (float)transpose_reduce12(mr, lane);
          }
        }
        if (EXACT) {
#pragma unroll
          for (int off = 16; off; off >>= 1) mb += __shfl_xor_sync(kFull, mb, off);
        }
        if constexpr (DET) {  // deterministic: this warp's slot of (dup, footprint); no atomics
          const int64_t si = (int64_t)ws.dj[i] * a.fps + it.sub;
          WCHECK(ws.dj[i] >= 0 && it.sub < a.fps);
          float* sl = a.slots + si * a.slotw;
          if (writer) sl[my_m] = red;
          if (EXACT && lane == 0) sl[kMom] = mb;
          if (lane == 0) a.slotmask[si] = 1;
        } else {
          WCHECK(wm >= kMom || (wm >= 0 && ws.pid[i] >= 0 && ws.pid[i] < a.N));
          if (wm < kMom) red_add(a.mom + (vN + ws.pid[i]) * kMom + wm, red);
          if (EXACT && lane == 0) red_add(a.mom_beta + vN + ws.pid[i], mb);
        }
      }
      __syncwarp();
    }
  }
  leave_queue(a, tid);
}

// Persistent grid: SMs x resident CTAs of this kernel (cached per kernel).
unsigned persistent_grid(void (*kernel)(RenderArgs), int64_t items) {
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
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kCta, 0);
      ctas = sms * (per_sm < 1 ? 1 : per_sm);
      if (n < 64) cache[n++] = {(const void*)kernel, dev, ctas};
    }
  }
  const int64_t need = (items + kWarpsPerCta - 1) / kWarpsPerCta;
  return (unsigned)(ctas < need ? ctas : (need > 0 ? need : 1));
}

template <int TS>
cudaError_t launch_fwd_ts(bool alpha, RenderArgs ra, cudaStream_t s) {
  const int64_t items = ra.BT * Geo<TS, (TS >= 16 ? WIPES_FWD_G : 1)>::S;
  void (*k)(RenderArgs);
  if (ra.stats) {
    ra.queue = Q_STATS;
    k = alpha ? k_render_fwd<TS, true, true> : k_render_fwd<TS, false, true>;
    k<<<persistent_grid(k, items), kCta, 0, s>>>(ra);
    return cudaGetLastError();
  }
  ra.queue = Q_FWD;
  k = alpha ? k_render_fwd<TS, true, false> : k_render_fwd<TS, false, false>;
  launch_begin(K_RENDER_FWD, s);
  k<<<persistent_grid(k, items), kCta, 0, s>>>(ra);
  launch_end(K_RENDER_FWD, s);
  return cudaGetLastError();
}

template <int TS, bool DET>
void (*pick_bwd(bool alpha, bool exact, bool f64))(RenderArgs) {
  if (f64) {
    if (exact)
      return alpha ? k_render_bwd<TS, true, true, true, DET> : k_render_bwd<TS, false, true, true, DET>;
    return alpha ? k_render_bwd<TS, true, false, true, DET> : k_render_bwd<TS, false, false, true, DET>;
  }
  if (exact)
    return alpha ? k_render_bwd<TS, true, true, false, DET> : k_render_bwd<TS, false, true, false, DET>;
  return alpha ? k_render_bwd<TS, true, false, false, DET> : k_render_bwd<TS, false, false, false, DET>;
}

template <int TS>
cudaError_t launch_bwd_ts(bool alpha, RenderArgs ra, cudaStream_t s) {
  ra.queue = Q_BWD;
  const int64_t items = ra.BT * Geo<TS>::S * (alpha ? 1 : ra.chunks);
  void (*k)(RenderArgs);
  if (ra.slots)
    k = pick_bwd<TS, true>(alpha, ra.mom_beta != nullptr, ra.f64 != 0);
  else
    k = pick_bwd<TS, false>(alpha, ra.mom_beta != nullptr, ra.f64 != 0);
  launch_begin(K_RENDER_BWD, s);
  k<<<persistent_grid(k, items), kCta, 0, s>>>(ra);
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
  ra.chunks = WIPES_BWD_CHUNKS > 0 ? WIPES_BWD_CHUNKS : (L.BT >= 16384 ? 2 : 4);
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
  ra.mom_beta = L.exact ? (float*)(ws + L.rbeta) : nullptr;
  ra.prevals = L.det ? (const uint32_t*)(ws + L.prevals) : nullptr;
  ra.slots = L.det ? (float*)(ws + L.slots) : nullptr;
  ra.slotmask = L.det ? (uint8_t*)(ws + L.slotmask) : nullptr;
  ra.fps = L.fps;
  ra.slotw = L.slotw;
  ra.stats = nullptr;
  ra.f64 = c.grad_accum == WIPES_ACCUM_F64;
#ifdef WIPES_FORCE_ACCUM  // A/B experiments only: 1 = FP32, 2 = FP64 everywhere
  ra.f64 = WIPES_FORCE_ACCUM == 2;
#endif
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

#ifdef WIPES_BWD_COUNT
extern "C" void wipes_debug_bwd_counters(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_bwd_cnt, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_bwd_cnt, z, sizeof(z));
  }
}
#endif

}  // namespace wipes
