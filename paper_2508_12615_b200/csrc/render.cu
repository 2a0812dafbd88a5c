// Per-tile render kernels, FP32 + SFU (MUFU) pipes.
//
//  forward  : PAPER.md:172 (Eq. 4, weighted sum) / PAPER.md:125 (Eq. 3, alpha
//             blending), with the Gaussian G' replaced by the wavelet W'
//             (PAPER.md:215, :272): w = alpha * G * 1/2 [1 + beta cos(f.d + phi)].
//  backward : analytic per-pair gradients ("explicit gradients for all
//             parameters"), reduced per warp with a 16-value
//             transpose-reduce of shuffles, then one atomic per (warp, record,
//             value) into the record-gradient buffer.
//
// One CTA per (view, tile); TS x TS threads, one pixel each. Warps own 8 x 4
// pixel sub-tiles; every staged record carries a sub-tile mask computed from
// its opacity extent (conservative), so a warp skips records that cannot
// reach its pixels (warp-uniform branch). Records are staged in shared memory
// in batches of up to 256 (one coalesced 64-byte record per loading thread).
// The exp is a single MUFU.EX2 (the -1/2 log2(e) scale and log2(alpha) are
// folded into the record); cos / sin are MUFU.COS / MUFU.SIN.
#include <cuda_fp16.h>

#include "common.cuh"

namespace wipes {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr float kLn2 = 0.6931471805599453f;
// unscaled conic = scaled / (-1/2 log2 e)
constexpr float kInvHalfLog2e = -1.3862943611198906f;  // = -2 ln 2

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
  int64_t N, T;
  int32_t W, H, GX;
  float alpha_min, skip_e, alpha_max, T_min;
  float bg0, bg1, bg2;
  float* image;          // [B,3,H,W]
  float* T_final;        // [B,H,W]
  int32_t* n_contrib;    // [B,H,W]
  const float* dLdC;     // [B,3,H,W]
  const float* T_in;
  const int32_t* nc_in;
  float* rgrad;          // [B*N, 13]
  unsigned long long* stats;  // STATS build: {tile-method candidates, in-ellipse, contributing}
};

// Sub-tile mask of a record for tile origin (X0, Y0): bit (sy * NSX + sx) set
// when the record's opacity-extent AABB (padded) may touch the 8x4 sub-tile.
template <int TS>
__device__ __forceinline__ uint32_t subtile_mask(const float4& r0, const float4& r3, int X0,
                                                 int Y0) {
  constexpr int NSX = TS / 8, NSY = TS / 4;
  __half2 e2 = *reinterpret_cast<const __half2*>(&r3.w);
  float rx = __low2float(e2) + 0.02f, ry = __high2float(e2) + 0.02f;
  float cx = (r3.y - (float)X0) + r0.x;  // centre relative to the tile origin
  float cy = (r3.z - (float)Y0) + r0.y;
  // sub-tile sx covers pixel centres [8 sx + 0.5, 8 sx + 7.5]
  float fx0 = ceilf((cx - rx - 7.5f) * 0.125f), fx1 = floorf((cx + rx - 0.5f) * 0.125f);
  float fy0 = ceilf((cy - ry - 3.5f) * 0.25f), fy1 = floorf((cy + ry - 0.5f) * 0.25f);
  int sx0 = (int)fmaxf(fx0, 0.f), sx1 = (int)fminf(fx1, (float)(NSX - 1));
  int sy0 = (int)fmaxf(fy0, 0.f), sy1 = (int)fminf(fy1, (float)(NSY - 1));
  if (!(fx0 <= fx1) || !(fy0 <= fy1) || sx0 > sx1 || sy0 > sy1) return 0u;
  uint32_t row = ((2u << sx1) - 1u) & ~((1u << sx0) - 1u);
  uint32_t m = 0;
#pragma unroll
  for (int sy = 0; sy < NSY; ++sy)
    if (sy >= sy0 && sy <= sy1) m |= row << (sy * NSX);
  return m;
}

// Shared exp/cos evaluation of one (pixel, record) pair, identical in forward
// and backward so both take the same alpha_min decisions.
struct PairEval {
  float dx, dy, ag, th, w;
  bool ok;
};

__device__ __forceinline__ void eval_pair(const float4& r0, const float4& r1, const float4& r2,
                                          const float4& r3, float px, float py, float skip_e,
                                          float alpha_min, PairEval& e, float& cs) {
  e.dx = __fsub_rn(__fsub_rn(px, r3.y), r0.x);
  e.dy = __fsub_rn(__fsub_rn(py, r3.z), r0.y);
  float t = __fmaf_rn(r0.z, e.dx, __fmul_rn(r0.w, e.dy));
  float u = __fmaf_rn(__fmul_rn(r1.x, e.dy), e.dy, r1.y);
  float ex = __fmaf_rn(t, e.dx, u);
  e.ok = ex >= skip_e;
  if (!e.ok) return;
  e.ag = ex2(ex);
  e.th = __fmaf_rn(r1.z, e.dx, __fmaf_rn(r1.w, e.dy, r2.x));
  cs = cos_a(e.th);
  e.w = __fmul_rn(e.ag, __fmaf_rn(r2.y, cs, 0.5f));
  e.ok = e.w >= alpha_min;
}

constexpr int kBatch = 256;

template <int TS, bool ALPHA, bool STATS>
__global__ void __launch_bounds__(TS* TS) k_render_fwd(RenderArgs a) {
  constexpr int NT = TS * TS;
  constexpr int NB = NT < kBatch ? NT : kBatch;
  constexpr int NSX = TS / 8;
  __shared__ float4 s_rec[NB][4];
  __shared__ uint32_t s_mask[NB];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t v = tile / a.T;
  const int64_t t_in_v = tile - v * a.T;
  const int ty = (int)(t_in_v / a.GX), tx = (int)(t_in_v - (int64_t)ty * a.GX);
  const int X0 = tx * TS, Y0 = ty * TS;
  const int sx = wid % NSX, sy = wid / NSX;
  const int x = X0 + sx * 8 + (lane & 7), y = Y0 + sy * 4 + (lane >> 3);
  const bool inside = x < a.W && y < a.H;
  const float px = (float)x + 0.5f, py = (float)y + 0.5f;
  const int start = a.toff[tile], end = a.toff[tile + 1];
  const float4* recv = a.rec + 4 * (v * a.N);
  float C0 = 0.f, C1 = 0.f, C2 = 0.f, T = 1.f;
  int last = 0;
  bool done = ALPHA ? !inside : false;
  bool warp_done = ALPHA ? __all_sync(kFull, done) : false;
  const uint32_t mybit = 1u << wid;
  int n_ell = 0, n_con = 0, stop_pos = end - start;  // STATS only
  for (int b0 = start; b0 < end; b0 += NB) {
    const int nb = min(NB, end - b0);
    __syncthreads();
    if (tid < nb) {
      const uint32_t pid = a.vals[b0 + tid];
      const float4* r = recv + 4 * (int64_t)pid;
      float4 r0 = __ldg(r), r1 = __ldg(r + 1), r2 = __ldg(r + 2), r3 = __ldg(r + 3);
      s_rec[tid][0] = r0; s_rec[tid][1] = r1; s_rec[tid][2] = r2; s_rec[tid][3] = r3;
      s_mask[tid] = subtile_mask<TS>(r0, r3, X0, Y0);
    }
    __syncthreads();
    if (!warp_done) {
      for (int j = 0; j < nb; ++j) {
        if (!(s_mask[j] & mybit)) continue;  // warp-uniform
        if (!done) {
          const float4 r0 = s_rec[j][0], r1 = s_rec[j][1], r2 = s_rec[j][2], r3 = s_rec[j][3];
          PairEval e;
          float cs;
          eval_pair(r0, r1, r2, r3, px, py, a.skip_e, a.alpha_min, e, cs);
          if (STATS && inside) {
            const float4 q0 = r0, q1 = r1;
            float t = __fmaf_rn(q0.z, e.dx, __fmul_rn(q0.w, e.dy));
            float u = __fmaf_rn(__fmul_rn(q1.x, e.dy), e.dy, q1.y);
            if (__fmaf_rn(t, e.dx, u) >= a.skip_e) ++n_ell;
          }
          if (e.ok) {
            if (!ALPHA) {
              if (STATS && inside) ++n_con;
              C0 = __fmaf_rn(r2.z, e.w, C0);
              C1 = __fmaf_rn(r2.w, e.w, C1);
              C2 = __fmaf_rn(r3.x, e.w, C2);
            } else {
              const float al = fminf(a.alpha_max, e.w);
              const float Tn = __fmul_rn(T, __fsub_rn(1.f, al));
              if (Tn < a.T_min) {
                done = true;
                if (STATS) stop_pos = b0 + j - start + 1;
              } else {
                if (STATS) ++n_con;
                const float aT = __fmul_rn(al, T);
                C0 = __fmaf_rn(r2.z, aT, C0);
                C1 = __fmaf_rn(r2.w, aT, C1);
                C2 = __fmaf_rn(r3.x, aT, C2);
                T = Tn;
                last = b0 + j - start + 1;
              }
            }
          }
        }
        if (ALPHA && __all_sync(kFull, done)) { warp_done = true; break; }
      }
    }
    if (ALPHA) {
      if (__syncthreads_count(!done) == 0) break;
    }
  }
  if (STATS) {
    unsigned long long c3[3] = {inside ? (unsigned long long)stop_pos : 0ull,
                                (unsigned long long)n_ell, (unsigned long long)n_con};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      unsigned long long v = c3[k];
#pragma unroll
      for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
      if (lane == 0) atomicAdd(a.stats + k, v);
    }
    return;
  }
  if (!inside) return;
  const int64_t HW = (int64_t)a.H * a.W;
  const int64_t pix = (int64_t)y * a.W + x;
  if (ALPHA) {
    C0 = __fmaf_rn(T, a.bg0, C0);
    C1 = __fmaf_rn(T, a.bg1, C1);
    C2 = __fmaf_rn(T, a.bg2, C2);
    a.T_final[v * HW + pix] = T;
    a.n_contrib[v * HW + pix] = last;
  }
  float* img = a.image + v * 3 * HW + pix;
  img[0] = C0;
  img[HW] = C1;
  img[2 * HW] = C2;
}

// 16-value warp transpose-reduce: returns, in every lane L, the warp-wide sum
// of value index (L >> 1) & 15.
__device__ __forceinline__ float transpose_reduce16(float (&v)[16], int lane) {
  {
    const bool up = lane & 16;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float send = up ? v[k] : v[k + 8];
      float keep = up ? v[k + 8] : v[k];
      v[k] = keep + __shfl_xor_sync(kFull, send, 16);
    }
  }
  {
    const bool up = lane & 8;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float send = up ? v[k] : v[k + 4];
      float keep = up ? v[k + 4] : v[k];
      v[k] = keep + __shfl_xor_sync(kFull, send, 8);
    }
  }
  {
    const bool up = lane & 4;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      float send = up ? v[k] : v[k + 2];
      float keep = up ? v[k + 2] : v[k];
      v[k] = keep + __shfl_xor_sync(kFull, send, 4);
    }
  }
  {
    const bool up = lane & 2;
    float send = up ? v[0] : v[1];
    float keep = up ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(kFull, send, 2);
  }
  return v[0] + __shfl_xor_sync(kFull, v[0], 1);
}

template <int TS, bool ALPHA>
__global__ void __launch_bounds__(TS* TS) k_render_bwd(RenderArgs a) {
  constexpr int NT = TS * TS;
  constexpr int NB = NT < kBatch ? NT : kBatch;
  constexpr int NSX = TS / 8;
  __shared__ float4 s_rec[NB][4];
  __shared__ float4 s_aux[NB];  // unscaled conic (a, b, c), 1/alpha
  __shared__ uint32_t s_mask[NB];
  __shared__ int32_t s_rid[NB];
  __shared__ int32_t s_maxlast;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t v = tile / a.T;
  const int64_t t_in_v = tile - v * a.T;
  const int ty = (int)(t_in_v / a.GX), tx = (int)(t_in_v - (int64_t)ty * a.GX);
  const int X0 = tx * TS, Y0 = ty * TS;
  const int sx = wid % NSX, sy = wid / NSX;
  const int x = X0 + sx * 8 + (lane & 7), y = Y0 + sy * 4 + (lane >> 3);
  const bool inside = x < a.W && y < a.H;
  const float px = (float)x + 0.5f, py = (float)y + 0.5f;
  const int start = a.toff[tile];
  int end = a.toff[tile + 1];
  const int64_t HW = (int64_t)a.H * a.W;
  const int64_t pix = v * HW + (int64_t)y * a.W + x;
  float g0 = 0.f, g1 = 0.f, g2 = 0.f;
  float T = 1.f, S0 = 0.f, S1 = 0.f, S2 = 0.f;
  int last = 0;
  if (inside) {
    const float* gp = a.dLdC + v * 3 * HW + (int64_t)y * a.W + x;
    g0 = gp[0]; g1 = gp[HW]; g2 = gp[2 * HW];
    if (ALPHA) {
      T = a.T_in[pix];
      last = a.nc_in[pix];
      S0 = T * a.bg0; S1 = T * a.bg1; S2 = T * a.bg2;
    }
  }
  if (ALPHA) {
    if (tid == 0) s_maxlast = 0;
    __syncthreads();
    if (last > 0) atomicMax(&s_maxlast, last);
    __syncthreads();
    end = start + s_maxlast;
  }
  const uint32_t mybit = 1u << wid;
  const int64_t vN = v * a.N;
  const float4* recv = a.rec + 4 * vN;
  const int nbatch = (end - start + NB - 1) / NB;
  for (int bi = 0; bi < nbatch; ++bi) {
    // ALPHA walks batches back to front; SUM front to back (order-free).
    const int b0 = ALPHA ? max(start, end - (bi + 1) * NB) : start + bi * NB;
    const int nb = ALPHA ? (end - bi * NB) - b0 : min(NB, end - b0);
    __syncthreads();
    if (tid < nb) {
      const uint32_t pid = a.vals[b0 + tid];
      const float4* r = recv + 4 * (int64_t)pid;
      float4 r0 = __ldg(r), r1 = __ldg(r + 1), r2 = __ldg(r + 2), r3 = __ldg(r + 3);
      s_rec[tid][0] = r0; s_rec[tid][1] = r1; s_rec[tid][2] = r2; s_rec[tid][3] = r3;
      s_aux[tid] = make_float4(r0.z * kInvHalfLog2e, r0.w * (0.5f * kInvHalfLog2e),
                               r1.x * kInvHalfLog2e, ex2(-r1.y));
      s_mask[tid] = subtile_mask<TS>(r0, r3, X0, Y0);
      s_rid[tid] = (int32_t)pid;
    }
    __syncthreads();
    for (int jj = 0; jj < nb; ++jj) {
      const int j = ALPHA ? nb - 1 - jj : jj;
      if (!(s_mask[j] & mybit)) continue;  // warp-uniform
      const int pos = b0 + j - start;      // index within the tile list
      const float4 r0 = s_rec[j][0], r1 = s_rec[j][1], r2 = s_rec[j][2], r3 = s_rec[j][3];
      PairEval e;
      float cs = 0.f;
      bool valid = inside && (!ALPHA || pos < last);
      if (valid) {
        eval_pair(r0, r1, r2, r3, px, py, a.skip_e, a.alpha_min, e, cs);
        valid = e.ok;
      }
      if (!__any_sync(kFull, valid)) continue;
      float vals[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) vals[k] = 0.f;
      if (valid) {
        const float4 aux = s_aux[j];
        const float sn = sin_a(e.th);
        const float gdc = __fmaf_rn(r2.z, g0, __fmaf_rn(r2.w, g1, __fmul_rn(r3.x, g2)));
        float gw;
        if (!ALPHA) {
          gw = gdc;
          vals[RG_CR] = e.w * g0;
          vals[RG_CG] = e.w * g1;
          vals[RG_CB] = e.w * g2;
        } else {
          const float al = fminf(a.alpha_max, e.w);
          const float ri = rcp_a(1.f - al);
          const float Tk = T * ri;
          const float sdg = __fmaf_rn(S0, g0, __fmaf_rn(S1, g1, __fmul_rn(S2, g2)));
          const float dLda = __fmaf_rn(Tk, gdc, -sdg * ri);
          const float aT = al * Tk;
          vals[RG_CR] = aT * g0;
          vals[RG_CG] = aT * g1;
          vals[RG_CB] = aT * g2;
          S0 = __fmaf_rn(r2.z, aT, S0);
          S1 = __fmaf_rn(r2.w, aT, S1);
          S2 = __fmaf_rn(r3.x, aT, S2);
          T = Tk;
          gw = (e.w < a.alpha_max) ? dLda : 0.f;
        }
        const float s = -r2.y * e.ag * sn;    // dw/dtheta
        const float gs = gw * s;
        const float gww = gw * e.w;
        vals[RG_FX] = gs * e.dx;
        vals[RG_FY] = gs * e.dy;
        vals[RG_PHI] = gs;
        vals[RG_MUX] = __fmaf_rn(gww, __fmaf_rn(aux.x, e.dx, aux.y * e.dy), -gs * r1.z);
        vals[RG_MUY] = __fmaf_rn(gww, __fmaf_rn(aux.y, e.dx, aux.z * e.dy), -gs * r1.w);
        const float hg = -0.5f * gww;
        vals[RG_A] = hg * e.dx * e.dx;
        vals[RG_B] = -gww * e.dx * e.dy;
        vals[RG_C] = hg * e.dy * e.dy;
        vals[RG_BETA] = gw * 0.5f * e.ag * cs;
        vals[RG_ALPHA] = gww * aux.w;
      }
      const float red = transpose_reduce16(vals, lane);
      const int k = lane >> 1;
      if (!(lane & 1) && k < kRecGrads)
        atomicAdd(a.rgrad + (vN + s_rid[j]) * kRecGrads + k, red);
    }
  }
}

template <int TS>
cudaError_t launch_fwd_ts(bool alpha, const RenderArgs& ra, unsigned grid, cudaStream_t s) {
  if (ra.stats) {
    if (alpha) k_render_fwd<TS, true, true><<<grid, TS * TS, 0, s>>>(ra);
    else k_render_fwd<TS, false, true><<<grid, TS * TS, 0, s>>>(ra);
    return cudaGetLastError();
  }
  launch_begin(K_RENDER_FWD, s);
  if (alpha) k_render_fwd<TS, true, false><<<grid, TS * TS, 0, s>>>(ra);
  else k_render_fwd<TS, false, false><<<grid, TS * TS, 0, s>>>(ra);
  launch_end(K_RENDER_FWD, s);
  return cudaGetLastError();
}

template <int TS>
cudaError_t launch_bwd_ts(bool alpha, const RenderArgs& ra, unsigned grid, cudaStream_t s) {
  launch_begin(K_RENDER_BWD, s);
  if (alpha) k_render_bwd<TS, true><<<grid, TS * TS, 0, s>>>(ra);
  else k_render_bwd<TS, false><<<grid, TS * TS, 0, s>>>(ra);
  launch_end(K_RENDER_BWD, s);
  return cudaGetLastError();
}

RenderArgs make_args(const wipes_config& c, const Layout& L, char* ws, int final_in_b) {
  RenderArgs ra;
  ra.rec = (const float4*)(ws + L.rec);
  ra.vals = (const uint32_t*)(ws + (final_in_b ? L.valsB : L.valsA));
  ra.toff = (const int32_t*)(ws + L.toff);
  ra.N = L.N;
  ra.T = L.T;
  ra.W = c.width; ra.H = c.height; ra.GX = L.GX;
  ra.alpha_min = c.alpha_min;
  // conservative early-out on the exponent: e < log2(alpha_min) - 1e-4 implies
  // alpha*W < alpha_min after the MUFU roundings
  ra.skip_e = c.alpha_min > 0.f ? (float)(log2((double)c.alpha_min) - 1e-4) : -INFINITY;
  ra.alpha_max = c.alpha_max;
  ra.T_min = c.T_min;
  ra.bg0 = c.background[0]; ra.bg1 = c.background[1]; ra.bg2 = c.background[2];
  ra.image = nullptr; ra.T_final = nullptr; ra.n_contrib = nullptr;
  ra.dLdC = nullptr; ra.T_in = nullptr; ra.nc_in = nullptr;
  ra.rgrad = (float*)(ws + L.rgrad);
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
  const unsigned grid = (unsigned)L.BT;
  switch (c.tile) {
    case 8: return launch_fwd_ts<8>(alpha, ra, grid, s);
    case 16: return launch_fwd_ts<16>(alpha, ra, grid, s);
    default: return launch_fwd_ts<32>(alpha, ra, grid, s);
  }
}

cudaError_t launch_render_bwd(const wipes_config& c, const Layout& L, char* ws, int final_in_b,
                              const float* dLdC, const float* T_final,
                              const int32_t* n_contrib, cudaStream_t s) {
  if (L.BT == 0) return cudaSuccess;
  RenderArgs ra = make_args(c, L, ws, final_in_b);
  ra.dLdC = dLdC; ra.T_in = T_final; ra.nc_in = n_contrib;
  const bool alpha = c.blend == WIPES_BLEND_ALPHA;
  const unsigned grid = (unsigned)L.BT;
  switch (c.tile) {
    case 8: return launch_bwd_ts<8>(alpha, ra, grid, s);
    case 16: return launch_bwd_ts<16>(alpha, ra, grid, s);
    default: return launch_bwd_ts<32>(alpha, ra, grid, s);
  }
}

}  // namespace wipes
