// NEXT-4: the time-conditioned deformation field of PAPER.md Eq. 8,
// the D-3DGS network of Eq. 5, on the tcgen05 GEMM of gemm.cu
// (include/wipes.h "NEXT-4"; R34-R36).
//
// Forward (rows m = f*N + i): k_mlp_embed writes the positional encoding
// [gamma(x_i), gamma(t_f)] (bf16, zero-padded to E8) into the first E8 columns
// of the concat buffer `cat` [M, E8 + W]; layer l is one GEMM with a fused
// bias + ReLU + bf16 epilogue (layer `skip` writes its output into cat's last
// W columns, so the skip layer reads [gamma, h] as one K = E8 + W operand);
// the head GEMM adds its bias in fp32; k_mlp_apply forms the frame rows.
// Backward: k_mlp_dout builds dL/dout (13 columns, bf16 for the GEMMs, fp32
// for the head bias); per layer one split-K GEMM dW = dZ^T In (both operands
// MN-major straight from the row-major activations, atomic fp32 epilogue) and
// one GEMM dIn = dZ W (W read MN-major) whose epilogue applies the ReLU mask
// of the layer below and sums the result over the rows (that layer's bias
// gradient).
#include <cuda_bf16.h>

#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace wipes {

namespace {

constexpr int kMlpMaxDepth = 32;
constexpr int kMlpMaxFrames = 128;
constexpr int kOutCols = 16;  // 13 outputs padded to one MMA N step
constexpr int kMaxE8 = 3 * (1 + 2 * 16) + (1 + 2 * 16) + 8;  // Lx, Lt <= 16

struct MlpLayout {
  int W, D, skip, Lx, Lt, E, E8, catw;
  bool x3;     // split-bf16 operands (WIPES_MLP_BF16X3, R38)
  int R;       // 3 with x3 (every activation buffer holds [hi | hi | lo]), else 1
  size_t wb3[kMlpMaxDepth], whb3;  // x3: backward weights [W_hi; W_lo; W_hi] (3 rows blocks)
  int64_t M;
  int K[kMlpMaxDepth], Kp[kMlpMaxDepth];
  int64_t thW[kMlpMaxDepth], thb[kMlpMaxDepth], thWh, thbh, P;
  size_t wbf[kMlpMaxDepth], whbf, cat, h[kMlpMaxDepth], out, dout_bf, dout_f, dz[2], dws, total;
  size_t wpart, bpart;  // fused layer backward partials (width 256 only)
};

bool mlp_cfg_ok(const wipes_mlp_config& c) {
  return (c.precision == WIPES_MLP_BF16X3 || c.precision == WIPES_MLP_BF16) && c.width >= 16 && c.width <= 256 && c.width % 16 == 0 && c.depth >= 1 &&
         c.depth <= kMlpMaxDepth && c.skip >= -1 && c.skip <= c.depth - 2 && c.Lx >= 0 &&
         c.Lx <= 16 && c.Lt >= 0 && c.Lt <= 16;
}

MlpLayout mlp_layout(const wipes_mlp_config& c, int64_t M) {
  MlpLayout L;
  L.W = c.width; L.D = c.depth; L.skip = c.skip; L.Lx = c.Lx; L.Lt = c.Lt;
  L.E = 3 * (1 + 2 * c.Lx) + (1 + 2 * c.Lt);
  L.E8 = (L.E + 7) / 8 * 8;
  L.x3 = c.precision == WIPES_MLP_BF16X3;
  L.R = L.x3 ? 3 : 1;
  // x3: cat = [e_hi | e_hi | e_lo | h_hi | h_hi | h_lo] (layer 0 reads the first
  // 3 E8 columns, the layer after the skip all of them)
  L.catw = L.R * (L.E8 + L.W);
  L.M = M;
  int64_t o = 0;
  for (int l = 0; l < L.D; ++l) {
    L.K[l] = l == 0 ? L.E : (l == L.skip + 1 ? L.E + L.W : L.W);
    L.Kp[l] = l == 0 ? L.E8 : (l == L.skip + 1 ? L.E8 + L.W : L.W);
    L.thW[l] = o; o += (int64_t)L.W * L.K[l];
    L.thb[l] = o; o += L.W;
  }
  L.thWh = o; o += 13 * (int64_t)L.W;
  L.thbh = o; o += 13;
  L.P = o;
  size_t b = 0;
  auto take = [&](size_t bytes) { size_t r = b; b = align_up(b + bytes, 256); return r; };
  int kmax = 0;
  const size_t R = (size_t)L.R;
  for (int l = 0; l < L.D; ++l) {
    L.wbf[l] = take(2 * R * (size_t)L.W * L.Kp[l]);
    L.wb3[l] = L.x3 ? take(2 * R * (size_t)L.W * L.Kp[l]) : 0;
    kmax = L.Kp[l] > kmax ? L.Kp[l] : kmax;
  }
  L.whbf = take(2 * R * (size_t)kOutCols * L.W);
  L.whb3 = L.x3 ? take(2 * R * (size_t)kOutCols * L.W) : 0;
  L.cat = take(2 * (size_t)M * L.catw);
  for (int l = 0; l < L.D; ++l) L.h[l] = l == L.skip ? 0 : take(2 * R * (size_t)M * L.W);
  L.out = take(4 * (size_t)M * kOutCols);
  L.dout_bf = take(2 * R * (size_t)M * kOutCols);
  L.dout_f = take(4 * (size_t)M * kOutCols);
  L.dz[0] = take(2 * R * (size_t)M * L.W);
  L.dz[1] = take(2 * R * (size_t)M * L.W);
  L.dws = take(4 * (size_t)L.W * kmax);
  L.wpart = L.bpart = 0;
  if (L.W == 256 && !L.x3) {
    L.wpart = take(4 * (size_t)kMlpBwdMaxGroups * 256 * 256);
    L.bpart = take(4 * (size_t)kMlpBwdMaxGroups * 4 * 256);
  }
  L.total = b;
  return L;
}

// theta (fp32, true widths) -> padded bf16 weights of every layer and the head.
// All layers and the head in one launch (blockIdx.y = layer).
struct WeightJobs {
  int n;
  struct Job { int64_t thW; int rows, rows_valid, Kp, K; bool has_cat; __nv_bfloat16* dst; } j[kMlpMaxDepth + 1];
};
__global__ void k_mlp_weights_all(const float* theta, int E, int E8, const __grid_constant__ WeightJobs w) {
  const WeightJobs::Job& jb = w.j[blockIdx.y];
  const int64_t n = (int64_t)jb.rows * jb.Kp;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx / jb.Kp), c = (int)(idx - (int64_t)j * jb.Kp);
    float v = 0.f;
    if (j < jb.rows_valid) {
      int src = -1;
      if (!jb.has_cat) src = c < jb.K ? c : -1;
      else src = c < E ? c : (c < E8 ? -1 : c - E8 + E);
      if (src >= 0) v = theta[jb.thW + (int64_t)j * jb.K + src];
    }
    jb.dst[idx] = __float2bfloat16_rn(v);
  }
}

// x3 (split-bf16, R38): weight w -> hi = bf16(w), lo = bf16(w - hi).
// Forward layout [rows, 3 Kp]: per input segment (the encoding and, after the
// skip, the hidden part) three blocks [hi | lo | hi] against activations
// [hi | hi | lo]; backward layout [3 rows, Kp] = [W_hi; W_lo; W_hi] (the dL/dIn
// GEMM reduces over the output rows against dL/dz = [hi | hi | lo]).
struct WeightJobsX3 {
  int n;
  struct Job {
    int64_t thW;
    int rows, rows_valid, Kp, K;
    bool has_cat;
    __nv_bfloat16 *dst, *dstb;
  } j[kMlpMaxDepth + 1];
};
__device__ __forceinline__ float mlp_wsrc(const float* theta, const WeightJobsX3::Job& jb, int E,
                                          int E8, int j, int c) {
  if (j >= jb.rows_valid) return 0.f;
  int src;
  if (!jb.has_cat) src = c < jb.K ? c : -1;
  else src = c < E ? c : (c < E8 ? -1 : c - E8 + E);
  return src >= 0 ? theta[jb.thW + (int64_t)j * jb.K + src] : 0.f;
}
__device__ __forceinline__ __nv_bfloat16 split_part(float v, int b) {
  const __nv_bfloat16 hi = __float2bfloat16_rn(v);
  return b == 1 ? __float2bfloat16_rn(v - __bfloat162float(hi)) : hi;
}
__global__ void k_mlp_weights_x3(const float* theta, int E, int E8,
                                 const __grid_constant__ WeightJobsX3 w) {
  const WeightJobsX3::Job& jb = w.j[blockIdx.y];
  const int Kp3 = 3 * jb.Kp;
  const int64_t n = (int64_t)jb.rows * Kp3;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    // forward layout: row j, column cc of [rows, 3 Kp]
    {
      const int j = (int)(idx / Kp3), cc = (int)(idx - (int64_t)j * Kp3);
      int b, c;
      if (!jb.has_cat) {
        b = cc / jb.Kp; c = cc - b * jb.Kp;
      } else if (cc < 3 * E8) {
        b = cc / E8; c = cc - b * E8;
      } else {
        const int r = cc - 3 * E8, Wd = jb.Kp - E8;
        b = r / Wd; c = E8 + (r - b * Wd);
      }
      jb.dst[idx] = split_part(mlp_wsrc(theta, jb, E, E8, j, c), b);
    }
    // backward layout: row rr of [3 rows, Kp], column c
    {
      const int rr = (int)(idx / jb.Kp), c = (int)(idx - (int64_t)rr * jb.Kp);
      const int b = rr / jb.rows, j = rr - b * jb.rows;
      jb.dstb[idx] = split_part(mlp_wsrc(theta, jb, E, E8, j, c), b);
    }
  }
}

struct EmbedArgs {
  const float* mean;
  int64_t N, row0, rows;
  int32_t f0, Lx, Lt, E8, catw;
  int32_t x3;  // write [hi | hi | lo] blocks of E8 columns (the encoding's lo part)
  float t[kMlpMaxFrames];
  __nv_bfloat16* cat;
};

// LX, LT > 0: compile-time frequency counts (the encoding stays in registers);
// 0: the runtime values in a (local-memory buffer).
template <int LX, int LT>
__global__ void __launch_bounds__(128) k_mlp_embed(const __grid_constant__ EmbedArgs a) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.rows) return;
  const int lx = LX > 0 ? LX : a.Lx, lt = LX > 0 ? LT : a.Lt;
  const int64_t m = a.row0 + r;
  const int64_t f = m / a.N, i = m - f * a.N;
  const float x[3] = {a.mean[3 * i], a.mean[3 * i + 1], a.mean[3 * i + 2]};
  const float t = a.t[f - a.f0];
  // built in registers, written as 16-byte vectors (E8 is a multiple of 8)
  constexpr int kE8 = LX > 0 ? (3 * (1 + 2 * LX) + (1 + 2 * LT) + 7) / 8 * 8 : kMaxE8;
  __align__(16) __nv_bfloat16 buf[kE8];
  int c = 0;
#pragma unroll
  for (int d = 0; d < 3; ++d) buf[c++] = __float2bfloat16_rn(x[d]);
#pragma unroll
  for (int k = 0; k < (LX > 0 ? LX : 16); ++k) {
    if (LX == 0 && k >= lx) break;
    const float sc = (float)(1 << k);
    float sn[3], cs[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) sincosf(sc * x[d], &sn[d], &cs[d]);
#pragma unroll
    for (int d = 0; d < 3; ++d) buf[c++] = __float2bfloat16_rn(sn[d]);
#pragma unroll
    for (int d = 0; d < 3; ++d) buf[c++] = __float2bfloat16_rn(cs[d]);
  }
  buf[c++] = __float2bfloat16_rn(t);
#pragma unroll
  for (int k = 0; k < (LX > 0 ? LT : 16); ++k) {
    if (LX == 0 && k >= lt) break;
    float sn, cs;
    sincosf((float)(1 << k) * t, &sn, &cs);
    buf[c++] = __float2bfloat16_rn(sn);
    buf[c++] = __float2bfloat16_rn(cs);
  }
  const int e8 = LX > 0 ? kE8 : a.E8;
#pragma unroll
  for (int q = 0; q < kE8; ++q)
    if (q >= c && q < e8) buf[q] = __float2bfloat16_rn(0.f);
  uint4* row = reinterpret_cast<uint4*>(a.cat + m * a.catw);
  const uint4* src = reinterpret_cast<const uint4*>(buf);
#pragma unroll
  for (int v = 0; v < kE8 / 8; ++v)
    if (v < e8 / 8) row[v] = src[v];
  if (a.x3) {  // second hi block, then lo = bf16(value - hi) recomputed in fp32
    uint4* row2 = reinterpret_cast<uint4*>(a.cat + m * a.catw + e8);
#pragma unroll
    for (int v = 0; v < kE8 / 8; ++v)
      if (v < e8 / 8) row2[v] = src[v];
    c = 0;
    for (int d = 0; d < 3; ++d) { buf[c] = __float2bfloat16_rn(x[d] - __bfloat162float(buf[c])); ++c; }
    for (int k = 0; k < lx; ++k) {
      const float sc = (float)(1 << k);
      float sn[3], cs[3];
      for (int d = 0; d < 3; ++d) sincosf(sc * x[d], &sn[d], &cs[d]);
      for (int d = 0; d < 3; ++d) { buf[c] = __float2bfloat16_rn(sn[d] - __bfloat162float(buf[c])); ++c; }
      for (int d = 0; d < 3; ++d) { buf[c] = __float2bfloat16_rn(cs[d] - __bfloat162float(buf[c])); ++c; }
    }
    buf[c] = __float2bfloat16_rn(t - __bfloat162float(buf[c]));
    ++c;
    for (int k = 0; k < lt; ++k) {
      float sn, cs;
      sincosf((float)(1 << k) * t, &sn, &cs);
      buf[c] = __float2bfloat16_rn(sn - __bfloat162float(buf[c])); ++c;
      buf[c] = __float2bfloat16_rn(cs - __bfloat162float(buf[c])); ++c;
    }
    uint4* row3 = reinterpret_cast<uint4*>(a.cat + m * a.catw + 2 * e8);
#pragma unroll
    for (int v = 0; v < kE8 / 8; ++v)
      if (v < e8 / 8) row3[v] = src[v];
  }
}

struct ApplyArgs {
  int64_t N, M;
  const float* out;  // [M, 16]
  wipes_params canon, frame;
  int32_t sh_coeffs;
};

__global__ void __launch_bounds__(128) k_mlp_apply(const __grid_constant__ ApplyArgs a) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= a.M) return;
  const int64_t i = m % a.N;
  const float* o = a.out + m * kOutCols;
  float* fm = const_cast<float*>(a.frame.mean);
  float* fq = const_cast<float*>(a.frame.quat);
  float* fs = const_cast<float*>(a.frame.scale);
  float* ff = const_cast<float*>(a.frame.freq);
  for (int d = 0; d < 3; ++d) fm[3 * m + d] = a.canon.mean[3 * i + d] + o[d];
  for (int d = 0; d < 4; ++d) fq[4 * m + d] = a.canon.quat[4 * i + d] + o[3 + d];
  for (int d = 0; d < 3; ++d) fs[3 * m + d] = a.canon.scale[3 * i + d] * expf(o[7 + d]);
  for (int d = 0; d < 3; ++d) ff[3 * m + d] = a.canon.freq[3 * i + d] + o[10 + d];
  if (a.canon.phase && a.frame.phase) const_cast<float*>(a.frame.phase)[m] = a.canon.phase[i];
  if (a.canon.opacity && a.frame.opacity)
    const_cast<float*>(a.frame.opacity)[m] = a.canon.opacity[i];
  if (a.canon.color && a.frame.color)
    for (int d = 0; d < 3; ++d) const_cast<float*>(a.frame.color)[3 * m + d] = a.canon.color[3 * i + d];
  if (a.canon.sh && a.frame.sh)
    for (int d = 0; d < 3 * a.sh_coeffs; ++d)
      const_cast<float*>(a.frame.sh)[3 * a.sh_coeffs * m + d] = a.canon.sh[3 * a.sh_coeffs * i + d];
}

// dL/dout = (g_mu_t, g_q_t, g_s_t * s_t, g_f_t) (s_t = s exp(ds)), bf16 + fp32.
__global__ void __launch_bounds__(128) k_mlp_dout(int64_t N, int64_t M, const float* out,
                                                  const float* scale, wipes_grads g,
                                                  __nv_bfloat16* dbf, float* df, int x3) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  const int64_t i = m % N;
  float v[kOutCols];
  for (int d = 0; d < 3; ++d) v[d] = g.mean[3 * m + d];
  for (int d = 0; d < 4; ++d) v[3 + d] = g.quat[4 * m + d];
  for (int d = 0; d < 3; ++d)
    v[7 + d] = g.scale[3 * m + d] * (scale[3 * i + d] * expf(out[m * kOutCols + 7 + d]));
  for (int d = 0; d < 3; ++d) v[10 + d] = g.freq[3 * m + d];
  for (int d = 13; d < kOutCols; ++d) v[d] = 0.f;
  // one row = 32 B of bf16 + 64 B of fp32: 16-byte vector stores
  static_assert(kOutCols == 16, "row of 16 outputs");
  uint4 u[2];
  uint32_t* w = reinterpret_cast<uint32_t*>(u);
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    const __nv_bfloat162 pr = __floats2bfloat162_rn(v[2 * h], v[2 * h + 1]);
    w[h] = *reinterpret_cast<const uint32_t*>(&pr);
  }
  if (x3) {  // [hi | hi | lo] rows of 3 x 16 (R38)
    uint4 l[2];
    uint32_t* wl = reinterpret_cast<uint32_t*>(l);
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&w[h]);
      const __nv_bfloat162 lo = __floats2bfloat162_rn(v[2 * h] - __low2float(hi),
                                                      v[2 * h + 1] - __high2float(hi));
      wl[h] = *reinterpret_cast<const uint32_t*>(&lo);
    }
    uint4* db = reinterpret_cast<uint4*>(dbf + m * 3 * kOutCols);
    db[0] = u[0]; db[1] = u[1]; db[2] = u[0]; db[3] = u[1]; db[4] = l[0]; db[5] = l[1];
  } else {
    uint4* db = reinterpret_cast<uint4*>(dbf + m * kOutCols);
    db[0] = u[0];
    db[1] = u[1];
  }
  float4* d4 = reinterpret_cast<float4*>(df + m * kOutCols);
#pragma unroll
  for (int q = 0; q < 4; ++q) d4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
}

// Head-bias gradient: column sums of dL/dout (fp32) over the rows.
__global__ void __launch_bounds__(256) k_mlp_dout_colsum(const float* df, int64_t M, float* gb) {
  __shared__ float part[8][13];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float acc[13];
  for (int d = 0; d < 13; ++d) acc[d] = 0.f;
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < M;
       m += (int64_t)gridDim.x * blockDim.x)
    for (int d = 0; d < 13; ++d) acc[d] += df[m * kOutCols + d];
  for (int d = 0; d < 13; ++d) {
    float x = acc[d];
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) part[w][d] = x;
  }
  __syncthreads();
  if (threadIdx.x < 13) {
    float x = 0.f;
    for (int k = 0; k < 8; ++k) x += part[k][threadIdx.x];
    atomicAdd(gb + threadIdx.x, x);
  }
}

// Canonical gradients: sums over the F frames (fixed order: deterministic).
__global__ void __launch_bounds__(128) k_mlp_canon(int64_t N, int32_t F, const float* out,
                                                   wipes_grads gf, wipes_grads gc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  float gm[3] = {0, 0, 0}, gq[4] = {0, 0, 0, 0}, gs[3] = {0, 0, 0}, gfr[3] = {0, 0, 0};
  for (int f = 0; f < F; ++f) {
    const int64_t m = (int64_t)f * N + i;
    for (int d = 0; d < 3; ++d) gm[d] += gf.mean[3 * m + d];
    for (int d = 0; d < 4; ++d) gq[d] += gf.quat[4 * m + d];
    for (int d = 0; d < 3; ++d) gs[d] += gf.scale[3 * m + d] * expf(out[m * kOutCols + 7 + d]);
    for (int d = 0; d < 3; ++d) gfr[d] += gf.freq[3 * m + d];
  }
  if (gc.mean) for (int d = 0; d < 3; ++d) gc.mean[3 * i + d] = gm[d];
  if (gc.quat) for (int d = 0; d < 4; ++d) gc.quat[4 * i + d] = gq[d];
  if (gc.scale) for (int d = 0; d < 3; ++d) gc.scale[3 * i + d] = gs[d];
  if (gc.freq) for (int d = 0; d < 3; ++d) gc.freq[3 * i + d] = gfr[d];
}

// Padded dW scratch [rows, Kp] -> theta-gradient layout (true widths).
__global__ void k_mlp_unpad(const float* dws, int rows, int Kp, int E, int E8, int K,
                            bool has_cat, float* g) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)rows * K) return;
  const int j = (int)(idx / K), k = (int)(idx - (int64_t)j * K);
  const int c = !has_cat ? k : (k < E ? k : k - E + E8);
  g[idx] = dws[(int64_t)j * Kp + c];
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// dst[row * ldd + col] (+)= sum_p parts[p n + i] for i = row * cols + col
// (deterministic: thread row y sums the parts p = y (mod blockDim.y) in order,
// then the row sums are added in order y = 0, 1, ..). cols, ldd, n % 4 == 0.
// Up to two independent jobs per launch (blockIdx.y).
struct PartJob {
  const float* parts;
  int np;
  int64_t n, cols, ldd;
  float* dst;
  bool add;
};
struct PartJobs { PartJob j[2]; };

__global__ void k_mlp_partsum(const __grid_constant__ PartJobs jobs) {
  __shared__ float4 red[1024];
  const PartJob& jb = jobs.j[blockIdx.y];
  const int64_t i = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if ((int64_t)blockIdx.x * blockDim.x * 4 >= jb.n) return;  // whole block idle (uniform)
  const int S = blockDim.y, y = threadIdx.y;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (i < jb.n) {
    int p = y;
    for (; p + 3 * S < jb.np; p += 4 * S) {  // four loads in flight per thread
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(jb.parts + (int64_t)(p + u * S) * jb.n + i));
#pragma unroll
      for (int u = 0; u < 4; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
    for (; p < jb.np; p += S) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(jb.parts + (int64_t)p * jb.n + i));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  red[y * blockDim.x + threadIdx.x] = acc;
  __syncthreads();
  if (y == 0 && i < jb.n) {
    float* d = jb.dst + (i / jb.cols) * jb.ldd + (i % jb.cols);
    float4 t = jb.add ? *reinterpret_cast<const float4*>(d) : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < S; ++k) {
      const float4 v = red[k * blockDim.x + threadIdx.x];
      t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
    }
    *reinterpret_cast<float4*>(d) = t;
  }
}

PartJob part_job(const float* parts, int np, int64_t n, float* dst, bool add, int64_t cols = 0,
                 int64_t ldd = 0) {
  PartJob j;
  j.parts = parts; j.np = np; j.n = n; j.dst = dst; j.add = add;
  j.cols = cols ? cols : n;
  j.ldd = cols ? ldd : n;
  return j;
}

// the weight and bias partial sums of one fused layer in one launch
void partsum2(const PartJob& a, const PartJob& b, cudaStream_t s) {
  PartJobs jobs;
  jobs.j[0] = a;
  jobs.j[1] = b;
  const int64_t nmax = a.n > b.n ? a.n : b.n;
  launch_begin(K_MLP_MISC, s);
  k_mlp_partsum<<<dim3(nblk(nmax / 4, 128), 2), dim3(128, 8), 0, s>>>(jobs);
  launch_end(K_MLP_MISC, s);
}

bool mlp_unfused_env() {
  static const bool unfused = getenv("WIPES_MLP_UNFUSED") != nullptr;
  return unfused;
}

cudaError_t gemm(const void* A, const void* B, void* C, int64_t M, int64_t N, int64_t K,
                 int64_t lda, int64_t ldb, int64_t ldc, int epi, bool amn, bool bmn,
                 const float* bias, const void* mask, int64_t ldm, int split, cudaStream_t s,
                 float* colsum = nullptr, int64_t split3 = 0) {
  wipes_gemm_args g;
  g.colsum = colsum;
  g.split3 = split3;
  g.A = A; g.B = B; g.C = C; g.bias = bias; g.mask = mask;
  g.M = M; g.N = N; g.K = K; g.lda = lda; g.ldb = ldb; g.ldc = ldc; g.ldm = ldm;
  g.a_mn_major = amn; g.b_mn_major = bmn; g.epilogue = epi; g.split_k = split;
  return launch_gemm(g, s);
}

}  // namespace

// ---------------------------------------------------------------------------
// x3 (WIPES_MLP_BF16X3, R38): the same network with every operand a
// split-bf16 pair. Activation buffers hold [hi | hi | lo] column blocks (the
// GEMM epilogue writes them, split3 = width), weights [hi | lo | hi] per input
// segment, so each layer is ONE bf16 GEMM over K' = 3K forming
// hi.hi + hi.lo + lo.hi (the lo.lo term, ~2^-18 relative, is dropped) with fp32
// accumulation. The layer-by-layer generic GEMM only (the fused bf16 kernels of
// mlp_fused.cu keep single-bf16 layouts).
// ---------------------------------------------------------------------------
cudaError_t mlp_forward_x3(const MlpLayout& L, const float* theta, int64_t N, int32_t F,
                           const float* times, const wipes_params& canon,
                           const wipes_params& frame, int32_t sh_coeffs, char* ws,
                           cudaStream_t s) {
  const int64_t M = L.M;
  {
    WeightJobsX3 wj;
    wj.n = L.D + 1;
    for (int l = 0; l <= L.D; ++l) {
      WeightJobsX3::Job& jb = wj.j[l];
      if (l < L.D) {
        jb.thW = L.thW[l]; jb.rows = L.W; jb.rows_valid = L.W; jb.Kp = L.Kp[l]; jb.K = L.K[l];
        jb.has_cat = l == L.skip + 1;
        jb.dst = (__nv_bfloat16*)(ws + L.wbf[l]); jb.dstb = (__nv_bfloat16*)(ws + L.wb3[l]);
      } else {
        jb.thW = L.thWh; jb.rows = kOutCols; jb.rows_valid = 13; jb.Kp = L.W; jb.K = L.W;
        jb.has_cat = false;
        jb.dst = (__nv_bfloat16*)(ws + L.whbf); jb.dstb = (__nv_bfloat16*)(ws + L.whb3);
      }
    }
    launch_begin(K_MLP_MISC, s);
    k_mlp_weights_x3<<<dim3(64, wj.n), 256, 0, s>>>(theta, L.E, L.E8, wj);
    launch_end(K_MLP_MISC, s);
  }
  __nv_bfloat16* cat = (__nv_bfloat16*)(ws + L.cat);
  const int64_t E3 = 3 * (int64_t)L.E8, W3 = 3 * (int64_t)L.W;
  static thread_local EmbedArgs ea;
  for (int f0 = 0; f0 < F; f0 += kMlpMaxFrames) {
    const int nf = F - f0 < kMlpMaxFrames ? F - f0 : kMlpMaxFrames;
    ea.mean = canon.mean; ea.N = N; ea.row0 = (int64_t)f0 * N; ea.rows = (int64_t)nf * N;
    ea.f0 = f0; ea.Lx = L.Lx; ea.Lt = L.Lt; ea.E8 = L.E8; ea.catw = L.catw; ea.cat = cat;
    ea.x3 = 1;
    for (int k = 0; k < nf; ++k) ea.t[k] = times[f0 + k];
    launch_begin(K_MLP_MISC, s);
    if (L.Lx == 10 && L.Lt == 6)
      k_mlp_embed<10, 6><<<nblk(ea.rows, 128), 128, 0, s>>>(ea);
    else
      k_mlp_embed<0, 0><<<nblk(ea.rows, 128), 128, 0, s>>>(ea);
    launch_end(K_MLP_MISC, s);
  }
  cudaError_t e = cudaSuccess;
  for (int l = 0; l < L.D && e == cudaSuccess; ++l) {
    const void* in;
    int64_t ldin, K3;
    if (l == 0) { in = cat; ldin = L.catw; K3 = E3; }
    else if (l == L.skip + 1) { in = cat; ldin = L.catw; K3 = L.catw; }
    else if (l - 1 == L.skip) { in = cat + E3; ldin = L.catw; K3 = W3; }
    else { in = ws + L.h[l - 1]; ldin = W3; K3 = W3; }
    void* outp = l == L.skip ? (void*)(cat + E3) : (void*)(ws + L.h[l]);
    const int64_t ldo = l == L.skip ? L.catw : W3;
    e = gemm(in, ws + L.wbf[l], outp, M, L.W, K3, ldin, 3 * (int64_t)L.Kp[l], ldo,
             WIPES_GEMM_EPI_BIAS_RELU_BF16, false, false, theta + L.thb[l], nullptr, 0, 1, s,
             nullptr, L.W);
  }
  if (e != cudaSuccess) return e;
  const int last = L.D - 1;
  const void* hl = last == L.skip ? (const void*)(cat + E3) : (const void*)(ws + L.h[last]);
  const int64_t ldh = last == L.skip ? L.catw : W3;
  e = gemm(hl, ws + L.whbf, ws + L.out, M, 13, W3, ldh, W3, kOutCols, WIPES_GEMM_EPI_BIAS_F32,
           false, false, theta + L.thbh, nullptr, 0, 1, s);
  if (e != cudaSuccess) return e;
  ApplyArgs aa;
  aa.N = N; aa.M = M; aa.out = (const float*)(ws + L.out); aa.canon = canon; aa.frame = frame;
  aa.sh_coeffs = sh_coeffs;
  launch_begin(K_MLP_MISC, s);
  k_mlp_apply<<<nblk(M, 128), 128, 0, s>>>(aa);
  launch_end(K_MLP_MISC, s);
  return cudaGetLastError();
}

// dW (rows x cols, fp32, += into C with leading dimension ldc) = dz^T in over
// the M rows, split-bf16: dz_hi.in_hi + dz_hi.in_lo + dz_lo.in_hi (three
// accumulating GEMMs; dz and in are [hi | hi | lo] blocks of width dzw / inw).
cudaError_t mlp_dw_x3(const __nv_bfloat16* dz, int64_t dzw, const __nv_bfloat16* in, int64_t ldin,
                      int64_t inw, int64_t cols, int64_t rows, int64_t M, float* C, int64_t ldc,
                      int split, cudaStream_t s) {
  const int64_t ldz = 3 * dzw;
  const __nv_bfloat16* a[3] = {dz, dz, dz + 2 * dzw};
  const __nv_bfloat16* b[3] = {in, in + 2 * inw, in};
  for (int t = 0; t < 3; ++t) {
    cudaError_t e = gemm(a[t], b[t], C, rows, cols, M, ldz, ldin, ldc, WIPES_GEMM_EPI_ATOMIC_F32,
                         true, true, nullptr, nullptr, 0, split, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t mlp_backward_x3(const MlpLayout& L, const float* theta, int64_t N, int32_t F,
                            const wipes_params& canon, const wipes_grads& gfr, float* g_theta,
                            const wipes_grads& gcan, char* ws, cudaStream_t s) {
  const int64_t M = L.M;
  cudaError_t e = cudaMemsetAsync(g_theta, 0, sizeof(float) * L.P, s);
  if (e != cudaSuccess || M == 0) return e;
  __nv_bfloat16* cat = (__nv_bfloat16*)(ws + L.cat);
  const float* out = (const float*)(ws + L.out);
  __nv_bfloat16* dbf = (__nv_bfloat16*)(ws + L.dout_bf);
  float* dfp = (float*)(ws + L.dout_f);
  const int64_t E3 = 3 * (int64_t)L.E8, W3 = 3 * (int64_t)L.W;
  launch_begin(K_MLP_MISC, s);
  k_mlp_dout<<<nblk(M, 128), 128, 0, s>>>(N, M, out, canon.scale, gfr, dbf, dfp, 1);
  launch_end(K_MLP_MISC, s);
  launch_begin(K_MLP_MISC, s);
  k_mlp_canon<<<nblk(N, 128), 128, 0, s>>>(N, F, out, gfr, gcan);
  launch_end(K_MLP_MISC, s);
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  auto split_for = [&](int64_t tiles) {
    int64_t sp = (2 * sms + tiles - 1) / tiles;
    const int64_t chunks = (M + 63) / 64;
    return (int)(sp < 1 ? 1 : (sp > chunks ? chunks : sp));
  };
  const int last = L.D - 1;
  const __nv_bfloat16* hl = last == L.skip ? cat + E3 : (const __nv_bfloat16*)(ws + L.h[last]);
  const int64_t ldh = last == L.skip ? L.catw : W3;
  float* dws = (float*)(ws + L.dws);
  // head: dWh = dout^T h_last (13 x W), dbh = colsum(dout), dh_last = dout Wh
  e = cudaMemsetAsync(dws, 0, sizeof(float) * 13 * L.W, s);
  if (e != cudaSuccess) return e;
  e = mlp_dw_x3(dbf, kOutCols, hl, ldh, L.W, L.W, 13, M, dws, L.W,
                split_for((L.W + 255) / 256), s);
  if (e != cudaSuccess) return e;
  launch_begin(K_MLP_MISC, s);
  k_mlp_unpad<<<nblk(13 * (int64_t)L.W, 256), 256, 0, s>>>(dws, 13, L.W, L.E, L.E8, L.W, false,
                                                           g_theta + L.thWh);
  launch_end(K_MLP_MISC, s);
  launch_begin(K_MLP_MISC, s);
  k_mlp_dout_colsum<<<2 * sms, 256, 0, s>>>(dfp, M, g_theta + L.thbh);
  launch_end(K_MLP_MISC, s);
  __nv_bfloat16* dz = (__nv_bfloat16*)(ws + L.dz[0]);
  __nv_bfloat16* dz2 = (__nv_bfloat16*)(ws + L.dz[1]);
  e = gemm(dbf, ws + L.whb3, dz, M, L.W, 3 * kOutCols, 3 * kOutCols, L.W, W3,
           WIPES_GEMM_EPI_MASK_BF16, false, true, nullptr, hl, ldh, 1, s, g_theta + L.thb[last],
           L.W);
  if (e != cudaSuccess) return e;
  for (int l = last; l >= 0; --l) {
    e = cudaMemsetAsync(dws, 0, sizeof(float) * (size_t)L.W * L.Kp[l], s);
    if (e != cudaSuccess) return e;
    const bool has_cat = l == L.skip + 1;
    if (l == 0 || has_cat) {  // the encoding segment: dws columns [0, E8)
      e = mlp_dw_x3(dz, L.W, cat, L.catw, L.E8, L.E8, L.W, M, dws, L.Kp[l],
                    split_for((L.W + 127) / 128), s);
      if (e != cudaSuccess) return e;
    }
    if (l > 0) {  // the hidden segment
      const __nv_bfloat16* hin = (l - 1 == L.skip) ? cat + E3
                                                   : (const __nv_bfloat16*)(ws + L.h[l - 1]);
      const int64_t ldin = (l - 1 == L.skip) ? L.catw : W3;
      e = mlp_dw_x3(dz, L.W, hin, ldin, L.W, L.W, L.W, M, dws + (has_cat ? L.E8 : 0), L.Kp[l],
                    split_for(((L.W + 127) / 128) * ((L.W + 255) / 256)), s);
      if (e != cudaSuccess) return e;
    }
    launch_begin(K_MLP_MISC, s);
    k_mlp_unpad<<<nblk((int64_t)L.W * L.K[l], 256), 256, 0, s>>>(
        dws, L.W, L.Kp[l], L.E, L.E8, L.K[l], has_cat, g_theta + L.thW[l]);
    launch_end(K_MLP_MISC, s);
    if (l == 0) break;
    // dz_(l-1) = (dz W_l)[:, hidden part] * (h_(l-1) > 0), split; its column sums
    // are the bias gradient of layer l-1
    const __nv_bfloat16* wl = (const __nv_bfloat16*)(ws + L.wb3[l]) + (has_cat ? L.E8 : 0);
    const void* mask = (l - 1 == L.skip) ? (const void*)(cat + E3) : (const void*)(ws + L.h[l - 1]);
    const int64_t ldm = (l - 1 == L.skip) ? L.catw : W3;
    e = gemm(dz, wl, dz2, M, L.W, W3, W3, L.Kp[l], W3, WIPES_GEMM_EPI_MASK_BF16, false, true,
             nullptr, mask, ldm, 1, s, g_theta + L.thb[l - 1], L.W);
    if (e != cudaSuccess) return e;
    __nv_bfloat16* t = dz; dz = dz2; dz2 = t;
  }
  return cudaGetLastError();
}

bool mlp_config_valid(const wipes_mlp_config& c) { return mlp_cfg_ok(c); }
int64_t mlp_param_count(const wipes_mlp_config& c) { return mlp_layout(c, 0).P; }
size_t mlp_workspace_bytes(const wipes_mlp_config& c, int64_t rows) {
  return mlp_layout(c, rows).total;
}

cudaError_t launch_mlp_forward(const wipes_mlp_config& c, const float* theta, int64_t N,
                               int32_t F, const float* times, const wipes_params& canon,
                               const wipes_params& frame, int32_t sh_coeffs, int32_t train,
                               char* ws, cudaStream_t s) {
  const int64_t M = N * (int64_t)F;
  const MlpLayout L = mlp_layout(c, M);
  if (M == 0) return cudaSuccess;
  if (L.x3) return mlp_forward_x3(L, theta, N, F, times, canon, frame, sh_coeffs, ws, s);
  // bf16 weights (rounded to nearest even)
  {
    WeightJobs wj;
    wj.n = L.D + 1;
    for (int l = 0; l <= L.D; ++l) {
      WeightJobs::Job& jb = wj.j[l];
      if (l < L.D) {
        jb.thW = L.thW[l]; jb.rows = L.W; jb.rows_valid = L.W; jb.Kp = L.Kp[l]; jb.K = L.K[l];
        jb.has_cat = l == L.skip + 1; jb.dst = (__nv_bfloat16*)(ws + L.wbf[l]);
      } else {
        jb.thW = L.thWh; jb.rows = kOutCols; jb.rows_valid = 13; jb.Kp = L.W; jb.K = L.W;
        jb.has_cat = false; jb.dst = (__nv_bfloat16*)(ws + L.whbf);
      }
    }
    launch_begin(K_MLP_MISC, s);
    k_mlp_weights_all<<<dim3(64, wj.n), 256, 0, s>>>(theta, L.E, L.E8, wj);
    launch_end(K_MLP_MISC, s);
  }
  __nv_bfloat16* cat = (__nv_bfloat16*)(ws + L.cat);
  // fused path (mlp_fused.cu): all layers of a 128-row tile on chip. Measured
  // faster for inference only (0.60 vs 0.66 ms at 300k rows); with train = 1
  // its activation stores make it slower (0.76 ms), so training keeps the
  // layer-by-layer schedule unless WIPES_MLP_FUSED=1.
  const bool unfused = mlp_unfused_env();
  static const bool fused_train = getenv("WIPES_MLP_FUSED") != nullptr;
  if (!unfused && (!train || fused_train)) {
    MlpFusedDesc d;
    std::memset(&d, 0, sizeof(d));
    d.W = L.W; d.D = L.D; d.skip = L.skip; d.Lx = L.Lx; d.Lt = L.Lt; d.E8 = L.E8;
    d.catw = L.catw; d.train = train; d.shc = sh_coeffs; d.F = F; d.N = N; d.M = M;
    d.times = times; d.theta = theta; d.thbh = L.thbh;
    for (int l = 0; l < L.D; ++l) {
      d.thb[l] = L.thb[l];
      d.wbf[l] = (const __nv_bfloat16*)(ws + L.wbf[l]);
      d.Kp[l] = L.Kp[l];
      d.h[l] = l == L.skip ? nullptr : (__nv_bfloat16*)(ws + L.h[l]);
    }
    d.whbf = (const __nv_bfloat16*)(ws + L.whbf);
    d.cat = cat;
    d.canon = canon; d.frame = frame;
    d.out = (float*)(ws + L.out);
    cudaError_t fe = cudaSuccess;
    if (launch_mlp_fused_fwd(d, s, &fe)) return fe;
  }
  // positional encoding
  static thread_local EmbedArgs ea;
  for (int f0 = 0; f0 < F; f0 += kMlpMaxFrames) {
    const int nf = F - f0 < kMlpMaxFrames ? F - f0 : kMlpMaxFrames;
    ea.mean = canon.mean; ea.N = N; ea.row0 = (int64_t)f0 * N; ea.rows = (int64_t)nf * N;
    ea.f0 = f0; ea.Lx = L.Lx; ea.Lt = L.Lt; ea.E8 = L.E8; ea.catw = L.catw; ea.cat = cat;
    for (int k = 0; k < nf; ++k) ea.t[k] = times[f0 + k];
    launch_begin(K_MLP_MISC, s);
    if (L.Lx == 10 && L.Lt == 6)  // the D-3DGS encoding: unrolled, in registers
      k_mlp_embed<10, 6><<<nblk(ea.rows, 128), 128, 0, s>>>(ea);
    else
      k_mlp_embed<0, 0><<<nblk(ea.rows, 128), 128, 0, s>>>(ea);
    launch_end(K_MLP_MISC, s);
  }
  // layers
  cudaError_t e = cudaSuccess;
  for (int l = 0; l < L.D && e == cudaSuccess; ++l) {
    const void* in;
    int64_t ldin;
    if (l == 0 || l == L.skip + 1) { in = cat; ldin = L.catw; }
    else if (l - 1 == L.skip) { in = cat + L.E8; ldin = L.catw; }
    else { in = ws + L.h[l - 1]; ldin = L.W; }
    void* outp = l == L.skip ? (void*)(cat + L.E8) : (void*)(ws + L.h[l]);
    const int64_t ldo = l == L.skip ? L.catw : L.W;
    if (l >= 1 && l != L.skip + 1 && L.W == 256 && !unfused) {
      // x read once (CTA pairs split the output columns), transposed epilogue
      MlpFwdLayerDesc d;
      d.W = L.W; d.M = M; d.x = (const __nv_bfloat16*)in; d.x_ld = ldin;
      d.w = (const __nv_bfloat16*)(ws + L.wbf[l]); d.bias = theta + L.thb[l];
      d.out = (__nv_bfloat16*)outp; d.out_ld = ldo;
      cudaError_t fe = cudaSuccess;
      if (launch_mlp_fwd_layer(d, s, &fe)) {
        e = fe;
        continue;
      }
    }
    e = gemm(in, ws + L.wbf[l], outp, M, L.W, L.Kp[l], ldin, L.Kp[l], ldo,
             WIPES_GEMM_EPI_BIAS_RELU_BF16, false, false, theta + L.thb[l], nullptr, 0, 1, s);
  }
  if (e != cudaSuccess) return e;
  const int last = L.D - 1;
  const void* hl = last == L.skip ? (const void*)(cat + L.E8) : (const void*)(ws + L.h[last]);
  const int64_t ldh = last == L.skip ? L.catw : L.W;
  e = gemm(hl, ws + L.whbf, ws + L.out, M, 13, L.W, ldh, L.W, kOutCols, WIPES_GEMM_EPI_BIAS_F32,
           false, false, theta + L.thbh, nullptr, 0, 1, s);
  if (e != cudaSuccess) return e;
  ApplyArgs aa;
  aa.N = N; aa.M = M; aa.out = (const float*)(ws + L.out); aa.canon = canon; aa.frame = frame;
  aa.sh_coeffs = sh_coeffs;
  launch_begin(K_MLP_MISC, s);
  k_mlp_apply<<<nblk(M, 128), 128, 0, s>>>(aa);
  launch_end(K_MLP_MISC, s);
  return cudaGetLastError();
}

cudaError_t launch_mlp_backward(const wipes_mlp_config& c, const float* theta, int64_t N,
                                int32_t F, const wipes_params& canon, const wipes_grads& gfr,
                                float* g_theta, const wipes_grads& gcan, char* ws,
                                cudaStream_t s) {
  const int64_t M = N * (int64_t)F;
  const MlpLayout L = mlp_layout(c, M);
  if (L.x3) return mlp_backward_x3(L, theta, N, F, canon, gfr, g_theta, gcan, ws, s);
  cudaError_t e = cudaMemsetAsync(g_theta, 0, sizeof(float) * L.P, s);
  if (e != cudaSuccess || M == 0) return e;
  __nv_bfloat16* cat = (__nv_bfloat16*)(ws + L.cat);
  const float* out = (const float*)(ws + L.out);
  __nv_bfloat16* dbf = (__nv_bfloat16*)(ws + L.dout_bf);
  float* dfp = (float*)(ws + L.dout_f);
  launch_begin(K_MLP_MISC, s);
  k_mlp_dout<<<nblk(M, 128), 128, 0, s>>>(N, M, out, canon.scale, gfr, dbf, dfp, L.x3 ? 1 : 0);
  launch_end(K_MLP_MISC, s);
  launch_begin(K_MLP_MISC, s);
  k_mlp_canon<<<nblk(N, 128), 128, 0, s>>>(N, F, out, gfr, gcan);
  launch_end(K_MLP_MISC, s);
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  auto split_for = [&](int64_t tiles) {  // split-K so that ~2 CTAs per SM run
    int64_t sp = (2 * sms + tiles - 1) / tiles;
    const int64_t chunks = (M + 63) / 64;
    return (int)(sp < 1 ? 1 : (sp > chunks ? chunks : sp));
  };
  // head: dWh = dout^T h_last, dbh = colsum(dout), dh_last = dout Wh (masked)
  const int last = L.D - 1;
  const __nv_bfloat16* hl = last == L.skip ? cat + L.E8 : (const __nv_bfloat16*)(ws + L.h[last]);
  const int64_t ldh = last == L.skip ? L.catw : L.W;
  float* dws = (float*)(ws + L.dws);
  e = cudaMemsetAsync(dws, 0, sizeof(float) * 13 * L.W, s);
  if (e != cudaSuccess) return e;
  e = gemm(dbf, hl, dws, 13, L.W, M, kOutCols, ldh, L.W, WIPES_GEMM_EPI_ATOMIC_F32, true, true,
           nullptr, nullptr, 0, split_for(1 * ((L.W + 255) / 256)), s);
  if (e != cudaSuccess) return e;
  launch_begin(K_MLP_MISC, s);
  k_mlp_unpad<<<nblk(13 * (int64_t)L.W, 256), 256, 0, s>>>(dws, 13, L.W, L.E, L.E8, L.W, false,
                                                           g_theta + L.thWh);
  launch_end(K_MLP_MISC, s);
  launch_begin(K_MLP_MISC, s);
  k_mlp_dout_colsum<<<2 * sms, 256, 0, s>>>(dfp, M, g_theta + L.thbh);
  launch_end(K_MLP_MISC, s);
  __nv_bfloat16* dz = (__nv_bfloat16*)(ws + L.dz[0]);
  __nv_bfloat16* dz2 = (__nv_bfloat16*)(ws + L.dz[1]);
  int hgroups = 0;
  if (L.W == 256 && !mlp_unfused_env()) {  // thin-K stream: mlp_fused.cu k_mlp_head_bwd
    MlpHeadBwdDesc hd;
    hd.M = M; hd.h_ld = ldh; hd.dout = dbf; hd.wh = (const __nv_bfloat16*)(ws + L.whbf);
    hd.h = hl; hd.dz = dz; hd.bpart = (float*)(ws + L.bpart); hd.W = L.W;
    hd.max_groups = kMlpBwdMaxGroups;
    cudaError_t he = cudaSuccess;
    hgroups = launch_mlp_head_bwd(hd, s, &he);
    if (he != cudaSuccess) return he;
    if (hgroups > 0) {
      partsum2(part_job(hd.bpart, 2 * hgroups, L.W, g_theta + L.thb[last], true),
               part_job(nullptr, 0, 0, nullptr, false), s);  // (second job empty)
    }
  }
  if (hgroups == 0) {
    e = gemm(dbf, ws + L.whbf, dz, M, L.W, kOutCols, kOutCols, L.W, L.W, WIPES_GEMM_EPI_MASK_BF16,
             false, true, nullptr, hl, ldh, 1, s, g_theta + L.thb[last]);
    if (e != cudaSuccess) return e;
  }
  for (int l = last; l >= 0; --l) {
    // dz = dL/dz_l [M, W]; input of layer l:
    const void* in;
    int64_t ldin;
    if (l == 0 || l == L.skip + 1) { in = cat; ldin = L.catw; }
    else if (l - 1 == L.skip) { in = cat + L.E8; ldin = L.catw; }
    else { in = ws + L.h[l - 1]; ldin = L.W; }
    const bool has_cat = l == L.skip + 1;
    if (l >= 1 && L.W == 256 && !mlp_unfused_env()) {
      // both GEMMs of the layer in one pass over dz and h_(l-1) (mlp_fused.cu);
      // after the skip the input is [encoding | h]: the fused pass takes the h
      // part, a narrow GEMM the encoding columns of dW
      MlpBwdDesc d;
      d.W = L.W; d.M = M;
      d.dz = dz;
      d.act = (const __nv_bfloat16*)in + (has_cat ? L.E8 : 0);
      d.act_ld = ldin;
      d.wl = (const __nv_bfloat16*)(ws + L.wbf[l]) + (has_cat ? L.E8 : 0);
      d.w_ld = L.Kp[l];
      d.dzo = dz2;
      d.wpart = (float*)(ws + L.wpart); d.bpart = (float*)(ws + L.bpart);
      d.max_groups = kMlpBwdMaxGroups;
      cudaError_t fe = cudaSuccess;
      const int groups = launch_mlp_bwd_layer(d, s, &fe);
      if (fe != cudaSuccess) return fe;
      if (groups > 0) {
        const int64_t n = (int64_t)L.W * L.W;
        const PartJob bj = part_job(d.bpart, 2 * groups, L.W, g_theta + L.thb[l - 1], true);
        if (!has_cat) {
          partsum2(part_job(d.wpart, groups, n, g_theta + L.thW[l], false), bj, s);
        } else {
          e = cudaMemsetAsync(dws, 0, sizeof(float) * (size_t)L.W * L.Kp[l], s);
          if (e != cudaSuccess) return e;
          e = gemm(dz, in, dws, L.W, L.E8, M, L.W, ldin, L.Kp[l], WIPES_GEMM_EPI_ATOMIC_F32, true,
                   true, nullptr, nullptr, 0, split_for((L.W + 127) / 128), s);
          if (e != cudaSuccess) return e;
          partsum2(part_job(d.wpart, groups, n, dws + L.E8, false, L.W, L.Kp[l]), bj, s);
          launch_begin(K_MLP_MISC, s);
          k_mlp_unpad<<<nblk((int64_t)L.W * L.K[l], 256), 256, 0, s>>>(
              dws, L.W, L.Kp[l], L.E, L.E8, L.K[l], true, g_theta + L.thW[l]);
          launch_end(K_MLP_MISC, s);
        }
        __nv_bfloat16* t = dz; dz = dz2; dz2 = t;
        continue;
      }
    }
    e = cudaMemsetAsync(dws, 0, sizeof(float) * (size_t)L.W * L.Kp[l], s);
    if (e != cudaSuccess) return e;
    const int64_t tiles = ((L.W + 127) / 128) * ((L.Kp[l] + 255) / 256);
    e = gemm(dz, in, dws, L.W, L.Kp[l], M, L.W, ldin, L.Kp[l], WIPES_GEMM_EPI_ATOMIC_F32, true,
             true, nullptr, nullptr, 0, split_for(tiles), s);
    if (e != cudaSuccess) return e;
    launch_begin(K_MLP_MISC, s);
    k_mlp_unpad<<<nblk((int64_t)L.W * L.K[l], 256), 256, 0, s>>>(
        dws, L.W, L.Kp[l], L.E, L.E8, L.K[l], has_cat, g_theta + L.thW[l]);
    launch_end(K_MLP_MISC, s);
    if (l == 0) break;
    // dz_(l-1) = (dz W_l)[:, h part] * (h_(l-1) > 0)
    const __nv_bfloat16* wl = (const __nv_bfloat16*)(ws + L.wbf[l]) + (has_cat ? L.E8 : 0);
    const void* mask = (l - 1 == L.skip) ? (const void*)(cat + L.E8) : (const void*)(ws + L.h[l - 1]);
    const int64_t ldm = (l - 1 == L.skip) ? L.catw : L.W;
    // its epilogue also sums dz_(l-1) over the rows: the bias gradient of layer l-1
    e = gemm(dz, wl, dz2, M, L.W, L.W, L.W, L.Kp[l], L.W, WIPES_GEMM_EPI_MASK_BF16, false, true,
             nullptr, mask, ldm, 1, s, g_theta + L.thb[l - 1]);
    if (e != cudaSuccess) return e;
    __nv_bfloat16* t = dz; dz = dz2; dz2 = t;
  }
  return cudaGetLastError();
}

}  // namespace wipes
