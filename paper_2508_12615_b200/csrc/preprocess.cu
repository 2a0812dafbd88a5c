// Preprocess kernels — compiled with
// --fmad=false so every FP64 expression rounds exactly as written, in the
// pinned order of DESIGN.md "Pinned preprocess arithmetic" (the integer
// decisions — tile rects and counts — must match the CPU oracle bit for bit).
//
//  k_pre2d      : PAPER.md:299 (Cholesky / RS covariances), Eq. 4 inputs.
//  k_pre3d      : PAPER.md:106 (Sigma = R S S^T R^T), :116-122 (Eq. 2, J W),
//                 :194-198 (Eq. 7), :212 (frequency transform, R3).
//  k_pre2d_bwd / k_pre3d_bwd : chain rule of the above ("explicit gradients
//                 for all parameters"), in FP64.
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cuda_fp16.h>

#include "common.cuh"

namespace wipes {

namespace {

constexpr double kLog2e = 1.4426950408889634;
#ifndef WIPES_PRE3D_MINB
#define WIPES_PRE3D_MINB 3  // min CTAs/SM, FP64 3D backward (168 registers, small spills: C3 0.512 -> 0.441 ms vs 2)
#endif
#ifndef WIPES_PRE3D_BWD_PRIM_ONCE
#define WIPES_PRE3D_BWD_PRIM_ONCE 0  // 1: quaternion/R/S3 once per row (C3 bwd 0.451 vs 0.441 ms per view: registers)
#endif
#ifndef WIPES_PRE3D_VMINOR
#define WIPES_PRE3D_VMINOR 0  // 1: views of a primitive in adjacent threads for flat colour too
                              // (C3 k_pre3d 0.419 -> 0.452 ms: the scattered record writes cost
                              // more than the 465 MB of parameter re-reads save)
#endif
#ifndef WIPES_PRE3D_FWD_MINB
#define WIPES_PRE3D_FWD_MINB 8  // min CTAs/SM, FP64 3D forward (measured faster at 64 registers)
#endif

struct PreOut {
  int4* rect;
  int32_t* count;
  uint8_t* flag;
  uint32_t* dkey;
  float4* rec;
  uint8_t* cull_flags;
  int32_t* arrive;  // WsHeader::arrive, zeroed here for the binning kernels that follow
};

__device__ __forceinline__ bool fin(double x) { return isfinite(x); }

__device__ __forceinline__ uint32_t orderable(float v) {
  uint32_t u = __float_as_uint(v);
  return (u >> 31) ? ~u : (u | 0x80000000u);
}

struct Cfg2 {
  int32_t W, H, tile, GX, GY, extent, alpha_blend, row_mod, row_rem;
  double alpha_min, det_min, diag;  // diag = cov_eps + dilation
};

// Steps 3-7 of O1 on Sigma' (diag offset already added) and the
// render record. Returns the cull flag.
__device__ int finish2d(const Cfg2& c, double mux, double muy, double sxx, double sxy,
                        double syy, double alpha, int4* rect, int32_t* count, double* conic,
                        double* ext) {
  *rect = make_int4(0, 0, 0, 0);
  *count = 0;
  double det = sxx * syy - sxy * sxy;
  if (!(det >= c.det_min) || !(sxx > 0.0) || !(syy > 0.0)) return 2;
  if (!(alpha >= c.alpha_min)) return 3;
  conic[0] = syy / det;
  conic[1] = -sxy / det;
  conic[2] = sxx / det;
  double rx, ry;
  // opacity-aware extent: alpha*W >= alpha_min  =>  |dx| <= k sqrt(sxx), |dy| <= k sqrt(syy)
  double k = (c.alpha_min > 0.0) ? sqrt(2.0 * log(alpha / c.alpha_min)) : (double)INFINITY;
  ext[0] = k * sqrt(sxx);
  ext[1] = k * sqrt(syy);
  if (c.extent == WIPES_EXTENT_OPACITY) {
    rx = ext[0];
    ry = ext[1];
  } else {
    double m = 0.5 * (sxx + syy);
    double lam = m + sqrt(fmax(m * m - det, 0.0));
    rx = 3.0 * sqrt(lam);
    ry = rx;
  }
  const double ts = (double)c.tile;
  double fx0 = floor((mux - rx) / ts), fx1 = floor((mux + rx) / ts) + 1.0;
  double fy0 = floor((muy - ry) / ts), fy1 = floor((muy + ry) / ts) + 1.0;
  fx0 = fmin(fmax(fx0, 0.0), (double)c.GX);
  fx1 = fmin(fmax(fx1, 0.0), (double)c.GX);
  fy0 = fmin(fmax(fy0, 0.0), (double)c.GY);
  fy1 = fmin(fmax(fy1, 0.0), (double)c.GY);
  int x0 = (int)fx0, x1 = (int)fx1, y0 = (int)fy0, y1 = (int)fy1;
  int ny = max(0, y1 - y0);
  if (c.row_mod > 1) ny = rows_in_band(y0, y1, c.row_mod, c.row_rem);
  int n = max(0, x1 - x0) * ny;
  *rect = make_int4(x0, y0, x1, y1);
  *count = n;
  return n == 0 ? 4 : 0;
}

__device__ void write_record(float4* rec, double mux, double muy, const double* conic,
                             double alpha, double fpx, double fpy, double phi, double beta,
                             double cr, double cg, double cb, const double* ext) {
  double ax = fmin(fmax(floor(mux), -1073741824.0), 1073741824.0);
  double ay = fmin(fmax(floor(muy), -1073741824.0), 1073741824.0);
  float4 r0, r1, r2, r3;
  r0.x = (float)ax;
  r0.y = (float)ay;
  r0.z = (float)(mux - ax);
  r0.w = (float)(muy - ay);
  r1.x = (float)(-0.5 * kLog2e * conic[0]);
  r1.y = (float)(-kLog2e * conic[1]);
  r1.z = (float)(-0.5 * kLog2e * conic[2]);
  r1.w = (float)log2(alpha);
  r2.x = (float)fpx;
  r2.y = (float)fpy;
  r2.z = (float)phi;
  r2.w = (float)(0.5 * beta);
  r3.x = (float)cr;
  r3.y = (float)cg;
  r3.z = (float)cb;
  // opacity-extent half widths as fp16, rounded UP (sub-tile culling only)
  __half2 e2 = __halves2half2(__float2half_ru((float)ext[0] * 1.0001f),
                              __float2half_ru((float)ext[1] * 1.0001f));
  r3.w = *reinterpret_cast<float*>(&e2);
  rec[0] = r0; rec[1] = r1; rec[2] = r2; rec[3] = r3;
}

__device__ __forceinline__ void zero_record(float4* rec) {
  float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  rec[0] = z; rec[1] = z; rec[2] = z; rec[3] = z;
}

// 2D covariance by mode (O1 step 1, pinned order).
__device__ __forceinline__ void cov2d(int mode, double p0, double p1, double p2, double* s) {
  if (mode == WIPES_COV2_SIGMA) {
    s[0] = p0; s[1] = p1; s[2] = p2;
  } else if (mode == WIPES_COV2_CHOLESKY) {
    s[0] = p0 * p0;
    s[1] = p0 * p1;
    s[2] = (p1 * p1) + (p2 * p2);
  } else {
    double cs = cos(p0), sn = sin(p0);
    double sx2 = p1 * p1, sy2 = p2 * p2;
    s[0] = (cs * cs) * sx2 + (sn * sn) * sy2;
    s[1] = (cs * sn) * (sx2 - sy2);
    s[2] = (sn * sn) * sx2 + (cs * cs) * sy2;
  }
}

struct Pre2DArgs {
  Cfg2 c;
  int32_t cov2;
  int64_t N;
  const float *mean, *cov, *freq, *phase, *color, *opacity, *depth;
  PreOut o;
};

#ifndef WIPES_PRE_BWD_TU  // forward kernels: this TU is built with --fmad=false (pinned FP64)
__global__ void __launch_bounds__(256) k_pre2d(Pre2DArgs a) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 4) a.o.arrive[i] = 0;
  if (i >= a.N) return;
  const Cfg2& c = a.c;
  double mux = a.mean[2 * i], muy = a.mean[2 * i + 1];
  double p0 = a.cov[3 * i], p1 = a.cov[3 * i + 1], p2 = a.cov[3 * i + 2];
  double fx = a.freq[2 * i], fy = a.freq[2 * i + 1];
  double phi = a.phase ? (double)a.phase[i] : 0.0;
  double cr = a.color[3 * i], cg = a.color[3 * i + 1], cb = a.color[3 * i + 2];
  double al = a.opacity[i];
  double dep = (c.alpha_blend && a.depth) ? (double)a.depth[i] : 0.0;
  int4 rect = make_int4(0, 0, 0, 0);
  int32_t cnt = 0;
  int flag;
  double conic[3] = {0, 0, 0}, ext[2] = {0, 0};
  bool ok = fin(mux) && fin(muy) && fin(p0) && fin(p1) && fin(p2) && fin(fx) && fin(fy) &&
            fin(phi) && fin(cr) && fin(cg) && fin(cb) && fin(al) && fin(dep);
  if (!ok) {
    flag = 5;
  } else {
    double s[3];
    cov2d(a.cov2, p0, p1, p2, s);
    flag = finish2d(c, mux, muy, s[0] + c.diag, s[1], s[2] + c.diag, al, &rect, &cnt, conic,
                    ext);
  }
  a.o.rect[i] = rect;
  a.o.count[i] = cnt;
  a.o.flag[i] = (uint8_t)flag;
  a.o.dkey[i] = c.alpha_blend ? orderable((float)dep) : 0u;
  if (a.o.cull_flags) a.o.cull_flags[i] = (uint8_t)flag;
  if (flag == 0)
    write_record(a.o.rec + 4 * i, mux, muy, conic, al, fx, fy, phi, 1.0, cr, cg, cb, ext);
  else
    zero_record(a.o.rec + 4 * i);
}

#endif

// ---------------------------------------------------------------- 3D ------
struct Proj3 {
  double p[3];
  double Rq[9], qn[4], qnorm;
  double S3[6];  // 00 01 02 11 12 22
  double j00, j02, j11, j12, thx, thy;
  bool clx, cly;
  double M[6];
  double g[3];
  double Sp[3];
};

__device__ __forceinline__ double s3at(const double* S, int i, int j) {
  int k = (i <= j) ? (i == 0 ? j : (i == 1 ? 2 + j : 5)) : (j == 0 ? i : (j == 1 ? 2 + i : 5));
  return S[k];
}

// O2 steps 1-9 in the pinned order. PINNED = false (backward
// only, where no integer decision is taken) replaces divisions by reciprocals.
// The view-independent half: normalised quaternion, rotation and S3 = R S^2 R^T.
template <bool PINNED = true>
__device__ __forceinline__ void project3_prim(const double* s, const double* q, Proj3& P) {
  double w = q[0], qx = q[1], qy = q[2], qz = q[3];
  double n = sqrt(((w * w + qx * qx) + qy * qy) + qz * qz);
  if (PINNED) {
    w = w / n; qx = qx / n; qy = qy / n; qz = qz / n;
  } else {
    const double rn = 1.0 / n;
    w *= rn; qx *= rn; qy *= rn; qz *= rn;
  }
  P.qn[0] = w; P.qn[1] = qx; P.qn[2] = qy; P.qn[3] = qz; P.qnorm = n;
  double* R = P.Rq;
  R[0] = 1.0 - 2.0 * ((qy * qy) + (qz * qz));
  R[1] = 2.0 * ((qx * qy) - (w * qz));
  R[2] = 2.0 * ((qx * qz) + (w * qy));
  R[3] = 2.0 * ((qx * qy) + (w * qz));
  R[4] = 1.0 - 2.0 * ((qx * qx) + (qz * qz));
  R[5] = 2.0 * ((qy * qz) - (w * qx));
  R[6] = 2.0 * ((qx * qz) - (w * qy));
  R[7] = 2.0 * ((qy * qz) + (w * qx));
  R[8] = 1.0 - 2.0 * ((qx * qx) + (qy * qy));
  double s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
  int k = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j)
      P.S3[k++] = (((R[3 * i] * s2[0]) * R[3 * j] + (R[3 * i + 1] * s2[1]) * R[3 * j + 1]) +
                   (R[3 * i + 2] * s2[2]) * R[3 * j + 2]);
}

// The per-view half (P.S3 from project3_prim): camera-space mean, EWA Jacobian,
// Sigma' = M S3 M^T and the rotated frequency.
template <bool PINNED = true>
__device__ __forceinline__ void project3_view(const float* cam, int32_t W, int32_t H,
                                              int32_t ewa_clamp, const double* mu,
                                              const double* f, Proj3& P) {
  double Rv[9];
  for (int k = 0; k < 9; ++k) Rv[k] = cam[k];
  double t0 = cam[9], t1 = cam[10], t2 = cam[11];
  double fx = cam[12], fy = cam[13];
  P.p[0] = ((Rv[0] * mu[0] + Rv[1] * mu[1]) + Rv[2] * mu[2]) + t0;
  P.p[1] = ((Rv[3] * mu[0] + Rv[4] * mu[1]) + Rv[5] * mu[2]) + t1;
  P.p[2] = ((Rv[6] * mu[0] + Rv[7] * mu[1]) + Rv[8] * mu[2]) + t2;
  double x = P.p[0], y = P.p[1], z = P.p[2];
  const double rz = PINNED ? 0.0 : 1.0 / z;
  double tx = PINNED ? x / z : x * rz, ty = PINNED ? y / z : y * rz;
  P.clx = P.cly = false;
  if (ewa_clamp) {
    double limx = (1.3 * (double)W) / (2.0 * fx);
    double limy = (1.3 * (double)H) / (2.0 * fy);
    P.clx = (tx < -limx || tx > limx);
    P.cly = (ty < -limy || ty > limy);
    tx = fmin(fmax(tx, -limx), limx);
    ty = fmin(fmax(ty, -limy), limy);
  }
  P.thx = tx; P.thy = ty;
  if (PINNED) {
    P.j00 = fx / z;
    P.j11 = fy / z;
    P.j02 = -(fx * tx) / z;
    P.j12 = -(fy * ty) / z;
  } else {
    P.j00 = fx * rz;
    P.j11 = fy * rz;
    P.j02 = -(fx * tx) * rz;
    P.j12 = -(fy * ty) * rz;
  }
  for (int jj = 0; jj < 3; ++jj) {
    P.M[jj] = P.j00 * Rv[jj] + P.j02 * Rv[6 + jj];
    P.M[3 + jj] = P.j11 * Rv[3 + jj] + P.j12 * Rv[6 + jj];
  }
  double T[2][3];
  for (int i = 0; i < 2; ++i)
    for (int kk = 0; kk < 3; ++kk)
      T[i][kk] = ((P.M[3 * i] * s3at(P.S3, 0, kk) + P.M[3 * i + 1] * s3at(P.S3, 1, kk)) +
                  P.M[3 * i + 2] * s3at(P.S3, 2, kk));
  P.Sp[0] = ((T[0][0] * P.M[0] + T[0][1] * P.M[1]) + T[0][2] * P.M[2]);
  P.Sp[1] = ((T[0][0] * P.M[3] + T[0][1] * P.M[4]) + T[0][2] * P.M[5]);
  P.Sp[2] = ((T[1][0] * P.M[3] + T[1][1] * P.M[4]) + T[1][2] * P.M[5]);
  P.g[0] = ((Rv[0] * f[0] + Rv[1] * f[1]) + Rv[2] * f[2]);
  P.g[1] = ((Rv[3] * f[0] + Rv[4] * f[1]) + Rv[5] * f[2]);
  P.g[2] = ((Rv[6] * f[0] + Rv[7] * f[1]) + Rv[8] * f[2]);
}

template <bool PINNED = true>
__device__ void project3(const float* cam, int32_t W, int32_t H, int32_t ewa_clamp,
                         const double* mu, const double* s, const double* q, const double* f,
                         Proj3& P) {
  project3_prim<PINNED>(s, q, P);
  project3_view<PINNED>(cam, W, H, ewa_clamp, mu, f, P);
}

// ------------------------------------------------ exact projection (NEXT-1) --
// Exact z-marginal of the modulated ray-space Gaussian (DESIGN.md
// R4): with the full ray-space covariance Sigma_hat (J3 row 3 = [0 0 1]),
// S2 its undilated upper-left 2x2, sigma = (Sigma_hat_xz, Sigma_hat_yz),
// v = Sigma_hat_zz - sigma^T S2^-1 sigma and f_hat = (J3 R)^-T f:
//   f' = f_hat_xy + f_hat_z S2^-1 sigma,  beta = exp(-1/2 f_hat_z^2 v).
// Written once, generic over the scalar (double in the forward, a forward-mode
// dual number in the backward, where it yields the exact Jacobian).
struct Dual {
  double v, d;
};
__device__ __forceinline__ Dual mk(double v) { return {v, 0.0}; }
__device__ __forceinline__ Dual operator+(Dual a, Dual b) { return {a.v + b.v, a.d + b.d}; }
__device__ __forceinline__ Dual operator-(Dual a, Dual b) { return {a.v - b.v, a.d - b.d}; }
__device__ __forceinline__ Dual operator-(Dual a) { return {-a.v, -a.d}; }
__device__ __forceinline__ Dual operator*(Dual a, Dual b) { return {a.v * b.v, a.d * b.v + a.v * b.d}; }
__device__ __forceinline__ Dual operator*(double a, Dual b) { return {a * b.v, a * b.d}; }
__device__ __forceinline__ Dual operator*(Dual a, double b) { return {a.v * b, a.d * b}; }
__device__ __forceinline__ Dual operator+(Dual a, double b) { return {a.v + b, a.d}; }
__device__ __forceinline__ Dual operator-(double a, Dual b) { return {a - b.v, -b.d}; }
__device__ __forceinline__ Dual operator/(Dual a, Dual b) {
  const double r = 1.0 / b.v;
  return {a.v * r, (a.d - a.v * r * b.d) * r};
}
__device__ __forceinline__ Dual operator/(Dual a, double b) { return {a.v / b, a.d / b}; }
__device__ __forceinline__ Dual operator/(double a, Dual b) {
  const double r = 1.0 / b.v;
  return {a * r, -a * r * r * b.d};
}
__device__ __forceinline__ Dual sqrtT(Dual a) {
  const double s = sqrt(a.v);
  return {s, a.d / (2.0 * s)};
}
__device__ __forceinline__ Dual expT(Dual a) {
  const double e = exp(a.v);
  return {e, e * a.d};
}
__device__ __forceinline__ double sqrtT(double a) { return sqrt(a); }
__device__ __forceinline__ double expT(double a) { return exp(a); }
__device__ __forceinline__ double val(double a) { return a; }
__device__ __forceinline__ double val(Dual a) { return a.v; }
template <typename T>
__device__ __forceinline__ T cst(double a);
template <>
__device__ __forceinline__ double cst<double>(double a) { return a; }
template <>
__device__ __forceinline__ Dual cst<Dual>(double a) { return mk(a); }
template <typename T>
__device__ __forceinline__ T clampT(T a, double lo, double hi) {  // zero partial when clamped
  if (val(a) < lo) return cst<T>(lo);
  if (val(a) > hi) return cst<T>(hi);
  return a;
}

// out = (mu'x, mu'y, conic a, b, c, f'x, f'y, beta); false if behind near/far.
template <typename T>
__device__ bool exact_rec(const float* cam, int32_t W, int32_t H, int32_t ewa_clamp,
                          double diag, const T* mu, const T* s, const T* q, const T* f,
                          T* out) {
  double Rv[9];
  for (int k = 0; k < 9; ++k) Rv[k] = cam[k];
  const double fx = cam[12], fy = cam[13], cx = cam[14], cy = cam[15];
  T p[3];
  for (int r = 0; r < 3; ++r)
    p[r] = Rv[3 * r] * mu[0] + Rv[3 * r + 1] * mu[1] + Rv[3 * r + 2] * mu[2] + (double)cam[9 + r];
  const T x = p[0], y = p[1], z = p[2];
  if (!(val(z) >= (double)cam[16] && val(z) <= (double)cam[17])) return false;
  const T n = sqrtT(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const T w = q[0] / n, qx = q[1] / n, qy = q[2] / n, qz = q[3] / n;
  T R[9];
  R[0] = 1.0 - 2.0 * (qy * qy + qz * qz);
  R[1] = 2.0 * (qx * qy - w * qz);
  R[2] = 2.0 * (qx * qz + w * qy);
  R[3] = 2.0 * (qx * qy + w * qz);
  R[4] = 1.0 - 2.0 * (qx * qx + qz * qz);
  R[5] = 2.0 * (qy * qz - w * qx);
  R[6] = 2.0 * (qx * qz - w * qy);
  R[7] = 2.0 * (qy * qz + w * qx);
  R[8] = 1.0 - 2.0 * (qx * qx + qy * qy);
  const T s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
  T S3[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      S3[i][j] = R[3 * i] * s2[0] * R[3 * j] + R[3 * i + 1] * s2[1] * R[3 * j + 1] +
                 R[3 * i + 2] * s2[2] * R[3 * j + 2];
  T tx = x / z, ty = y / z;
  if (ewa_clamp) {
    const double limx = (1.3 * (double)W) / (2.0 * fx), limy = (1.3 * (double)H) / (2.0 * fy);
    tx = clampT(tx, -limx, limx);
    ty = clampT(ty, -limy, limy);
  }
  const T j00 = fx / z, j11 = fy / z, j02 = -(fx * tx) / z, j12 = -(fy * ty) / z;
  T M3[3][3];
  for (int c = 0; c < 3; ++c) {
    M3[0][c] = j00 * Rv[c] + j02 * Rv[6 + c];
    M3[1][c] = j11 * Rv[3 + c] + j12 * Rv[6 + c];
    M3[2][c] = cst<T>(Rv[6 + c]);
  }
  T Sh[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j) {
      T acc = cst<T>(0.0);
      for (int a = 0; a < 3; ++a) {
        const T ta = M3[i][0] * S3[0][a] + M3[i][1] * S3[1][a] + M3[i][2] * S3[2][a];
        acc = acc + ta * M3[j][a];
      }
      Sh[i][j] = acc;
    }
  T g[3];
  for (int r = 0; r < 3; ++r) g[r] = Rv[3 * r] * f[0] + Rv[3 * r + 1] * f[1] + Rv[3 * r + 2] * f[2];
  const T fhx = (z * g[0]) / fx, fhy = (z * g[1]) / fy;
  const T fhz = g[2] - j02 * fhx - j12 * fhy;
  const T a2 = Sh[0][0], b2 = Sh[0][1], d2 = Sh[1][1], sx = Sh[0][2], sy = Sh[1][2];
  const T det2 = a2 * d2 - b2 * b2;
  const T ux = (d2 * sx - b2 * sy) / det2, uy = (a2 * sy - b2 * sx) / det2;
  const T vv = Sh[2][2] - (sx * ux + sy * uy);
  out[0] = fx * (x / z) + cx;
  out[1] = fy * (y / z) + cy;
  const T sxx = a2 + diag, sxy = b2, syy = d2 + diag;
  const T det = sxx * syy - sxy * sxy;
  out[2] = syy / det;
  out[3] = -sxy / det;
  out[4] = sxx / det;
  out[5] = fhx + fhz * ux;
  out[6] = fhy + fhz * uy;
  out[7] = expT(-0.5 * (fhz * fhz * vv));
  return true;
}

// ------------------------------------------------- SH colour (NEXT-3) ----
// Real SH basis up to degree 3 in the 3DGS sign convention (R33),
// with its gradient in d (the polynomial extension; the caller projects it
// through the normalisation d = v / |v|).
__device__ __forceinline__ void sh_basis(int deg, double x, double y, double z, double* Y,
                                         double (*dY)[3]) {
  const double c0 = 0.28209479177387814, c1 = 0.4886025119029199;
  const double c2a = 1.0925484305920792, c2b = 0.31539156525252005, c2c = 0.5462742152960396;
  const double c3a = 0.5900435899266435, c3b = 2.890611442640554, c3c = 0.4570457994644658,
               c3d = 0.3731763325901154, c3e = 1.445305721320277;
  Y[0] = c0;
  if (dY) dY[0][0] = dY[0][1] = dY[0][2] = 0.0;
  if (deg < 1) return;
  Y[1] = -c1 * y; Y[2] = c1 * z; Y[3] = -c1 * x;
  if (dY) {
    dY[1][0] = 0; dY[1][1] = -c1; dY[1][2] = 0;
    dY[2][0] = 0; dY[2][1] = 0; dY[2][2] = c1;
    dY[3][0] = -c1; dY[3][1] = 0; dY[3][2] = 0;
  }
  if (deg < 2) return;
  const double xx = x * x, yy = y * y, zz = z * z;
  Y[4] = c2a * x * y;
  Y[5] = -c2a * y * z;
  Y[6] = c2b * (2.0 * zz - xx - yy);
  Y[7] = -c2a * x * z;
  Y[8] = c2c * (xx - yy);
  if (dY) {
    dY[4][0] = c2a * y; dY[4][1] = c2a * x; dY[4][2] = 0;
    dY[5][0] = 0; dY[5][1] = -c2a * z; dY[5][2] = -c2a * y;
    dY[6][0] = -2.0 * c2b * x; dY[6][1] = -2.0 * c2b * y; dY[6][2] = 4.0 * c2b * z;
    dY[7][0] = -c2a * z; dY[7][1] = 0; dY[7][2] = -c2a * x;
    dY[8][0] = 2.0 * c2c * x; dY[8][1] = -2.0 * c2c * y; dY[8][2] = 0;
  }
  if (deg < 3) return;
  Y[9] = -c3a * y * (3.0 * xx - yy);
  Y[10] = c3b * x * y * z;
  Y[11] = -c3c * y * (4.0 * zz - xx - yy);
  Y[12] = c3d * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
  Y[13] = -c3c * x * (4.0 * zz - xx - yy);
  Y[14] = c3e * z * (xx - yy);
  Y[15] = -c3a * x * (xx - 3.0 * yy);
  if (dY) {
    dY[9][0] = -6.0 * c3a * x * y; dY[9][1] = -c3a * (3.0 * xx - 3.0 * yy); dY[9][2] = 0;
    dY[10][0] = c3b * y * z; dY[10][1] = c3b * x * z; dY[10][2] = c3b * x * y;
    dY[11][0] = 2.0 * c3c * x * y; dY[11][1] = -c3c * (4.0 * zz - xx - 3.0 * yy);
    dY[11][2] = -8.0 * c3c * y * z;
    dY[12][0] = -6.0 * c3d * x * z; dY[12][1] = -6.0 * c3d * y * z;
    dY[12][2] = c3d * (6.0 * zz - 3.0 * xx - 3.0 * yy);
    dY[13][0] = -c3c * (4.0 * zz - 3.0 * xx - yy); dY[13][1] = 2.0 * c3c * x * y;
    dY[13][2] = -8.0 * c3c * x * z;
    dY[14][0] = 2.0 * c3e * x * z; dY[14][1] = -2.0 * c3e * y * z; dY[14][2] = c3e * (xx - yy);
    dY[15][0] = -c3a * (3.0 * xx - 3.0 * yy); dY[15][1] = 6.0 * c3a * x * y; dY[15][2] = 0;
  }
}

// sum_k w_k grad Y_k(d) without materialising the 16 x 3 Jacobian.
template <typename T>
__device__ __forceinline__ void sh_grad_dir(int deg, T x, T y, T z, const T* w, T* gd) {
  const T c1 = (T) 0.4886025119029199;
  const T c2a = (T)1.0925484305920792, c2b = (T)0.31539156525252005, c2c = (T)0.5462742152960396;
  const T c3a = (T)0.5900435899266435, c3b = (T)2.890611442640554, c3c = (T)0.4570457994644658,
          c3d = (T)0.3731763325901154, c3e = (T)1.445305721320277;
  T gx = 0, gy = 0, gz = 0;
  if (deg >= 1) {
    gy -= c1 * w[1]; gz += c1 * w[2]; gx -= c1 * w[3];
  }
  if (deg >= 2) {
    gx += c2a * y * w[4]; gy += c2a * x * w[4];
    gy -= c2a * z * w[5]; gz -= c2a * y * w[5];
    gx -= (T)2 * c2b * x * w[6]; gy -= (T)2 * c2b * y * w[6]; gz += (T)4 * c2b * z * w[6];
    gx -= c2a * z * w[7]; gz -= c2a * x * w[7];
    gx += (T)2 * c2c * x * w[8]; gy -= (T)2 * c2c * y * w[8];
  }
  if (deg >= 3) {
    const T xx = x * x, yy = y * y, zz = z * z;
    gx -= (T)6 * c3a * x * y * w[9]; gy -= c3a * ((T)3 * xx - (T)3 * yy) * w[9];
    gx += c3b * y * z * w[10]; gy += c3b * x * z * w[10]; gz += c3b * x * y * w[10];
    gx += (T)2 * c3c * x * y * w[11]; gy -= c3c * ((T)4 * zz - xx - (T)3 * yy) * w[11];
    gz -= (T)8 * c3c * y * z * w[11];
    gx -= (T)6 * c3d * x * z * w[12]; gy -= (T)6 * c3d * y * z * w[12];
    gz += c3d * ((T)6 * zz - (T)3 * xx - (T)3 * yy) * w[12];
    gx -= c3c * ((T)4 * zz - (T)3 * xx - yy) * w[13]; gy += (T)2 * c3c * x * y * w[13];
    gz -= (T)8 * c3c * x * z * w[13];
    gx += (T)2 * c3e * x * z * w[14]; gy -= (T)2 * c3e * y * z * w[14]; gz += c3e * (xx - yy) * w[14];
    gx -= c3a * ((T)3 * xx - (T)3 * yy) * w[15]; gy += (T)6 * c3a * x * y * w[15];
  }
  gd[0] = gx; gd[1] = gy; gd[2] = gz;
}

// Unit view direction d = (mu - C) / |mu - C|, C = -R^T t; returns |mu - C|.
__device__ __forceinline__ double view_dir(const float* cam, const double* mu, double* d) {
  double v[3];
  for (int j = 0; j < 3; ++j) {
    const double Cj = -((double)cam[j] * cam[9] + (double)cam[3 + j] * cam[10] +
                        (double)cam[6 + j] * cam[11]);
    v[j] = mu[j] - Cj;
  }
  const double n = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  for (int j = 0; j < 3; ++j) d[j] = v[j] / n;
  return n;
}

struct Pre3DArgs {
  Cfg2 c;
  int32_t ewa_clamp, exact;
  int32_t sh_deg;   // -1: flat RGB `color`; 0..3: SH colour from `sh`
  int64_t N, view_stride;
  const float *mean, *scale, *quat, *freq, *phase, *color, *opacity, *sh;
  PreOut o;
  CamBlock cams;
};

#ifndef WIPES_PRE_BWD_TU  // forward kernels
// One (view, primitive) record from its loaded parameters. With have_prim the
// caller has already run project3_prim (once for all views of the primitive);
// the arithmetic is the same either way (the halves are independent).
template <bool EXACT>
__device__ __forceinline__ void pre3d_record(const Pre3DArgs& a, const float* cam, int64_t o,
                                             bool ok, const double* mu, const double* s,
                                             const double* q, const double* f, double phi,
                                             double cr, double cg, double cb, double al,
                                             bool have_prim, Proj3& P) {
  const Cfg2& c = a.c;
  int4 rect = make_int4(0, 0, 0, 0);
  int32_t cnt = 0;
  int flag = 0;
  uint32_t dk = 0;
  double conic[3] = {0, 0, 0}, ext[2] = {0, 0};
  double mux = 0, muy = 0, fpx = 0, fpy = 0, beta = 1.0;
  if (!ok) {
    flag = 5;
  } else {
    if (have_prim)
      project3_view(cam, c.W, c.H, a.ewa_clamp, mu, f, P);
    else
      project3(cam, c.W, c.H, a.ewa_clamp, mu, s, q, f, P);
    double x = P.p[0], y = P.p[1], z = P.p[2];
    double nz = cam[16], fz = cam[17];
    if (!(z >= nz && z <= fz)) {
      flag = 1;
    } else {
      double fx = cam[12], fy = cam[13], cx = cam[14], cy = cam[15];
      mux = (fx * (x / z)) + cx;
      muy = (fy * (y / z)) + cy;
      fpx = (z * P.g[0]) / fx;
      fpy = (z * P.g[1]) / fy;
      if (EXACT) {  // f' and beta of the exact z-marginal (no integer decision uses them)
        // sigma = M S3 Rv2^T, s22 = Rv2 S3 Rv2^T (Rv2 = third row of the view rotation)
        double t2[3];
        for (int k = 0; k < 3; ++k)
          t2[k] = s3at(P.S3, k, 0) * cam[6] + s3at(P.S3, k, 1) * cam[7] + s3at(P.S3, k, 2) * cam[8];
        const double sgx = P.M[0] * t2[0] + P.M[1] * t2[1] + P.M[2] * t2[2];
        const double sgy = P.M[3] * t2[0] + P.M[4] * t2[1] + P.M[5] * t2[2];
        const double s22 = cam[6] * t2[0] + cam[7] * t2[1] + cam[8] * t2[2];
        const double det2 = P.Sp[0] * P.Sp[2] - P.Sp[1] * P.Sp[1];  // undilated S2
        const double ux = (P.Sp[2] * sgx - P.Sp[1] * sgy) / det2;
        const double uy = (P.Sp[0] * sgy - P.Sp[1] * sgx) / det2;
        const double vv = s22 - (sgx * ux + sgy * uy);
        const double fhz = P.g[2] - P.j02 * fpx - P.j12 * fpy;
        fpx = fpx + fhz * ux;
        fpy = fpy + fhz * uy;
        beta = exp(-0.5 * fhz * fhz * vv);
      }
      float dz = (float)z;
      dk = orderable(dz);
      flag = finish2d(c, mux, muy, P.Sp[0] + c.diag, P.Sp[1], P.Sp[2] + c.diag, al, &rect,
                      &cnt, conic, ext);
    }
  }
  a.o.rect[o] = rect;
  a.o.count[o] = cnt;
  a.o.flag[o] = (uint8_t)flag;
  a.o.dkey[o] = dk;
  if (a.o.cull_flags) a.o.cull_flags[o] = (uint8_t)flag;
  if (flag == 0)
    write_record(a.o.rec + 4 * o, mux, muy, conic, al, fpx, fpy, phi, beta, cr, cg, cb, ext);
  else
    zero_record(a.o.rec + 4 * o);
}

__device__ __forceinline__ bool params_finite(const double* mu, const double* s, const double* q,
                                              const double* f, double phi, double al, double cr,
                                              double cg, double cb) {
  double qq = ((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]) + q[3] * q[3];
  return fin(mu[0]) && fin(mu[1]) && fin(mu[2]) && fin(s[0]) && fin(s[1]) && fin(s[2]) &&
         fin(q[0]) && fin(q[1]) && fin(q[2]) && fin(q[3]) && fin(f[0]) && fin(f[1]) &&
         fin(f[2]) && fin(phi) && fin(al) && fin(cr) && fin(cg) && fin(cb) && (qq > 0.0);
}

// One thread per (view, primitive) record.
template <bool EXACT, bool SH>
__global__ void __launch_bounds__(128, (EXACT || SH) ? 2 : WIPES_PRE3D_FWD_MINB) k_pre3d(const __grid_constant__ Pre3DArgs a) {
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid < 4) a.o.arrive[gid] = 0;
  if (gid >= (int64_t)a.cams.nv * a.N) return;
  // SH with shared parameters: view-minor order, so a primitive's
  // coefficients (48 floats) are read once from HBM for all its views
  const bool vminor = (SH || WIPES_PRE3D_VMINOR) && a.view_stride == 0;
  int vl = vminor ? (int)(gid % a.cams.nv) : (int)(gid / a.N);
  int64_t i = vminor ? gid / a.cams.nv : gid - (int64_t)vl * a.N;
  int v = a.cams.v0 + vl;
  int64_t o = (int64_t)v * a.N + i;
  int64_t pi = (int64_t)v * a.view_stride + i;
  const float* cam = a.cams.v[vl];
  double mu[3] = {a.mean[3 * pi], a.mean[3 * pi + 1], a.mean[3 * pi + 2]};
  double s[3] = {a.scale[3 * pi], a.scale[3 * pi + 1], a.scale[3 * pi + 2]};
  double q[4] = {a.quat[4 * pi], a.quat[4 * pi + 1], a.quat[4 * pi + 2], a.quat[4 * pi + 3]};
  double f[3] = {a.freq[3 * pi], a.freq[3 * pi + 1], a.freq[3 * pi + 2]};
  double phi = a.phase ? (double)a.phase[pi] : 0.0;
  double cr = 0.0, cg = 0.0, cb = 0.0;
  if (!SH) { cr = a.color[3 * pi]; cg = a.color[3 * pi + 1]; cb = a.color[3 * pi + 2]; }
  double al = a.opacity[pi];
  bool ok = params_finite(mu, s, q, f, phi, al, cr, cg, cb);
  if (SH && ok) {  // NEXT-3: view-dependent colour from SH
    double d[3], Y[16];
    view_dir(cam, mu, d);
    sh_basis(a.sh_deg, d[0], d[1], d[2], Y, nullptr);
    const int K = (a.sh_deg + 1) * (a.sh_deg + 1);
    const float* shp = a.sh + (int64_t)3 * K * pi;
    double rgb[3] = {0.5, 0.5, 0.5};
    for (int k = 0; k < K; ++k)
      for (int ch = 0; ch < 3; ++ch) rgb[ch] += Y[k] * (double)shp[3 * k + ch];
    cr = fmax(rgb[0], 0.0); cg = fmax(rgb[1], 0.0); cb = fmax(rgb[2], 0.0);
    ok = fin(rgb[0]) && fin(rgb[1]) && fin(rgb[2]);
  }
  Proj3 P;
  pre3d_record<EXACT>(a, cam, o, ok, mu, s, q, f, phi, cr, cg, cb, al, false, P);
}

#ifndef WIPES_PRE3D_LOOP
#define WIPES_PRE3D_LOOP 1  // shared parameters, flat colour: one thread per primitive
#endif
#ifndef WIPES_PRE3D_LOOP_MINB
#define WIPES_PRE3D_LOOP_MINB 4
#endif

// Shared parameters (view_stride 0), flat colour: one thread per primitive
// loads its parameters once, runs the view-independent half of the projection
// (quaternion normalisation, R, S3) once, and emits the records of all the
// launch's views in view order (record o = v N + i: coalesced per view).
template <bool EXACT>
__global__ void __launch_bounds__(128, WIPES_PRE3D_LOOP_MINB) k_pre3d_loop(const __grid_constant__ Pre3DArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 4) a.o.arrive[i] = 0;
  if (i >= a.N) return;
  double mu[3] = {a.mean[3 * i], a.mean[3 * i + 1], a.mean[3 * i + 2]};
  double s[3] = {a.scale[3 * i], a.scale[3 * i + 1], a.scale[3 * i + 2]};
  double q[4] = {a.quat[4 * i], a.quat[4 * i + 1], a.quat[4 * i + 2], a.quat[4 * i + 3]};
  double f[3] = {a.freq[3 * i], a.freq[3 * i + 1], a.freq[3 * i + 2]};
  const double phi = a.phase ? (double)a.phase[i] : 0.0;
  const double cr = a.color[3 * i], cg = a.color[3 * i + 1], cb = a.color[3 * i + 2];
  const double al = a.opacity[i];
  const bool ok = params_finite(mu, s, q, f, phi, al, cr, cg, cb);
  Proj3 P;
  if (ok) project3_prim(s, q, P);
  for (int vl = 0; vl < a.cams.nv; ++vl)
    pre3d_record<EXACT>(a, a.cams.v[vl], (int64_t)(a.cams.v0 + vl) * a.N + i, ok, mu, s, q, f,
                        phi, cr, cg, cb, al, true, P);
}

#endif

// ------------------------------------------------------------- backward ----
// conic -> covariance: G_Sigma = -A G_A A, G_A = [[ga, gb/2],[gb/2, gc]];
// returns (g_xx, g_xy (off-diagonal counted twice), g_yy).
__device__ __forceinline__ void conic_grad_to_cov(const double* A, double ga, double gb,
                                                  double gc, double* gs) {
  double a = A[0], b = A[1], c = A[2];
  double h = 0.5 * gb;
  // T1 = A Ga
  double t00 = a * ga + b * h, t01 = a * h + b * gc;
  double t10 = b * ga + c * h, t11 = b * h + c * gc;
  // T2 = -T1 A
  double s00 = -(t00 * a + t01 * b), s01 = -(t00 * b + t01 * c);
  double s10 = -(t10 * a + t11 * b), s11 = -(t10 * b + t11 * c);
  gs[0] = s00;
  gs[1] = s01 + s10;
  gs[2] = s11;
}

// Record gradients from the render kernel's 12 per-record moments (DESIGN.md
// §5): with hb = beta/2 and the FP64 conic (a, b, c), frequency f' and alpha,
//   dphi = -hb M6, df' = -hb (M7, M8), dmu' = A (M1, M2) + hb f' M6,
//   d(a, b, c) = (-M3/2, -M4, -M5/2), dalpha = M0 / alpha, dc = (M9, M10, M11).
__device__ __forceinline__ void moments_to_grads(const float* mom, const double* A, double fx,
                                                 double fy, double hb, double alpha,
                                                 double* g) {
  double m[kMoments];
  for (int k = 0; k < kMoments; ++k) m[k] = mom[k];
  g[RG_PHI] = -hb * m[6];
  g[RG_FX] = -hb * m[7];
  g[RG_FY] = -hb * m[8];
  g[RG_MUX] = A[0] * m[1] + A[1] * m[2] + hb * fx * m[6];
  g[RG_MUY] = A[1] * m[1] + A[2] * m[2] + hb * fy * m[6];
  g[RG_A] = -0.5 * m[3];
  g[RG_B] = -m[4];
  g[RG_C] = -0.5 * m[5];
  g[RG_BETA] = 0.0;
  g[RG_ALPHA] = m[0] / alpha;
  g[RG_CR] = m[9];
  g[RG_CG] = m[10];
  g[RG_CB] = m[11];
}

struct Bwd2DArgs {
  Cfg2 c;
  int32_t cov2;
  int64_t N;
  int64_t row0, row1;  // parameter rows [row0, row1) of this launch
  const float *cov, *freq, *opacity;
  const uint8_t* flag;
  const float* mom;
  wipes_grads g;
};

#ifdef WIPES_PRE_BWD_TU  // backward kernels: preprocess_bwd.cu builds them with FMA contraction
__global__ void __launch_bounds__(256) k_pre2d_bwd(Bwd2DArgs a) {
  int64_t i = a.row0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.row1) return;
  bool live = a.flag[i] == 0;
  double g[kRecGrads];
  for (int k = 0; k < kRecGrads; ++k) g[k] = 0.0;
  double A[3] = {0, 0, 0};
  double p0 = a.cov[3 * i], p1 = a.cov[3 * i + 1], p2 = a.cov[3 * i + 2];
  if (live) {
    double s[3];
    cov2d(a.cov2, p0, p1, p2, s);
    double sxx = s[0] + a.c.diag, sxy = s[1], syy = s[2] + a.c.diag;
    double det = sxx * syy - sxy * sxy;
    A[0] = syy / det; A[1] = -sxy / det; A[2] = sxx / det;
    moments_to_grads(a.mom + kMoments * i, A, a.freq[2 * i], a.freq[2 * i + 1], 0.5,
                     a.opacity[i], g);
  }
  if (a.g.mean) { a.g.mean[2 * i] = (float)g[RG_MUX]; a.g.mean[2 * i + 1] = (float)g[RG_MUY]; }
  if (a.g.freq) { a.g.freq[2 * i] = (float)g[RG_FX]; a.g.freq[2 * i + 1] = (float)g[RG_FY]; }
  if (a.g.phase) a.g.phase[i] = (float)g[RG_PHI];
  if (a.g.color) {
    a.g.color[3 * i] = (float)g[RG_CR];
    a.g.color[3 * i + 1] = (float)g[RG_CG];
    a.g.color[3 * i + 2] = (float)g[RG_CB];
  }
  if (a.g.opacity) a.g.opacity[i] = (float)g[RG_ALPHA];
  if (!a.g.cov) return;
  float* gc = a.g.cov + 3 * i;
  if (!live) { gc[0] = gc[1] = gc[2] = 0.f; return; }
  double gs[3];
  conic_grad_to_cov(A, g[RG_A], g[RG_B], g[RG_C], gs);
  if (a.cov2 == WIPES_COV2_SIGMA) {
    gc[0] = (float)gs[0]; gc[1] = (float)gs[1]; gc[2] = (float)gs[2];
  } else if (a.cov2 == WIPES_COV2_CHOLESKY) {
    gc[0] = (float)(2.0 * p0 * gs[0] + p1 * gs[1]);
    gc[1] = (float)(p0 * gs[1] + 2.0 * p1 * gs[2]);
    gc[2] = (float)(2.0 * p2 * gs[2]);
  } else {
    double cs = cos(p0), sn = sin(p0);
    double sx = p1, sy = p2;
    gc[0] = (float)((sx * sx - sy * sy) *
                    (-2.0 * cs * sn * gs[0] + (cs * cs - sn * sn) * gs[1] + 2.0 * cs * sn * gs[2]));
    gc[1] = (float)(2.0 * sx * (cs * cs * gs[0] + cs * sn * gs[1] + sn * sn * gs[2]));
    gc[2] = (float)(2.0 * sy * (sn * sn * gs[0] - cs * sn * gs[1] + cs * cs * gs[2]));
  }
}

struct Bwd3DArgs {
  Cfg2 c;
  int32_t ewa_clamp, accumulate;
  int64_t N, view_stride, nrows;
  int64_t row0;  // first (launch-local) parameter row: rows [row0, row0 + nrows)
  const float *mean, *scale, *quat, *freq;
  const float* opacity;
  const uint8_t* flag;
  const float* mom;
  const float* mom_beta;  // exact mode only
  const float* sh;        // SH colour mode only
  float* dc;              // SH: [B*N, 3] record colour gradients (k_pre3d_bwd -> k_sh_bwd)
  wipes_grads g;
  CamBlock cams;  // views [v0, v0 + nv) of this launch
};

// One thread per OUTPUT parameter row. With view_stride = 0 it sums the
// contributions of the launch's views in view order (deterministic); launches
// after the first (B > 128 views) add to the rows written before.
// EXACT adds the adjoint of the exact z-marginal (NEXT-1; R4):
// f' = f_hat_xy + f_hat_z u, u = S2^-1 sigma, beta = exp(-1/2 f_hat_z^2 v),
// v = Sigma_hat_zz - sigma.u, pulled back by hand onto f_hat, J (j02, j12)
// and the full 3x3 ray-space covariance Sigma_hat = M3 S3 M3^T.
template <bool EXACT>
__global__ void __launch_bounds__(128, WIPES_PRE3D_MINB) k_pre3d_bwd(const __grid_constant__ Bwd3DArgs a) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.nrows) return;
  const int64_t row = a.row0 + r;
  int v_lo, v_hi;
  int64_t i, pi;
  if (a.view_stride == 0) { v_lo = a.cams.v0; v_hi = a.cams.v0 + a.cams.nv; i = row; pi = row; }
  else {
    int vl = (int)(row / a.N);
    v_lo = a.cams.v0 + vl; v_hi = v_lo + 1; i = row - (int64_t)vl * a.N;
    pi = (int64_t)v_lo * a.view_stride + i;
  }
  double gmu[3] = {0, 0, 0}, gs_[3] = {0, 0, 0}, gq[4] = {0, 0, 0, 0}, gf[3] = {0, 0, 0};
  double gphi = 0, gcol[3] = {0, 0, 0}, gal = 0;
  double mu[3] = {a.mean[3 * pi], a.mean[3 * pi + 1], a.mean[3 * pi + 2]};
  double s[3] = {a.scale[3 * pi], a.scale[3 * pi + 1], a.scale[3 * pi + 2]};
  double q[4] = {a.quat[4 * pi], a.quat[4 * pi + 1], a.quat[4 * pi + 2], a.quat[4 * pi + 3]};
  double f[3] = {a.freq[3 * pi], a.freq[3 * pi + 1], a.freq[3 * pi + 2]};
  Proj3 P;
  bool have_prim = false;
  for (int v = v_lo; v < v_hi; ++v) {
    const int64_t o = (int64_t)v * a.N + i;
    if (a.flag[o] != 0) continue;
    const float* cam = a.cams.v[v - a.cams.v0];
    if (!have_prim || !WIPES_PRE3D_BWD_PRIM_ONCE) {  // the view-independent half once per row
      project3_prim<false>(s, q, P);
      have_prim = true;
    }
    project3_view<false>(cam, a.c.W, a.c.H, a.ewa_clamp, mu, f, P);
    double x = P.p[0], y = P.p[1], z = P.p[2];
    double fx = cam[12], fy = cam[13];
    const double rz = 1.0 / z, rz2 = rz * rz, rfx = 1.0 / fx, rfy = 1.0 / fy;
    double Rv[9];
    for (int k = 0; k < 9; ++k) Rv[k] = cam[k];
    // conic of the (diag-offset) Sigma' and the record gradients from moments
    double sxx = P.Sp[0] + a.c.diag, sxy = P.Sp[1], syy = P.Sp[2] + a.c.diag;
    double det = sxx * syy - sxy * sxy;
    const double rdet = 1.0 / det;
    double A[3] = {syy * rdet, -sxy * rdet, sxx * rdet};
    const double fhx = (z * P.g[0]) * rfx, fhy = (z * P.g[1]) * rfy;
    double fpx = fhx, fpy = fhy, hb = 0.5;
    // exact mode: sigma = (Sigma_hat_02, Sigma_hat_12), s22 = Sigma_hat_22
    double sg[2] = {0, 0}, s22 = 0, u[2] = {0, 0}, vv = 0, fhz = 0, beta = 1.0;
    double i00 = 0, i01 = 0, i11 = 0;
    if (EXACT) {
      double t2[3];
      for (int k = 0; k < 3; ++k)
        t2[k] = s3at(P.S3, k, 0) * Rv[6] + s3at(P.S3, k, 1) * Rv[7] + s3at(P.S3, k, 2) * Rv[8];
      sg[0] = P.M[0] * t2[0] + P.M[1] * t2[1] + P.M[2] * t2[2];
      sg[1] = P.M[3] * t2[0] + P.M[4] * t2[1] + P.M[5] * t2[2];
      s22 = Rv[6] * t2[0] + Rv[7] * t2[1] + Rv[8] * t2[2];
      const double rd2 = 1.0 / (P.Sp[0] * P.Sp[2] - P.Sp[1] * P.Sp[1]);  // undilated S2
      i00 = P.Sp[2] * rd2; i01 = -P.Sp[1] * rd2; i11 = P.Sp[0] * rd2;
      u[0] = i00 * sg[0] + i01 * sg[1];
      u[1] = i01 * sg[0] + i11 * sg[1];
      vv = s22 - (sg[0] * u[0] + sg[1] * u[1]);
      fhz = P.g[2] - P.j02 * fhx - P.j12 * fhy;
      fpx = fhx + fhz * u[0];
      fpy = fhy + fhz * u[1];
      beta = exp(-0.5 * fhz * fhz * vv);
      hb = 0.5 * beta;
    }
    double g[kRecGrads];
    moments_to_grads(a.mom + kMoments * o, A, fpx, fpy, hb, a.opacity[pi], g);
    if (a.dc) {
      a.dc[3 * o] = (float)g[RG_CR]; a.dc[3 * o + 1] = (float)g[RG_CG];
      a.dc[3 * o + 2] = (float)g[RG_CB];
    }
    gphi += g[RG_PHI];
    gcol[0] += g[RG_CR]; gcol[1] += g[RG_CG]; gcol[2] += g[RG_CB];
    gal += g[RG_ALPHA];
    double gFX = g[RG_FX], gFY = g[RG_FY];  // -> dL/df_hat_x, dL/df_hat_y
    double E[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // exact adjoint on Sigma_hat
    double dj02x = 0, dj12x = 0;
    if (EXACT) {
      const double gq = 0.5 * (double)a.mom_beta[o] * beta;  // dL/d(exponent of beta)
      const double g_fhz = gq * (-fhz * vv) + g[RG_FX] * u[0] + g[RG_FY] * u[1];
      const double g_v = gq * (-0.5 * fhz * fhz);
      const double gu0 = fhz * g[RG_FX] - g_v * sg[0], gu1 = fhz * g[RG_FY] - g_v * sg[1];
      const double w0 = i00 * gu0 + i01 * gu1, w1 = i01 * gu0 + i11 * gu1;
      E[0][0] = -w0 * u[0];
      E[0][1] = E[1][0] = -0.5 * (w0 * u[1] + w1 * u[0]);
      E[1][1] = -w1 * u[1];
      E[0][2] = E[2][0] = 0.5 * (w0 - g_v * u[0]);
      E[1][2] = E[2][1] = 0.5 * (w1 - g_v * u[1]);
      E[2][2] = g_v;
      gFX -= g_fhz * P.j02;
      gFY -= g_fhz * P.j12;
      dj02x = -g_fhz * fhx;
      dj12x = -g_fhz * fhy;
      for (int k = 0; k < 3; ++k) gf[k] += Rv[6 + k] * g_fhz;
    }
    double dp[3] = {0, 0, 0};
    dp[0] += g[RG_MUX] * fx * rz;
    dp[1] += g[RG_MUY] * fy * rz;
    dp[2] += -g[RG_MUX] * fx * x * rz2 - g[RG_MUY] * fy * y * rz2;
    dp[2] += gFX * P.g[0] * rfx + gFY * P.g[1] * rfy;
    double dg0 = gFX * z * rfx, dg1 = gFY * z * rfy;
    for (int k = 0; k < 3; ++k) gf[k] += Rv[k] * dg0 + Rv[3 + k] * dg1;
    double gsv[3];
    conic_grad_to_cov(A, g[RG_A], g[RG_B], g[RG_C], gsv);
    constexpr int NR = EXACT ? 3 : 2;  // rows of M3 = [M; Rv row 2] that carry gradient
    const double GS[3][3] = {{gsv[0] + E[0][0], 0.5 * gsv[1] + E[0][1], E[0][2]},
                             {0.5 * gsv[1] + E[1][0], gsv[2] + E[1][1], E[1][2]},
                             {E[2][0], E[2][1], E[2][2]}};
    const double M[3][3] = {{P.M[0], P.M[1], P.M[2]}, {P.M[3], P.M[4], P.M[5]},
                            {Rv[6], Rv[7], Rv[8]}};
    double GM[3][3];
    for (int r = 0; r < NR; ++r)
      for (int cc = 0; cc < 3; ++cc) {
        double acc = 0.0;
        for (int k = 0; k < NR; ++k) acc += GS[r][k] * M[k][cc];
        GM[r][cc] = acc;
      }
    double dM[2][3];
    for (int r = 0; r < 2; ++r)
      for (int cc = 0; cc < 3; ++cc) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += GM[r][k] * s3at(P.S3, k, cc);
        dM[r][cc] = 2.0 * acc;
      }
    double dS3[3][3];
    for (int r = 0; r < 3; ++r)
      for (int cc = 0; cc < 3; ++cc) {
        double acc = 0.0;
        for (int k = 0; k < NR; ++k) acc += M[k][r] * GM[k][cc];
        dS3[r][cc] = acc;
      }
    double dj00 = dM[0][0] * Rv[0] + dM[0][1] * Rv[1] + dM[0][2] * Rv[2];
    double dj02 = dM[0][0] * Rv[6] + dM[0][1] * Rv[7] + dM[0][2] * Rv[8] + dj02x;
    double dj11 = dM[1][0] * Rv[3] + dM[1][1] * Rv[4] + dM[1][2] * Rv[5];
    double dj12 = dM[1][0] * Rv[6] + dM[1][1] * Rv[7] + dM[1][2] * Rv[8] + dj12x;
    dp[2] += dj00 * (-fx * rz2) + dj11 * (-fy * rz2);
    double dtx_dx = P.clx ? 0.0 : rz, dtx_dz = P.clx ? 0.0 : -x * rz2;
    double dty_dy = P.cly ? 0.0 : rz, dty_dz = P.cly ? 0.0 : -y * rz2;
    dp[0] += dj02 * (-(fx * rz) * dtx_dx);
    dp[2] += dj02 * (fx * P.thx * rz2 - (fx * rz) * dtx_dz);
    dp[1] += dj12 * (-(fy * rz) * dty_dy);
    dp[2] += dj12 * (fy * P.thy * rz2 - (fy * rz) * dty_dz);
    for (int k = 0; k < 3; ++k) gmu[k] += Rv[k] * dp[0] + Rv[3 + k] * dp[1] + Rv[6 + k] * dp[2];
    const double* R = P.Rq;
    double dRq[9];
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) {
        double acc = 0.0;
        for (int b = 0; b < 3; ++b) acc += dS3[r][b] * R[3 * b + k];
        dRq[3 * r + k] = 2.0 * acc * s[k] * s[k];
      }
    for (int k = 0; k < 3; ++k) {
      double Wkk = 0.0;
      for (int r = 0; r < 3; ++r)
        for (int b = 0; b < 3; ++b) Wkk += R[3 * r + k] * dS3[r][b] * R[3 * b + k];
      gs_[k] += 2.0 * s[k] * Wkk;
    }
    double w = P.qn[0], qx = P.qn[1], qy = P.qn[2], qz = P.qn[3];
    double dqn[4];
    dqn[0] = dRq[1] * (-2 * qz) + dRq[2] * (2 * qy) + dRq[3] * (2 * qz) + dRq[5] * (-2 * qx) +
             dRq[6] * (-2 * qy) + dRq[7] * (2 * qx);
    dqn[1] = dRq[1] * (2 * qy) + dRq[2] * (2 * qz) + dRq[3] * (2 * qy) + dRq[4] * (-4 * qx) +
             dRq[5] * (-2 * w) + dRq[6] * (2 * qz) + dRq[7] * (2 * w) + dRq[8] * (-4 * qx);
    dqn[2] = dRq[0] * (-4 * qy) + dRq[1] * (2 * qx) + dRq[2] * (2 * w) + dRq[3] * (2 * qx) +
             dRq[5] * (2 * qz) + dRq[6] * (-2 * w) + dRq[7] * (2 * qz) + dRq[8] * (-4 * qy);
    dqn[3] = dRq[0] * (-4 * qz) + dRq[1] * (-2 * w) + dRq[2] * (2 * qx) + dRq[3] * (2 * w) +
             dRq[4] * (-4 * qz) + dRq[5] * (2 * qy) + dRq[6] * (2 * qx) + dRq[7] * (2 * qy);
    double dot = dqn[0] * P.qn[0] + dqn[1] * P.qn[1] + dqn[2] * P.qn[2] + dqn[3] * P.qn[3];
    const double rq = 1.0 / P.qnorm;
    for (int k = 0; k < 4; ++k) gq[k] += (dqn[k] - P.qn[k] * dot) * rq;
  }
  auto put = [&](float* dst, double v) { *dst = a.accumulate ? *dst + (float)v : (float)v; };
  if (a.g.mean) for (int k = 0; k < 3; ++k) put(&a.g.mean[3 * pi + k], gmu[k]);
  if (a.g.scale) for (int k = 0; k < 3; ++k) put(&a.g.scale[3 * pi + k], gs_[k]);
  if (a.g.quat) for (int k = 0; k < 4; ++k) put(&a.g.quat[4 * pi + k], gq[k]);
  if (a.g.freq) for (int k = 0; k < 3; ++k) put(&a.g.freq[3 * pi + k], gf[k]);
  if (a.g.phase) put(&a.g.phase[pi], gphi);
  if (a.g.color) for (int k = 0; k < 3; ++k) put(&a.g.color[3 * pi + k], gcol[k]);
  if (a.g.opacity) put(&a.g.opacity[pi], gal);
}

// Exact-mode (NEXT-1) backward: the record gradients (from the 12 moments and
// the beta moment) are pulled back through the exact projection by forward-mode
// differentiation of exact_rec: one dual-number pass per parameter direction
// (mu, s, q, f: 13), each giving the column J[:, k] of the 8-output Jacobian;
// phase, colour and opacity pass straight through the record.
__global__ void __launch_bounds__(128) k_pre3d_bwd_exact(const __grid_constant__ Bwd3DArgs a) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= a.nrows) return;
  const int64_t row = a.row0 + r;
  int v_lo, v_hi;
  int64_t i, pi;
  if (a.view_stride == 0) { v_lo = a.cams.v0; v_hi = a.cams.v0 + a.cams.nv; i = row; pi = row; }
  else {
    int vl = (int)(row / a.N);
    v_lo = a.cams.v0 + vl; v_hi = v_lo + 1; i = row - (int64_t)vl * a.N;
    pi = (int64_t)v_lo * a.view_stride + i;
  }
  double x0[13] = {a.mean[3 * pi], a.mean[3 * pi + 1], a.mean[3 * pi + 2],
                   a.scale[3 * pi], a.scale[3 * pi + 1], a.scale[3 * pi + 2],
                   a.quat[4 * pi], a.quat[4 * pi + 1], a.quat[4 * pi + 2], a.quat[4 * pi + 3],
                   a.freq[3 * pi], a.freq[3 * pi + 1], a.freq[3 * pi + 2]};
  double gx[13];
  for (int k = 0; k < 13; ++k) gx[k] = 0.0;
  double gphi = 0, gcol[3] = {0, 0, 0}, gal = 0;
  for (int v = v_lo; v < v_hi; ++v) {
    const int64_t o = (int64_t)v * a.N + i;
    if (a.flag[o] != 0) continue;
    const float* cam = a.cams.v[v - a.cams.v0];
    double r8[8];
    exact_rec<double>(cam, a.c.W, a.c.H, a.ewa_clamp, a.c.diag, x0, x0 + 3, x0 + 6, x0 + 10, r8);
    const double A[3] = {r8[2], r8[3], r8[4]};
    double g[kRecGrads];
    moments_to_grads(a.mom + kMoments * o, A, r8[5], r8[6], 0.5 * r8[7], a.opacity[pi], g);
    if (a.dc) {
      a.dc[3 * o] = (float)g[RG_CR]; a.dc[3 * o + 1] = (float)g[RG_CG];
      a.dc[3 * o + 2] = (float)g[RG_CB];
    }
    gphi += g[RG_PHI];
    gcol[0] += g[RG_CR]; gcol[1] += g[RG_CG]; gcol[2] += g[RG_CB];
    gal += g[RG_ALPHA];
    const double gr[8] = {g[RG_MUX], g[RG_MUY], g[RG_A], g[RG_B], g[RG_C],
                          g[RG_FX],  g[RG_FY],  0.5 * (double)a.mom_beta[o]};
#pragma unroll 1
    for (int k = 0; k < 13; ++k) {
      Dual xd[13];
      for (int j = 0; j < 13; ++j) xd[j] = {x0[j], j == k ? 1.0 : 0.0};
      Dual out[8];
      exact_rec<Dual>(cam, a.c.W, a.c.H, a.ewa_clamp, a.c.diag, xd, xd + 3, xd + 6, xd + 10, out);
      double acc = 0.0;
      for (int r = 0; r < 8; ++r) acc += gr[r] * out[r].d;
      gx[k] += acc;
    }
  }
  auto put = [&](float* dst, double v) { *dst = a.accumulate ? *dst + (float)v : (float)v; };
  if (a.g.mean) for (int k = 0; k < 3; ++k) put(&a.g.mean[3 * pi + k], gx[k]);
  if (a.g.scale) for (int k = 0; k < 3; ++k) put(&a.g.scale[3 * pi + k], gx[3 + k]);
  if (a.g.quat) for (int k = 0; k < 4; ++k) put(&a.g.quat[4 * pi + k], gx[6 + k]);
  if (a.g.freq) for (int k = 0; k < 3; ++k) put(&a.g.freq[3 * pi + k], gx[10 + k]);
  if (a.g.phase) put(&a.g.phase[pi], gphi);
  if (a.g.color) for (int k = 0; k < 3; ++k) put(&a.g.color[3 * pi + k], gcol[k]);
  if (a.g.opacity) put(&a.g.opacity[pi], gal);
}

// NEXT-3 backward of the SH colour: the record colour gradient dc = (M9, M10,
// M11) of each (view, primitive) gives dL/dsh_k = Y_k(d) dc (zero for a
// clamped channel) and, through the view direction d = (mu - C)/|mu - C|,
// dL/dmu += (I - d d^T)/|mu - C| sum_k (sh_k . dc) grad Y_k(d), ADDED to the
// mean gradient written by k_pre3d_bwd just before on the same stream.
#ifndef WIPES_SH_MINB
#define WIPES_SH_MINB 4
#endif
// GV lanes share one parameter row (lane l takes views l, l + GV, ...) and
// their partial sums are combined with xor shuffles in a fixed order.
template <int DEG, int GV>
__global__ void __launch_bounds__(128, WIPES_SH_MINB) k_sh_bwd(const __grid_constant__ Bwd3DArgs a) {
  constexpr int K = (DEG + 1) * (DEG + 1);
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t lrow = gid / GV;
  const int64_t row = a.row0 + lrow;
  const int gl = (int)(gid % GV);
  const bool active = lrow < a.nrows;  // whole groups only: no early return (shuffles)
  int v_lo = 0, v_hi = 0;
  int64_t i = 0, pi = 0;
  if (active) {
    if (a.view_stride == 0) { v_lo = a.cams.v0; v_hi = a.cams.v0 + a.cams.nv; i = row; pi = row; }
    else {
      int vl = (int)(row / a.N);
      v_lo = a.cams.v0 + vl; v_hi = v_lo + 1; i = row - (int64_t)vl * a.N;
      pi = (int64_t)v_lo * a.view_stride + i;
    }
  }
  double mu[3] = {0, 0, 0};
  if (active) { mu[0] = a.mean[3 * pi]; mu[1] = a.mean[3 * pi + 1]; mu[2] = a.mean[3 * pi + 2]; }
  const float* sh = a.sh + (int64_t)3 * K * pi;  // re-read per view (L1-resident)
  float gsh[3 * K];
#pragma unroll
  for (int k = 0; k < 3 * K; ++k) gsh[k] = 0.f;
  double gmu[3] = {0, 0, 0};
  for (int v = v_lo + gl; v < v_hi; v += GV) {
    const int64_t o = (int64_t)v * a.N + i;
    if (a.flag[o] != 0) continue;
    const float* cam = a.cams.v[v - a.cams.v0];
    double d[3], Y[16];
    const double n = view_dir(cam, mu, d);
    sh_basis(DEG, d[0], d[1], d[2], Y, nullptr);
    double dc[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      double c = 0.5;
#pragma unroll
      for (int k = 0; k < K; ++k) c += Y[k] * (double)sh[3 * k + ch];
      dc[ch] = c < 0.0 ? 0.0 : (double)a.dc[3 * o + ch];
    }
    // gradient path in FP32 (the clamp decision above is the forward's FP64 one)
    const float dcf[3] = {(float)dc[0], (float)dc[1], (float)dc[2]};
    float w[16];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      w[k] = sh[3 * k] * dcf[0] + sh[3 * k + 1] * dcf[1] + sh[3 * k + 2] * dcf[2];
      const float yk = (float)Y[k];
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) gsh[3 * k + ch] += yk * dcf[ch];
    }
    float gdf[3];
    sh_grad_dir<float>(DEG, (float)d[0], (float)d[1], (float)d[2], w, gdf);
    const double gd[3] = {gdf[0], gdf[1], gdf[2]};
    const double dd = d[0] * gd[0] + d[1] * gd[1] + d[2] * gd[2];
#pragma unroll
    for (int j = 0; j < 3; ++j) gmu[j] += (gd[j] - d[j] * dd) / n;
  }
  if (GV > 1) {
#pragma unroll
    for (int off = 1; off < GV; off <<= 1) {
#pragma unroll
      for (int k = 0; k < 3 * K; ++k) gsh[k] += __shfl_xor_sync(0xffffffffu, gsh[k], off);
#pragma unroll
      for (int j = 0; j < 3; ++j) gmu[j] += __shfl_xor_sync(0xffffffffu, gmu[j], off);
    }
  }
  if (!active || gl != 0) return;
  if (a.g.sh) {
    float* dst = a.g.sh + (int64_t)3 * K * pi;
#pragma unroll
    for (int k = 0; k < 3 * K; ++k) dst[k] = a.accumulate ? dst[k] + gsh[k] : gsh[k];
  }
  if (a.g.mean)
    for (int j = 0; j < 3; ++j) a.g.mean[3 * pi + j] += (float)gmu[j];
}

template <int DEG>
void launch_sh_bwd(const Bwd3DArgs& a, int views_per_row, cudaStream_t s) {
  auto go = [&](auto k, int gv) {
    const int64_t threads = a.nrows * gv;
    k<<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(a);
  };
  if (views_per_row >= 16) go(k_sh_bwd<DEG, 16>, 16);
  else if (views_per_row >= 8) go(k_sh_bwd<DEG, 8>, 8);
  else if (views_per_row >= 4) go(k_sh_bwd<DEG, 4>, 4);
  else if (views_per_row >= 2) go(k_sh_bwd<DEG, 2>, 2);
  else go(k_sh_bwd<DEG, 1>, 1);
}

#endif

Cfg2 make_cfg2(const wipes_config& c, const Layout& L) {
  Cfg2 r;
  r.W = c.width; r.H = c.height; r.tile = c.tile; r.GX = L.GX; r.GY = L.GY;
  r.extent = c.extent; r.alpha_blend = c.blend == WIPES_BLEND_ALPHA;
  r.row_mod = c.row_mod; r.row_rem = c.row_rem;
  r.alpha_min = (double)c.alpha_min;
  r.det_min = (double)c.det_min;
  r.diag = (double)c.cov_eps + (double)c.dilation;
  return r;
}

PreOut make_out(const Layout& L, char* ws, uint8_t* cull) {
  PreOut o;
  o.rect = (int4*)(ws + L.rect);
  o.count = (int32_t*)(ws + L.count);
  o.flag = (uint8_t*)(ws + L.flag);
  o.dkey = (uint32_t*)(ws + L.dkey);
  o.rec = (float4*)(ws + L.rec);
  o.cull_flags = cull;
  o.arrive = ((WsHeader*)(ws + L.hdr))->arrive;
  return o;
}

void fill_cams(CamBlock& cb, const wipes_camera* cams, int v0, int nv) {
  cb.v0 = v0; cb.nv = nv;
  for (int k = 0; k < nv; ++k) {
    const wipes_camera& c = cams[v0 + k];
    for (int j = 0; j < 9; ++j) cb.v[k][j] = c.R[j];
    for (int j = 0; j < 3; ++j) cb.v[k][9 + j] = c.t[j];
    cb.v[k][12] = c.fx; cb.v[k][13] = c.fy; cb.v[k][14] = c.cx; cb.v[k][15] = c.cy;
    cb.v[k][16] = c.near_z; cb.v[k][17] = c.far_z;
  }
}

}  // namespace

#ifndef WIPES_PRE_BWD_TU  // forward launchers
cudaError_t launch_preprocess2d(const wipes_config& c, const wipes_params& p, const Layout& L,
                                char* ws, uint8_t* cull_flags, cudaStream_t s) {
  if (L.N == 0) return cudaSuccess;
  Pre2DArgs a;
  a.c = make_cfg2(c, L);
  a.cov2 = c.cov2;
  a.N = L.N;
  a.mean = p.mean; a.cov = p.cov; a.freq = p.freq; a.phase = p.phase; a.color = p.color;
  a.opacity = p.opacity; a.depth = p.depth;
  a.o = make_out(L, ws, cull_flags);
  launch_begin(K_PRE2D, s);
  k_pre2d<<<(unsigned)((L.N + 255) / 256), 256, 0, s>>>(a);
  launch_end(K_PRE2D, s);
  return cudaGetLastError();
}

cudaError_t launch_preprocess3d(const wipes_config& c, const wipes_params& p, const Layout& L,
                                const wipes_camera* cams, char* ws, uint8_t* cull_flags,
                                cudaStream_t s) {
  if (L.N == 0) return cudaSuccess;
  static thread_local Pre3DArgs a;  // ~9 KB: keep off the host stack
  a.c = make_cfg2(c, L);
  a.ewa_clamp = c.ewa_clamp;
  a.exact = L.exact;
  a.sh_deg = c.color_mode == WIPES_COLOR_SH ? c.sh_degree : -1;
  a.sh = p.sh;
  a.N = L.N;
  a.view_stride = p.view_stride;
  a.mean = p.mean; a.scale = p.scale; a.quat = p.quat; a.freq = p.freq; a.phase = p.phase;
  a.color = p.color; a.opacity = p.opacity;
  a.o = make_out(L, ws, cull_flags);
  for (int v0 = 0; v0 < L.B; v0 += WIPES_MAX_CAMERAS_PER_LAUNCH) {
    int nv = L.B - v0 < WIPES_MAX_CAMERAS_PER_LAUNCH ? L.B - v0 : WIPES_MAX_CAMERAS_PER_LAUNCH;
    fill_cams(a.cams, cams, v0, nv);
    int64_t n = (int64_t)nv * L.N;
    launch_begin(K_PRE3D, s);
    const unsigned gr = (unsigned)((n + 127) / 128);
    if (WIPES_PRE3D_LOOP && a.sh_deg < 0 && a.view_stride == 0)
      (a.exact ? k_pre3d_loop<true> : k_pre3d_loop<false>)<<<(unsigned)((L.N + 127) / 128), 128, 0, s>>>(a);
    else if (a.sh_deg >= 0)
      (a.exact ? k_pre3d<true, true> : k_pre3d<false, true>)<<<gr, 128, 0, s>>>(a);
    else
      (a.exact ? k_pre3d<true, false> : k_pre3d<false, false>)<<<gr, 128, 0, s>>>(a);
    launch_end(K_PRE3D, s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

#endif

#ifdef WIPES_PRE_BWD_TU  // backward launchers
cudaError_t launch_preprocess2d_bwd(const wipes_config& c, const wipes_params& p,
                                    const Layout& L, char* ws, const wipes_grads& g,
                                    cudaStream_t s, int64_t row0, int64_t row1) {
  if (row1 < 0 || row1 > L.N) row1 = L.N;
  if (L.N == 0 || row1 <= row0) return cudaSuccess;
  Bwd2DArgs a;
  a.row0 = row0;
  a.row1 = row1;
  a.c = make_cfg2(c, L);
  a.cov2 = c.cov2;
  a.N = L.N;
  a.cov = p.cov;
  a.freq = p.freq;
  a.opacity = p.opacity;
  a.flag = (const uint8_t*)(ws + L.flag);
  a.mom = (const float*)(ws + L.rgrad);
  a.g = g;
  launch_begin(K_PRE2D_BWD, s);
  k_pre2d_bwd<<<(unsigned)((row1 - row0 + 255) / 256), 256, 0, s>>>(a);
  launch_end(K_PRE2D_BWD, s);
  return cudaGetLastError();
}

cudaError_t launch_preprocess3d_bwd(const wipes_config& c, const wipes_params& p,
                                    const Layout& L, const wipes_camera* cams, char* ws,
                                    const wipes_grads& g, cudaStream_t s, int64_t row0,
                                    int64_t row1) {
  const int64_t rows = p.view_stride == 0 ? L.N : (int64_t)L.B * L.N;
  if (row1 < 0 || row1 > rows) row1 = rows;
  if (L.N == 0 || row1 <= row0) return cudaSuccess;
  static thread_local Bwd3DArgs a;  // ~9 KB: keep off the host stack
  a.c = make_cfg2(c, L);
  a.ewa_clamp = c.ewa_clamp;
  a.N = L.N;
  a.view_stride = p.view_stride;
  a.mean = p.mean; a.scale = p.scale; a.quat = p.quat; a.freq = p.freq;
  a.opacity = p.opacity;
  a.flag = (const uint8_t*)(ws + L.flag);
  a.mom = (const float*)(ws + L.rgrad);
  a.mom_beta = L.exact ? (const float*)(ws + L.rbeta) : nullptr;
  a.sh = p.sh;
  a.g = g;
  const bool use_sh = c.color_mode == WIPES_COLOR_SH;
  a.dc = use_sh ? (float*)(ws + L.rdc) : nullptr;
  if (use_sh) a.g.color = nullptr;  // the record colour is not a parameter in SH mode
  for (int v0 = 0; v0 < L.B; v0 += WIPES_MAX_CAMERAS_PER_LAUNCH) {
    int nv = L.B - v0 < WIPES_MAX_CAMERAS_PER_LAUNCH ? L.B - v0 : WIPES_MAX_CAMERAS_PER_LAUNCH;
    fill_cams(a.cams, cams, v0, nv);
    a.accumulate = (p.view_stride == 0 && v0 > 0) ? 1 : 0;
    if (p.view_stride == 0) {  // primitive rows, every view chunk
      a.row0 = row0;
      a.nrows = row1 - row0;
    } else {  // (view, primitive) rows of this chunk's views within [row0, row1)
      const int64_t c0 = (int64_t)v0 * L.N, c1 = (int64_t)(v0 + nv) * L.N;
      const int64_t lo = row0 > c0 ? row0 : c0, hi = row1 < c1 ? row1 : c1;
      if (hi <= lo) continue;
      a.row0 = lo - c0;
      a.nrows = hi - lo;
    }
    launch_begin(K_PRE3D_BWD, s);
    static const bool dual = getenv("WIPES_EXACT_DUAL") != nullptr;
    if (L.exact && dual)  // forward-mode (dual number) cross-check of the hand adjoint
      k_pre3d_bwd_exact<<<(unsigned)((a.nrows + 127) / 128), 128, 0, s>>>(a);
    else if (L.exact)
      k_pre3d_bwd<true><<<(unsigned)((a.nrows + 127) / 128), 128, 0, s>>>(a);
    else
      k_pre3d_bwd<false><<<(unsigned)((a.nrows + 127) / 128), 128, 0, s>>>(a);
    launch_end(K_PRE3D_BWD, s);
    if (use_sh) {
      launch_begin(K_SH_BWD, s);
      const int vpr = p.view_stride == 0 ? nv : 1;  // views summed per parameter row
      switch (c.sh_degree) {
        case 0: launch_sh_bwd<0>(a, vpr, s); break;
        case 1: launch_sh_bwd<1>(a, vpr, s); break;
        case 2: launch_sh_bwd<2>(a, vpr, s); break;
        default: launch_sh_bwd<3>(a, vpr, s); break;
      }
      launch_end(K_SH_BWD, s);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

#endif

}  // namespace wipes
