// ============================================================================
// oracle/oracle.cpp — WIPES reference ORACLE (test infrastructure ONLY)
// ============================================================================
// This file is TEST INFRASTRUCTURE. Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it. The product
// path (paper_2508_12615_b200/) never links, imports or executes it, and it
// shares no code, header, table or constant generator with the CUDA path.
//
// What it computes, in double precision, plainly and slowly:
//   * the wavelet primitive W = G * 1/2 [1 + beta cos(f.(x-mu) + phi)]
//       PAPER.md:187-191 (Sec. 4.1, Eq. 6); beta/phi generalisation = DESIGN.md R1
//   * 2D covariance constructions (Sigma / Cholesky / RS)   PAPER.md:299 (Sec. 5.1)
//   * 3D -> 2D projection: Sigma' = upper-left 2x2 of J W Sigma W^T J^T
//       PAPER.md:116-122 (Sec. 3.1, Eq. 2); frequency transform PAPER.md:212
//       (Sec. 4.1) read contravariantly (R3); Eq. 7
//   * weighted-sum image formation C = sum_i c_i alpha_i W'_i
//       PAPER.md:169-174 (Sec. 3.2, Eq. 4) with G' -> W'
//   * front-to-back alpha blending C = sum_i c_i a_i prod_{j<i}(1-a_j)
//       PAPER.md:124-129 (Sec. 3.1, Eq. 3) with G' -> W'
//   * analytic gradients of all primitive parameters ("explicit gradients for
//       all parameters", Sec. 1) — chain rule of the above.
//   * the integer binning artefacts (tile rects, counts, (tile|depth) keys,
//       stable sort, per-tile CSR ranges) by closed form + std::stable_sort.
// Rendering is BRUTE FORCE: every pixel against every primitive, no tiling.
// The truncation rules (alpha_min skip, alpha_max clamp, T_min stop, extent
// cull) are per-(pixel, primitive) predicates (R7-R10).
//
// Floating-point: compiled with -O2 -ffp-contract=off -fno-fast-math. The
// integer-deciding preprocess follows the pinned expression order written in
// DESIGN.md section "Pinned preprocess arithmetic" (spec text, not code).
//
// Parity status: every function here is pinned by tests/test_oracle_*.py
// (closed forms, invariants, finite differences, FFT, brute-force compositing)
// EXCEPT the exact z-integration mode which is pinned by 1-D quadrature.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {

// ---- oracle's own configuration (independent of include/wipes.h) ----------
struct ora_cfg {
  int32_t width, height, tile;
  int32_t prim3d;       // 0: 2D primitives on the image plane; 1: 3D + camera
  int32_t alpha_blend;  // 0: weighted sum (Eq. 4); 1: alpha blending (Eq. 3)
  int32_t cov2;         // 2D covariance: 0 = Sigma given, 1 = Cholesky, 2 = RS
  int32_t extent;       // 0 = opacity-aware AABB, 1 = 3-sigma square
  int32_t ewa_clamp;    // 1 = clamp x/z, y/z at 1.3 x half-FOV inside J
  int32_t exact_proj;   // 0 = paper Eq. 7 (beta = 1); 1 = exact z-integral
  int32_t use_rect;     // 1 = also require "pixel's tile in rect" (opacity mode)
  double alpha_min, alpha_max, T_min;
  double dilation, cov_eps, det_min;
  double bg[3];
  int32_t color_per_view;  // 1: color is [B*N,3] per (view, primitive) (SH colours)
};

struct ora_cam {
  double R[9];  // world -> camera rotation, row-major (x_c = R x_w + t)
  double t[3];
  double fx, fy, cx, cy;
  double near_z, far_z;
};

// projected-record layout (doubles), one row of ORA_P per (view, primitive)
enum {
  P_MUX = 0, P_MUY, P_A, P_B, P_C, P_FX, P_FY, P_PHI, P_BETA, P_CR, P_CG, P_CB,
  P_ALPHA, P_DEPTH, P_SXX, P_SXY, P_SYY, P_RMARGIN, P_RX, P_RY, ORA_P
};
// record-gradient layout (doubles), one row of ORA_G per (view, primitive):
// d/d(mu'x, mu'y, conic a, conic b (off-diagonal value), conic c, f'x, f'y,
//     phi, beta, c_r, c_g, c_b, alpha)
enum {
  G_MUX = 0, G_MUY, G_A, G_B, G_C, G_FX, G_FY, G_PHI, G_BETA, G_CR, G_CG, G_CB,
  G_ALPHA, ORA_G
};

int ora_record_width(void) { return ORA_P; }
int ora_grad_width(void) { return ORA_G; }

// ---------------------------------------------------------------------------
// Kernel evaluation, PAPER.md:107-109 (Eq. 1) and 187-191 (Eq. 6).
// ---------------------------------------------------------------------------
double ora_eval_gaussian2(const double* conic, double dx, double dy) {
  double q = conic[0] * dx * dx + 2.0 * conic[1] * dx * dy + conic[2] * dy * dy;
  return std::exp(-0.5 * q);
}

double ora_eval_wavelet2(const double* conic, const double* f, double phi,
                         double beta, double dx, double dy) {
  double G = ora_eval_gaussian2(conic, dx, dy);
  double theta = f[0] * dx + f[1] * dy + phi;
  return G * 0.5 * (1.0 + beta * std::cos(theta));
}

// 3-D forms (Eq. 1 / Eq. 6 in world space) used by the z-integration pins.
double ora_eval_wavelet3(const double* inv_cov /*3x3 row-major*/,
                         const double* f, double phi, double beta,
                         const double* d) {
  double q = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) q += d[i] * inv_cov[3 * i + j] * d[j];
  double theta = f[0] * d[0] + f[1] * d[1] + f[2] * d[2] + phi;
  return std::exp(-0.5 * q) * 0.5 * (1.0 + beta * std::cos(theta));
}

// Order-preserving map of float bits: ascending float -> ascending uint32.
static inline uint32_t orderable_u32(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  return (u >> 31) ? ~u : (u | 0x80000000u);
}

static inline bool finite_all(const double* p, int n) {
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

static inline double frac_margin(double v) {
  // distance of v to the nearest integer, relative to max(1, |v|)
  double d = std::fabs(v - std::nearbyint(v));
  return d / std::max(1.0, std::fabs(v));
}

// Steps 2-7 of DESIGN.md "O1" on a 2x2 covariance (sxx, sxy, syy) already
// including the diagonal offset. Writes conic, extent, rect, count, flag.
static void finish_2d(const ora_cfg& c, double mux, double muy, double sxx,
                      double sxy, double syy, double alpha, int32_t* flag,
                      int32_t* rect, int32_t* count, double* rec) {
  const int GX = (c.width + c.tile - 1) / c.tile;
  const int GY = (c.height + c.tile - 1) / c.tile;
  rect[0] = rect[1] = rect[2] = rect[3] = 0;
  *count = 0;
  double det = sxx * syy - sxy * sxy;
  rec[P_SXX] = sxx; rec[P_SXY] = sxy; rec[P_SYY] = syy;
  if (!(det >= c.det_min) || !(sxx > 0.0) || !(syy > 0.0)) { *flag = 2; return; }
  if (!(alpha >= c.alpha_min)) { *flag = 3; return; }
  rec[P_A] = syy / det;
  rec[P_B] = -sxy / det;
  rec[P_C] = sxx / det;
  double rx, ry;
  if (c.extent == 0) {
    double k = (c.alpha_min > 0.0) ? std::sqrt(2.0 * std::log(alpha / c.alpha_min))
                                   : INFINITY;
    rx = k * std::sqrt(sxx);
    ry = k * std::sqrt(syy);
  } else {
    double m = 0.5 * (sxx + syy);
    double lam = m + std::sqrt(std::max(m * m - det, 0.0));
    rx = 3.0 * std::sqrt(lam);
    ry = rx;
  }
  rec[P_RX] = rx; rec[P_RY] = ry;
  const double ts = (double)c.tile;
  double vx0 = (mux - rx) / ts, vx1 = (mux + rx) / ts;
  double vy0 = (muy - ry) / ts, vy1 = (muy + ry) / ts;
  double fx0 = std::floor(vx0), fx1 = std::floor(vx1) + 1.0;
  double fy0 = std::floor(vy0), fy1 = std::floor(vy1) + 1.0;
  fx0 = std::min(std::max(fx0, 0.0), (double)GX);
  fx1 = std::min(std::max(fx1, 0.0), (double)GX);
  fy0 = std::min(std::max(fy0, 0.0), (double)GY);
  fy1 = std::min(std::max(fy1, 0.0), (double)GY);
  double m = INFINITY;
  if (std::isfinite(vx0)) m = std::min(m, frac_margin(vx0));
  if (std::isfinite(vx1)) m = std::min(m, frac_margin(vx1));
  if (std::isfinite(vy0)) m = std::min(m, frac_margin(vy0));
  if (std::isfinite(vy1)) m = std::min(m, frac_margin(vy1));
  rec[P_RMARGIN] = m;
  int32_t x0 = (int32_t)fx0, x1 = (int32_t)fx1, y0 = (int32_t)fy0, y1 = (int32_t)fy1;
  int32_t n = std::max(0, x1 - x0) * std::max(0, y1 - y0);
  rect[0] = x0; rect[1] = y0; rect[2] = x1; rect[3] = y1;
  *count = n;
  *flag = (n == 0) ? 4 : 0;
}

// ---------------------------------------------------------------------------
// 2D covariance constructions.
// ---------------------------------------------------------------------------
void ora_cov2d(int32_t mode, const double* p, double* out /*sxx,sxy,syy*/) {
  if (mode == 0) {
    out[0] = p[0]; out[1] = p[1]; out[2] = p[2];
  } else if (mode == 1) {  // L = [[l1, 0], [l2, l3]], Sigma = L L^T
    double l1 = p[0], l2 = p[1], l3 = p[2];
    out[0] = l1 * l1;
    out[1] = l1 * l2;
    out[2] = (l2 * l2) + (l3 * l3);
  } else {  // R(theta) diag(sx^2, sy^2) R(theta)^T, R = [[c,-s],[s,c]]
    double th = p[0], sx = p[1], sy = p[2];
    double cs = std::cos(th), sn = std::sin(th);
    double sx2 = sx * sx, sy2 = sy * sy;
    out[0] = (cs * cs) * sx2 + (sn * sn) * sy2;
    out[1] = (cs * sn) * (sx2 - sy2);
    out[2] = (sn * sn) * sx2 + (cs * cs) * sy2;
  }
}

// ---------------------------------------------------------------------------
// O1: 2D preprocess. One "view" (B = 1). Outputs per primitive.
// ---------------------------------------------------------------------------
void ora_project2d(const ora_cfg* cfg, int64_t N, const double* mean,
                   const double* cov, const double* freq, const double* phase,
                   const double* color, const double* opacity,
                   const double* depth, int32_t* flag, int32_t* rect,
                   int32_t* count, uint32_t* keylo, double* rec) {
  const ora_cfg& c = *cfg;
  for (int64_t i = 0; i < N; ++i) {
    double* r = rec + i * ORA_P;
    for (int k = 0; k < ORA_P; ++k) r[k] = 0.0;
    keylo[i] = 0;
    double in[12] = {mean[2 * i], mean[2 * i + 1], cov[3 * i], cov[3 * i + 1],
                     cov[3 * i + 2], freq[2 * i], freq[2 * i + 1],
                     phase ? phase[i] : 0.0, color[3 * i], color[3 * i + 1],
                     color[3 * i + 2], opacity[i]};
    double dep = (c.alpha_blend && depth) ? depth[i] : 0.0;
    r[P_MUX] = in[0]; r[P_MUY] = in[1];
    r[P_FX] = in[5]; r[P_FY] = in[6]; r[P_PHI] = in[7]; r[P_BETA] = 1.0;
    r[P_CR] = in[8]; r[P_CG] = in[9]; r[P_CB] = in[10]; r[P_ALPHA] = in[11];
    r[P_DEPTH] = dep;
    if (!finite_all(in, 12) || !std::isfinite(dep)) {
      flag[i] = 5; count[i] = 0;
      rect[4 * i] = rect[4 * i + 1] = rect[4 * i + 2] = rect[4 * i + 3] = 0;
      continue;
    }
    if (c.alpha_blend) keylo[i] = orderable_u32((float)dep);
    double s[3];
    ora_cov2d(c.cov2, in + 2, s);
    double d = c.cov_eps + c.dilation;
    finish_2d(c, in[0], in[1], s[0] + d, s[1], s[2] + d, in[11], &flag[i],
              rect + 4 * i, &count[i], r);
  }
}

// ---------------------------------------------------------------------------
// O2: 3D preprocess (PAPER.md:106 Sigma = R S S^T R^T; :116-122 Eq. 2, J W;
// :194-198 Eq. 7; :212 frequency transform). Per (view v, primitive i).
// ---------------------------------------------------------------------------
static void quat_to_rot(const double* q, double* R, double* qn, double* qnorm) {
  double w = q[0], x = q[1], y = q[2], z = q[3];
  double n = std::sqrt(((w * w + x * x) + y * y) + z * z);
  w = w / n; x = x / n; y = y / n; z = z / n;
  qn[0] = w; qn[1] = x; qn[2] = y; qn[3] = z;
  *qnorm = n;
  R[0] = 1.0 - 2.0 * ((y * y) + (z * z));
  R[1] = 2.0 * ((x * y) - (w * z));
  R[2] = 2.0 * ((x * z) + (w * y));
  R[3] = 2.0 * ((x * y) + (w * z));
  R[4] = 1.0 - 2.0 * ((x * x) + (z * z));
  R[5] = 2.0 * ((y * z) - (w * x));
  R[6] = 2.0 * ((x * z) - (w * y));
  R[7] = 2.0 * ((y * z) + (w * x));
  R[8] = 1.0 - 2.0 * ((x * x) + (y * y));
}

// everything a 3D primitive's projection needs for forward AND backward
struct proj3 {
  double p[3];        // camera-space mean
  double Rq[9];       // rotation from the normalised quaternion
  double qn[4], qnorm;
  double S3[6];       // Sigma3 unique entries (00,01,02,11,12,22)
  double J[4];        // j00, j02, j11, j12
  double tclamped[2]; // 1 if x/z (resp. y/z) was clamped
  double th[2];       // clamped tan values
  double M[6];        // 2x3 M = J Rv
  double g[3];        // Rv f
  double Sp[3];       // Sigma' (before the diagonal offset)
  // exact-mode extras
  double Shat[6];     // full ray-space covariance (00,01,02,11,12,22)
  double fhat[3];
};

static inline double S3at(const double* S, int i, int j) {
  static const int idx[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
  return S[idx[i][j]];
}

// Pinned expression order: DESIGN.md "Pinned preprocess arithmetic (3D)".
static void project3_core(const ora_cfg& c, const ora_cam& cam,
                          const double* mu, const double* s, const double* q,
                          const double* f, proj3& P) {
  const double* Rv = cam.R;
  for (int r = 0; r < 3; ++r)
    P.p[r] = ((Rv[3 * r] * mu[0] + Rv[3 * r + 1] * mu[1]) + Rv[3 * r + 2] * mu[2]) + cam.t[r];
  double x = P.p[0], y = P.p[1], z = P.p[2];
  quat_to_rot(q, P.Rq, P.qn, &P.qnorm);
  double s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
  const double* R = P.Rq;
  int k = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j)
      P.S3[k++] = (((R[3 * i] * s2[0]) * R[3 * j] + (R[3 * i + 1] * s2[1]) * R[3 * j + 1]) +
                   (R[3 * i + 2] * s2[2]) * R[3 * j + 2]);
  double tx = x / z, ty = y / z;
  P.tclamped[0] = P.tclamped[1] = 0.0;
  if (c.ewa_clamp) {
    double limx = (1.3 * (double)c.width) / (2.0 * cam.fx);
    double limy = (1.3 * (double)c.height) / (2.0 * cam.fy);
    if (tx < -limx || tx > limx) P.tclamped[0] = 1.0;
    if (ty < -limy || ty > limy) P.tclamped[1] = 1.0;
    tx = std::min(std::max(tx, -limx), limx);
    ty = std::min(std::max(ty, -limy), limy);
  }
  P.th[0] = tx; P.th[1] = ty;
  double j00 = cam.fx / z, j11 = cam.fy / z;
  double j02 = -(cam.fx * tx) / z, j12 = -(cam.fy * ty) / z;
  P.J[0] = j00; P.J[1] = j02; P.J[2] = j11; P.J[3] = j12;
  for (int jj = 0; jj < 3; ++jj) {
    P.M[jj] = j00 * Rv[jj] + j02 * Rv[6 + jj];
    P.M[3 + jj] = j11 * Rv[3 + jj] + j12 * Rv[6 + jj];
  }
  double T[2][3];
  for (int i = 0; i < 2; ++i)
    for (int kk = 0; kk < 3; ++kk)
      T[i][kk] = ((P.M[3 * i] * S3at(P.S3, 0, kk) + P.M[3 * i + 1] * S3at(P.S3, 1, kk)) +
                  P.M[3 * i + 2] * S3at(P.S3, 2, kk));
  P.Sp[0] = ((T[0][0] * P.M[0] + T[0][1] * P.M[1]) + T[0][2] * P.M[2]);
  P.Sp[1] = ((T[0][0] * P.M[3] + T[0][1] * P.M[4]) + T[0][2] * P.M[5]);
  P.Sp[2] = ((T[1][0] * P.M[3] + T[1][1] * P.M[4]) + T[1][2] * P.M[5]);
  for (int r = 0; r < 3; ++r)
    P.g[r] = ((Rv[3 * r] * f[0] + Rv[3 * r + 1] * f[1]) + Rv[3 * r + 2] * f[2]);
  // exact-mode quantities: full 3x3 ray-space covariance with J3 row 3 = [0 0 1]
  // and f_hat = (J3 Rv)^{-T} f.
  double M3[9] = {P.M[0], P.M[1], P.M[2], P.M[3], P.M[4], P.M[5], Rv[6], Rv[7], Rv[8]};
  k = 0;
  for (int i = 0; i < 3; ++i)
    for (int j = i; j < 3; ++j) {
      double acc = 0.0;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) acc += M3[3 * i + a] * S3at(P.S3, a, b) * M3[3 * j + b];
      P.Shat[k++] = acc;
    }
  P.fhat[0] = (z * P.g[0]) / cam.fx;
  P.fhat[1] = (z * P.g[1]) / cam.fy;
  // third component of J3^{-T} g with J3 = [[j00,0,j02],[0,j11,j12],[0,0,1]]
  P.fhat[2] = P.g[2] - j02 * P.fhat[0] - j12 * P.fhat[1];
}

void ora_project3d(const ora_cfg* cfg, int64_t N, int32_t B, const ora_cam* cams,
                   const double* mean, const double* scale, const double* quat,
                   const double* freq, const double* phase, const double* color,
                   const double* opacity, int64_t view_stride, int32_t* flag,
                   int32_t* rect, int32_t* count, uint32_t* keylo, double* rec) {
  const ora_cfg& c = *cfg;
  for (int32_t v = 0; v < B; ++v) {
    const ora_cam& cam = cams[v];
    for (int64_t i = 0; i < N; ++i) {
      const int64_t o = (int64_t)v * N + i;       // output row
      const int64_t pi = (int64_t)v * view_stride + i;  // parameter row
      double* r = rec + o * ORA_P;
      for (int k = 0; k < ORA_P; ++k) r[k] = 0.0;
      keylo[o] = 0;
      rect[4 * o] = rect[4 * o + 1] = rect[4 * o + 2] = rect[4 * o + 3] = 0;
      count[o] = 0;
      double in[17] = {mean[3 * pi], mean[3 * pi + 1], mean[3 * pi + 2],
                       scale[3 * pi], scale[3 * pi + 1], scale[3 * pi + 2],
                       quat[4 * pi], quat[4 * pi + 1], quat[4 * pi + 2], quat[4 * pi + 3],
                       freq[3 * pi], freq[3 * pi + 1], freq[3 * pi + 2],
                       phase ? phase[pi] : 0.0,
                       opacity[pi], 0.0, 0.0};
      r[P_PHI] = in[13];
      const double* col = c.color_per_view ? color + 3 * o : color + 3 * pi;
      r[P_CR] = col[0]; r[P_CG] = col[1]; r[P_CB] = col[2];
      r[P_ALPHA] = in[14];
      in[15] = ((in[6] * in[6] + in[7] * in[7]) + in[8] * in[8]) + in[9] * in[9];
      if (!finite_all(in, 15) || !finite_all(col, 3) || !(in[15] > 0.0)) {
        flag[o] = 5;
        continue;
      }
      proj3 P;
      project3_core(c, cam, in, in + 3, in + 6, in + 10, P);
      double x = P.p[0], y = P.p[1], z = P.p[2];
      if (!(z >= cam.near_z && z <= cam.far_z)) { flag[o] = 1; continue; }
      r[P_MUX] = (cam.fx * (x / z)) + cam.cx;
      r[P_MUY] = (cam.fy * (y / z)) + cam.cy;
      double fpx = (z * P.g[0]) / cam.fx, fpy = (z * P.g[1]) / cam.fy;
      double beta = 1.0;
      if (c.exact_proj) {
        // exact z-marginal: sigma = (Shat_xz, Shat_yz),
        // v = Shat_zz - sigma^T S2^{-1} sigma, f' = fhat_xy + fhat_z S2^{-1} sigma,
        // beta = exp(-1/2 fhat_z^2 v); S2 = undilated upper-left 2x2.
        double a = P.Shat[0], b = P.Shat[1], d = P.Shat[3];
        double det2 = a * d - b * b;
        double sx = P.Shat[2], sy = P.Shat[4];
        double ux = (d * sx - b * sy) / det2, uy = (-b * sx + a * sy) / det2;
        double vv = P.Shat[5] - (sx * ux + sy * uy);
        fpx = P.fhat[0] + P.fhat[2] * ux;
        fpy = P.fhat[1] + P.fhat[2] * uy;
        beta = std::exp(-0.5 * P.fhat[2] * P.fhat[2] * vv);
      }
      r[P_FX] = fpx; r[P_FY] = fpy; r[P_BETA] = beta;
      float dz = (float)z;
      r[P_DEPTH] = (double)dz;
      keylo[o] = orderable_u32(dz);
      double dd = c.cov_eps + c.dilation;
      finish_2d(c, r[P_MUX], r[P_MUY], P.Sp[0] + dd, P.Sp[1], P.Sp[2] + dd, in[14],
                &flag[o], rect + 4 * o, &count[o], r);
    }
  }
}

// ---------------------------------------------------------------------------
// O6: integer artefacts — offsets, (key, value) pairs, stable sort, CSR.
// ---------------------------------------------------------------------------
int64_t ora_bin(const ora_cfg* cfg, int64_t N, int32_t B, const int32_t* rect,
                const int32_t* count, const uint32_t* keylo, int64_t* offsets,
                uint64_t* keys, uint32_t* vals, int64_t* tile_offsets,
                int64_t capacity) {
  const ora_cfg& c = *cfg;
  const int64_t GX = (c.width + c.tile - 1) / c.tile;
  const int64_t GY = (c.height + c.tile - 1) / c.tile;
  const int64_t T = GX * GY;
  int64_t total = 0;
  for (int64_t o = 0; o < (int64_t)B * N; ++o) {
    offsets[o] = total;
    total += count[o];
  }
  if (!keys || total > capacity) return total;
  std::vector<std::pair<uint64_t, uint32_t>> kv;
  kv.reserve((size_t)total);
  for (int64_t o = 0; o < (int64_t)B * N; ++o) {
    if (count[o] == 0) continue;
    int64_t v = o / N, i = o % N;
    const int32_t* r = rect + 4 * o;
    for (int32_t ty = r[1]; ty < r[3]; ++ty)
      for (int32_t tx = r[0]; tx < r[2]; ++tx) {
        uint64_t tile_id = (uint64_t)(v * T + (int64_t)ty * GX + tx);
        uint64_t key = (tile_id << 32) | (uint64_t)(c.alpha_blend ? keylo[o] : 0u);
        kv.emplace_back(key, (uint32_t)i);
      }
  }
  std::stable_sort(kv.begin(), kv.end(),
                   [](const std::pair<uint64_t, uint32_t>& a,
                      const std::pair<uint64_t, uint32_t>& b) { return a.first < b.first; });
  for (int64_t j = 0; j < total; ++j) { keys[j] = kv[j].first; vals[j] = kv[j].second; }
  if (tile_offsets) {
    // CSR: tile_offsets[u] = #entries with (key >> 32) < u, u in [0, B*T]
    int64_t j = 0;
    for (int64_t u = 0; u <= (int64_t)B * T; ++u) {
      while (j < total && (int64_t)(keys[j] >> 32) < u) ++j;
      tile_offsets[u] = j;
    }
  }
  return total;
}

// ---------------------------------------------------------------------------
// O3-O5: brute-force render (+ optional backward) over a list of pixels.
// pix: flat pixel ids v*H*W + y*W + x (NULL = all, in that order).
// Outputs per listed pixel: color[3], T_final, margin, ncomp (# composited or
// # contributing), and optionally record gradients rgrad[B*N, ORA_G] of
// L = sum_pix dLdC[pix] . C[pix].
// ---------------------------------------------------------------------------
struct pair_eval {
  double dx, dy, G, theta, h, W, w;
};

static inline void eval_pair(const double* r, double px, double py, pair_eval& e) {
  e.dx = px - r[P_MUX];
  e.dy = py - r[P_MUY];
  double q = r[P_A] * e.dx * e.dx + 2.0 * r[P_B] * e.dx * e.dy + r[P_C] * e.dy * e.dy;
  e.G = std::exp(-0.5 * q);
  e.theta = r[P_FX] * e.dx + r[P_FY] * e.dy + r[P_PHI];
  e.h = 0.5 * (1.0 + r[P_BETA] * std::cos(e.theta));
  e.W = e.G * e.h;
  e.w = r[P_ALPHA] * e.W;
}

// d w / d(record quantities), scaled by gw = dL/dw, accumulated into g[ORA_G]
// (O5 in DESIGN.md): with s = d w/d theta = -1/2 beta alpha G sin(theta),
//   dw/dmu' = w (A d) - s f',  dw/d(a,b,c) = -1/2 w (dx^2, 2 dx dy, dy^2),
//   dw/df' = s d, dw/dphi = s, dw/dbeta = 1/2 alpha G cos(theta), dw/dalpha = W.
static inline void acc_w_grad(const double* r, const pair_eval& e, double gw, double* g) {
  double s = -0.5 * r[P_BETA] * r[P_ALPHA] * e.G * std::sin(e.theta);
  double Adx = r[P_A] * e.dx + r[P_B] * e.dy;
  double Ady = r[P_B] * e.dx + r[P_C] * e.dy;
  g[G_MUX] += gw * (e.w * Adx - s * r[P_FX]);
  g[G_MUY] += gw * (e.w * Ady - s * r[P_FY]);
  g[G_A] += gw * (-0.5 * e.w * e.dx * e.dx);
  g[G_B] += gw * (-0.5 * e.w * 2.0 * e.dx * e.dy);
  g[G_C] += gw * (-0.5 * e.w * e.dy * e.dy);
  g[G_FX] += gw * s * e.dx;
  g[G_FY] += gw * s * e.dy;
  g[G_PHI] += gw * s;
  g[G_BETA] += gw * 0.5 * r[P_ALPHA] * e.G * std::cos(e.theta);
  g[G_ALPHA] += gw * e.W;
}

// Running error bound companion of acc_w_grad (R23b): the same
// terms with every factor and every summand taken in absolute value, scaled by
// gwa = the absolute-term magnitude of dL/dw. Summed over pairs it gives S_q =
// sum of |terms| of record gradient q, the scale of the rounding error any
// finite-precision evaluation of those terms carries.
static inline void acc_w_grad_abs(const double* r, const pair_eval& e, double gwa, double* g) {
  double s = 0.5 * std::fabs(r[P_BETA] * r[P_ALPHA] * e.G * std::sin(e.theta));
  double w = std::fabs(e.w), dx = std::fabs(e.dx), dy = std::fabs(e.dy);
  double a = std::fabs(r[P_A]), b = std::fabs(r[P_B]), c = std::fabs(r[P_C]);
  g[G_MUX] += gwa * (w * (a * dx + b * dy) + s * std::fabs(r[P_FX]));
  g[G_MUY] += gwa * (w * (b * dx + c * dy) + s * std::fabs(r[P_FY]));
  g[G_A] += gwa * 0.5 * w * dx * dx;
  g[G_B] += gwa * w * dx * dy;
  g[G_C] += gwa * 0.5 * w * dy * dy;
  g[G_FX] += gwa * s * dx;
  g[G_FY] += gwa * s * dy;
  g[G_PHI] += gwa * s;
  g[G_BETA] += gwa * 0.5 * std::fabs(r[P_ALPHA] * e.G * std::cos(e.theta));
  g[G_ALPHA] += gwa * std::fabs(e.W);
}

static inline double rel_margin(double v, double thr) {
  if (thr == 0.0) return INFINITY;
  return std::fabs(v / thr - 1.0);
}

void ora_render(const ora_cfg* cfg, int64_t N, int32_t B, const double* rec,
                const int32_t* flag, const int32_t* rect, const uint32_t* keylo,
                int64_t npix, const int64_t* pix, double* color, double* T_out,
                double* margin, int32_t* ncomp, const double* dLdC, double* rgrad,
                int32_t nthreads, double* rgrad_abs) {
  const ora_cfg& c = *cfg;
  const int64_t H = c.height, W = c.width, HW = H * W;
  const int64_t GX = (c.width + c.tile - 1) / c.tile;
  if (!pix) npix = (int64_t)B * HW;
  // per-view evaluation order: ascending index (SUM) or (key lo, index) (ALPHA)
  std::vector<std::vector<int64_t>> order(B);
  for (int32_t v = 0; v < B; ++v) {
    auto& ord = order[v];
    for (int64_t i = 0; i < N; ++i)
      if (flag[(int64_t)v * N + i] == 0) ord.push_back(i);
    if (c.alpha_blend)
      std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
        return keylo[(int64_t)v * N + a] < keylo[(int64_t)v * N + b];
      });
  }
#ifdef _OPENMP
  int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#else
  int nt = 1;
#endif
  const int64_t G_SIZE = (int64_t)B * N * ORA_G;
  // per-thread gradient buffers merged in thread order (deterministic)
  std::vector<std::vector<double>> tg;
  bool per_thread = rgrad && (G_SIZE * (int64_t)nt * 8 <= (int64_t)2 << 30);
  if (rgrad) {
    std::memset(rgrad, 0, sizeof(double) * G_SIZE);
    if (rgrad_abs) std::memset(rgrad_abs, 0, sizeof(double) * G_SIZE);
    if (per_thread) tg.assign(nt, std::vector<double>());
  }
#pragma omp parallel num_threads(nt)
  {
#ifdef _OPENMP
    int tid = omp_get_thread_num();
#else
    int tid = 0;
#endif
    double* gbuf = nullptr;
    if (rgrad && per_thread) { tg[tid].assign(G_SIZE, 0.0); gbuf = tg[tid].data(); }
    std::vector<int64_t> comp_i;  // composited entries (ALPHA backward)
    std::vector<double> comp_a, comp_T, comp_w;
    std::vector<pair_eval> comp_e;
#pragma omp for schedule(dynamic, 16)
    for (int64_t k = 0; k < npix; ++k) {
      int64_t id = pix ? pix[k] : k;
      int64_t v = id / HW, rem = id % HW, yi = rem / W, xi = rem % W;
      double px = (double)xi + 0.5, py = (double)yi + 0.5;
      int64_t tile_x = xi / c.tile, tile_y = yi / c.tile;
      (void)GX;
      double C[3] = {0, 0, 0}, T = 1.0, mg = INFINITY;
      int32_t n = 0;
      comp_i.clear(); comp_a.clear(); comp_T.clear(); comp_w.clear(); comp_e.clear();
      const double* g3 = dLdC ? dLdC + 3 * k : nullptr;
      for (int64_t i : order[v]) {
        const int64_t o = v * N + i;
        const double* r = rec + o * ORA_P;
        if (c.use_rect || c.extent == 1) {
          const int32_t* rc = rect + 4 * o;
          if (!(tile_x >= rc[0] && tile_x < rc[2] && tile_y >= rc[1] && tile_y < rc[3])) continue;
        }
        pair_eval e;
        eval_pair(r, px, py, e);
        mg = std::min(mg, rel_margin(e.w, c.alpha_min));
        if (!c.alpha_blend) {
          if (!(e.w >= c.alpha_min)) continue;
          C[0] += r[P_CR] * e.w; C[1] += r[P_CG] * e.w; C[2] += r[P_CB] * e.w;
          ++n;
          if (rgrad) {
            double* g = (per_thread ? gbuf : nullptr);
            double loc[ORA_G] = {0};
            double gw = r[P_CR] * g3[0] + r[P_CG] * g3[1] + r[P_CB] * g3[2];
            loc[G_CR] = e.w * g3[0]; loc[G_CG] = e.w * g3[1]; loc[G_CB] = e.w * g3[2];
            acc_w_grad(r, e, gw, loc);
            if (g) {
              for (int q = 0; q < ORA_G; ++q) g[o * ORA_G + q] += loc[q];
            } else {
              for (int q = 0; q < ORA_G; ++q) {
#pragma omp atomic
                rgrad[o * ORA_G + q] += loc[q];
              }
            }
            if (rgrad_abs) {
              double la[ORA_G] = {0};
              const double gwa = std::fabs(r[P_CR] * g3[0]) + std::fabs(r[P_CG] * g3[1]) +
                                 std::fabs(r[P_CB] * g3[2]);
              la[G_CR] = std::fabs(e.w * g3[0]); la[G_CG] = std::fabs(e.w * g3[1]);
              la[G_CB] = std::fabs(e.w * g3[2]);
              acc_w_grad_abs(r, e, gwa, la);
              for (int q = 0; q < ORA_G; ++q) {
#pragma omp atomic
                rgrad_abs[o * ORA_G + q] += la[q];
              }
            }
          }
        } else {
          double a = std::min(c.alpha_max, e.w);
          mg = std::min(mg, rel_margin(e.w, c.alpha_max));
          if (!(a >= c.alpha_min)) continue;
          double Tn = T * (1.0 - a);
          mg = std::min(mg, rel_margin(Tn, c.T_min));
          if (Tn < c.T_min) break;
          C[0] += r[P_CR] * a * T; C[1] += r[P_CG] * a * T; C[2] += r[P_CB] * a * T;
          if (rgrad) {
            comp_i.push_back(o); comp_a.push_back(a); comp_T.push_back(T);
            comp_w.push_back(e.w); comp_e.push_back(e);
          }
          T = Tn;
          ++n;
        }
      }
      if (c.alpha_blend) {
        C[0] += T * c.bg[0]; C[1] += T * c.bg[1]; C[2] += T * c.bg[2];
        if (rgrad) {
          // back-to-front: S = colour accumulated behind entry k (incl. bg)
          double S[3] = {T * c.bg[0], T * c.bg[1], T * c.bg[2]};
          for (int64_t m = (int64_t)comp_i.size() - 1; m >= 0; --m) {
            const int64_t o = comp_i[m];
            const double* r = rec + o * ORA_P;
            double a = comp_a[m], Tk = comp_T[m];
            const double cc[3] = {r[P_CR], r[P_CG], r[P_CB]};
            double dLda = 0.0;
            for (int ch = 0; ch < 3; ++ch)
              dLda += g3[ch] * (cc[ch] * Tk - S[ch] / (1.0 - a));
            double loc[ORA_G] = {0};
            loc[G_CR] = a * Tk * g3[0]; loc[G_CG] = a * Tk * g3[1]; loc[G_CB] = a * Tk * g3[2];
            double gw = (comp_w[m] < c.alpha_max) ? dLda : 0.0;
            acc_w_grad(r, comp_e[m], gw, loc);
            if (rgrad_abs) {
              double la[ORA_G] = {0}, gwa = 0.0;
              for (int ch = 0; ch < 3; ++ch) {
                la[G_CR + ch] = std::fabs(a * Tk * g3[ch]);
                gwa += std::fabs(g3[ch]) * (std::fabs(cc[ch] * Tk) + std::fabs(S[ch]) / (1.0 - a));
              }
              if (comp_w[m] < c.alpha_max) acc_w_grad_abs(r, comp_e[m], gwa, la);
              for (int q = 0; q < ORA_G; ++q) {
#pragma omp atomic
                rgrad_abs[o * ORA_G + q] += la[q];
              }
            }
            for (int ch = 0; ch < 3; ++ch) S[ch] += cc[ch] * a * Tk;
            if (per_thread) {
              for (int q = 0; q < ORA_G; ++q) gbuf[o * ORA_G + q] += loc[q];
            } else {
              for (int q = 0; q < ORA_G; ++q) {
#pragma omp atomic
                rgrad[o * ORA_G + q] += loc[q];
              }
            }
          }
        }
      }
      if (color) { color[3 * k] = C[0]; color[3 * k + 1] = C[1]; color[3 * k + 2] = C[2]; }
      if (T_out) T_out[k] = T;
      if (margin) margin[k] = mg;
      if (ncomp) ncomp[k] = n;
    }
  }
  if (rgrad && per_thread) {
    for (int t = 0; t < nt; ++t)
      if (!tg[t].empty())
        for (int64_t q = 0; q < G_SIZE; ++q) rgrad[q] += tg[t][q];
  }
}

// ---------------------------------------------------------------------------
// Conic -> covariance chain: G_Sigma = -A G_A A with G_A symmetric, off-diag
// entries = gb/2 (b is the single off-diagonal value). Returns the gradient
// w.r.t. the unique entries (sxx, sxy, syy), sxy counted twice.
// ---------------------------------------------------------------------------
static void conic_to_cov_grad(const double* A /*a,b,c*/, double ga, double gb,
                              double gc, double* gs /*gxx,gxy,gyy*/) {
  double a = A[0], b = A[1], cc = A[2];
  double Ga[2][2] = {{ga, 0.5 * gb}, {0.5 * gb, gc}};
  double Am[2][2] = {{a, b}, {b, cc}};
  double T1[2][2], T2[2][2];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) T1[i][j] = Am[i][0] * Ga[0][j] + Am[i][1] * Ga[1][j];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) T2[i][j] = -(T1[i][0] * Am[0][j] + T1[i][1] * Am[1][j]);
  gs[0] = T2[0][0];
  gs[1] = T2[0][1] + T2[1][0];
  gs[2] = T2[1][1];
}

void ora_chain2d(const ora_cfg* cfg, int64_t N, const double* cov,
                 const int32_t* flag, const double* rec, const double* rgrad,
                 double* g_mean, double* g_cov, double* g_freq, double* g_phase,
                 double* g_color, double* g_opacity) {
  const ora_cfg& c = *cfg;
  for (int64_t i = 0; i < N; ++i) {
    const double* g = rgrad + i * ORA_G;
    const double* r = rec + i * ORA_P;
    bool live = flag[i] == 0;
    auto G = [&](int k) { return live ? g[k] : 0.0; };
    if (g_mean) { g_mean[2 * i] = G(G_MUX); g_mean[2 * i + 1] = G(G_MUY); }
    if (g_freq) { g_freq[2 * i] = G(G_FX); g_freq[2 * i + 1] = G(G_FY); }
    if (g_phase) g_phase[i] = G(G_PHI);
    if (g_color) { g_color[3 * i] = G(G_CR); g_color[3 * i + 1] = G(G_CG); g_color[3 * i + 2] = G(G_CB); }
    if (g_opacity) g_opacity[i] = G(G_ALPHA);
    if (g_cov) {
      double* gc = g_cov + 3 * i;
      gc[0] = gc[1] = gc[2] = 0.0;
      if (!live) continue;
      double A[3] = {r[P_A], r[P_B], r[P_C]};
      double gs[3];
      conic_to_cov_grad(A, g[G_A], g[G_B], g[G_C], gs);
      const double* p = cov + 3 * i;
      if (c.cov2 == 0) {
        gc[0] = gs[0]; gc[1] = gs[1]; gc[2] = gs[2];
      } else if (c.cov2 == 1) {
        double l1 = p[0], l2 = p[1], l3 = p[2];
        gc[0] = 2.0 * l1 * gs[0] + l2 * gs[1];
        gc[1] = l1 * gs[1] + 2.0 * l2 * gs[2];
        gc[2] = 2.0 * l3 * gs[2];
      } else {
        double th = p[0], sx = p[1], sy = p[2];
        double cs = std::cos(th), sn = std::sin(th);
        gc[0] = (sx * sx - sy * sy) *
                (-2.0 * cs * sn * gs[0] + (cs * cs - sn * sn) * gs[1] + 2.0 * cs * sn * gs[2]);
        gc[1] = 2.0 * sx * (cs * cs * gs[0] + cs * sn * gs[1] + sn * sn * gs[2]);
        gc[2] = 2.0 * sy * (sn * sn * gs[0] - cs * sn * gs[1] + cs * cs * gs[2]);
      }
    }
  }
}

// 3D chain (paper mode): record gradients of (view, primitive) -> mean, scale,
// quat, freq, phase, color, opacity. view_stride 0 => sum over views.
void ora_chain3d(const ora_cfg* cfg, int64_t N, int32_t B, const ora_cam* cams,
                 const double* mean, const double* scale, const double* quat,
                 const double* freq, const int32_t* flag, const double* rec,
                 const double* rgrad, int64_t view_stride, double* g_mean,
                 double* g_scale, double* g_quat, double* g_freq, double* g_phase,
                 double* g_color, double* g_opacity) {
  const ora_cfg& c = *cfg;
  int64_t NP = view_stride == 0 ? N : (int64_t)B * N;
  if (g_mean) std::memset(g_mean, 0, sizeof(double) * 3 * NP);
  if (g_scale) std::memset(g_scale, 0, sizeof(double) * 3 * NP);
  if (g_quat) std::memset(g_quat, 0, sizeof(double) * 4 * NP);
  if (g_freq) std::memset(g_freq, 0, sizeof(double) * 3 * NP);
  if (g_phase) std::memset(g_phase, 0, sizeof(double) * NP);
  if (g_color) std::memset(g_color, 0, sizeof(double) * 3 * NP);
  if (g_opacity) std::memset(g_opacity, 0, sizeof(double) * NP);
  for (int32_t v = 0; v < B; ++v) {
    const ora_cam& cam = cams[v];
    const double* Rv = cam.R;
    for (int64_t i = 0; i < N; ++i) {
      const int64_t o = (int64_t)v * N + i;
      if (flag[o] != 0) continue;
      const int64_t pi = (int64_t)v * view_stride + i;
      const double* g = rgrad + o * ORA_G;
      const double* r = rec + o * ORA_P;
      if (g_phase) g_phase[pi] += g[G_PHI];
      if (g_color) for (int k = 0; k < 3; ++k) g_color[3 * pi + k] += g[G_CR + k];
      if (g_opacity) g_opacity[pi] += g[G_ALPHA];
      proj3 P;
      project3_core(c, cam, mean + 3 * pi, scale + 3 * pi, quat + 4 * pi, freq + 3 * pi, P);
      double x = P.p[0], y = P.p[1], z = P.p[2];
      double fx = cam.fx, fy = cam.fy;
      double dp[3] = {0, 0, 0};
      // mu' = (fx x/z + cx, fy y/z + cy)
      dp[0] += g[G_MUX] * fx / z;
      dp[1] += g[G_MUY] * fy / z;
      dp[2] += -g[G_MUX] * fx * x / (z * z) - g[G_MUY] * fy * y / (z * z);
      // f' = (z gx/fx, z gy/fy), g = Rv f
      dp[2] += g[G_FX] * P.g[0] / fx + g[G_FY] * P.g[1] / fy;
      double dg[3] = {g[G_FX] * z / fx, g[G_FY] * z / fy, 0.0};
      if (g_freq)
        for (int k = 0; k < 3; ++k)
          g_freq[3 * pi + k] += Rv[k] * dg[0] + Rv[3 + k] * dg[1] + Rv[6 + k] * dg[2];
      // conic -> Sigma' (matrix form; symmetric)
      double A[3] = {r[P_A], r[P_B], r[P_C]};
      double gs[3];
      conic_to_cov_grad(A, g[G_A], g[G_B], g[G_C], gs);
      double GS[2][2] = {{gs[0], 0.5 * gs[1]}, {0.5 * gs[1], gs[2]}};
      double M[2][3] = {{P.M[0], P.M[1], P.M[2]}, {P.M[3], P.M[4], P.M[5]}};
      double S3[3][3];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) S3[a][b] = S3at(P.S3, a, b);
      // dL/dM = 2 G M S3 ; dL/dS3 = M^T G M
      double GM[2][3];
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) GM[a][b] = GS[a][0] * M[0][b] + GS[a][1] * M[1][b];
      double dM[2][3];
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) {
          double acc = 0.0;
          for (int k = 0; k < 3; ++k) acc += GM[a][k] * S3[k][b];
          dM[a][b] = 2.0 * acc;
        }
      double dS3[3][3];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) dS3[a][b] = M[0][a] * GM[0][b] + M[1][a] * GM[1][b];
      // dL/dJ = dL/dM Rv^T  (only j00, j02, j11, j12 are live)
      auto dJ = [&](int a, int b) {
        return dM[a][0] * Rv[3 * b] + dM[a][1] * Rv[3 * b + 1] + dM[a][2] * Rv[3 * b + 2];
      };
      double dj00 = dJ(0, 0), dj02 = dJ(0, 2), dj11 = dJ(1, 1), dj12 = dJ(1, 2);
      // j00 = fx/z, j11 = fy/z, j02 = -fx th_x/z, j12 = -fy th_y/z
      dp[2] += dj00 * (-fx / (z * z)) + dj11 * (-fy / (z * z));
      double tx = P.th[0], ty = P.th[1];
      // d th_x / dx = 1/z, d th_x/dz = -x/z^2 when not clamped
      double dtx_dx = P.tclamped[0] ? 0.0 : 1.0 / z;
      double dtx_dz = P.tclamped[0] ? 0.0 : -x / (z * z);
      double dty_dy = P.tclamped[1] ? 0.0 : 1.0 / z;
      double dty_dz = P.tclamped[1] ? 0.0 : -y / (z * z);
      // j02 = -fx tx / z: d/dz = fx tx/z^2 - (fx/z) dtx_dz ; d/dx = -(fx/z) dtx_dx
      dp[0] += dj02 * (-(fx / z) * dtx_dx);
      dp[2] += dj02 * (fx * tx / (z * z) - (fx / z) * dtx_dz);
      dp[1] += dj12 * (-(fy / z) * dty_dy);
      dp[2] += dj12 * (fy * ty / (z * z) - (fy / z) * dty_dz);
      if (g_mean)
        for (int k = 0; k < 3; ++k)
          g_mean[3 * pi + k] += Rv[k] * dp[0] + Rv[3 + k] * dp[1] + Rv[6 + k] * dp[2];
      // Sigma3 = Rq diag(s^2) Rq^T
      const double* R = P.Rq;
      const double* s = scale + 3 * pi;
      // W = Rq^T dS3 Rq ; dL/ds_k = 2 s_k W_kk ; dL/dRq = 2 dS3 Rq diag(s^2)
      double dRq[9];
      for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k) {
          double acc = 0.0;
          for (int b = 0; b < 3; ++b) acc += dS3[a][b] * R[3 * b + k];
          dRq[3 * a + k] = 2.0 * acc * s[k] * s[k];
        }
      if (g_scale)
        for (int k = 0; k < 3; ++k) {
          double Wkk = 0.0;
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) Wkk += R[3 * a + k] * dS3[a][b] * R[3 * b + k];
          g_scale[3 * pi + k] += 2.0 * s[k] * Wkk;
        }
      if (g_quat) {
        double w = P.qn[0], qx = P.qn[1], qy = P.qn[2], qz = P.qn[3];
        // dR/dq-hat entries (rows r00..r22; cols w, x, y, z)
        const double D[9][4] = {
            {0, 0, -4 * qy, -4 * qz},
            {-2 * qz, 2 * qy, 2 * qx, -2 * w},
            {2 * qy, 2 * qz, 2 * w, 2 * qx},
            {2 * qz, 2 * qy, 2 * qx, 2 * w},
            {0, -4 * qx, 0, -4 * qz},
            {-2 * qx, -2 * w, 2 * qz, 2 * qy},
            {-2 * qy, 2 * qz, -2 * w, 2 * qx},
            {2 * qx, 2 * w, 2 * qz, 2 * qy},
            {0, -4 * qx, -4 * qy, 0}};
        double dqn[4] = {0, 0, 0, 0};
        for (int e = 0; e < 9; ++e)
          for (int k = 0; k < 4; ++k) dqn[k] += dRq[e] * D[e][k];
        // through q-hat = q/|q|: dq = (dqn - qn (qn . dqn)) / |q|
        double dot = dqn[0] * P.qn[0] + dqn[1] * P.qn[1] + dqn[2] * P.qn[2] + dqn[3] * P.qn[3];
        for (int k = 0; k < 4; ++k) g_quat[4 * pi + k] += (dqn[k] - P.qn[k] * dot) / P.qnorm;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Exact-mode (NEXT-1) record quantities of one (view, primitive)
// as a plain function of its 13 parameters (mu 3, scale 3, quat 4, freq 3):
// out = (mu'x, mu'y, conic a, b, c, f'x, f'y, beta). Same formulas as
// ora_project3d's exact branch. Returns false if culled.
// ---------------------------------------------------------------------------
static bool exact_record(const ora_cfg& c, const ora_cam& cam, const double* prm, double* out) {
  proj3 P;
  project3_core(c, cam, prm, prm + 3, prm + 6, prm + 10, P);
  double x = P.p[0], y = P.p[1], z = P.p[2];
  if (!(z >= cam.near_z && z <= cam.far_z)) return false;
  out[0] = (cam.fx * (x / z)) + cam.cx;
  out[1] = (cam.fy * (y / z)) + cam.cy;
  double dd = c.cov_eps + c.dilation;
  double sxx = P.Sp[0] + dd, sxy = P.Sp[1], syy = P.Sp[2] + dd;
  double det = sxx * syy - sxy * sxy;
  out[2] = syy / det; out[3] = -sxy / det; out[4] = sxx / det;
  double a = P.Shat[0], b = P.Shat[1], d = P.Shat[3];
  double det2 = a * d - b * b;
  double sx = P.Shat[2], sy = P.Shat[4];
  double ux = (d * sx - b * sy) / det2, uy = (-b * sx + a * sy) / det2;
  double vv = P.Shat[5] - (sx * ux + sy * uy);
  out[5] = P.fhat[0] + P.fhat[2] * ux;
  out[6] = P.fhat[1] + P.fhat[2] * uy;
  out[7] = std::exp(-0.5 * P.fhat[2] * P.fhat[2] * vv);
  return true;
}

// 3D chain for EXACT projection: parameter gradients = J^T g_rec with the
// Jacobian J of exact_record taken by central differences in double (h = 1e-6
// relative). view_stride 0 => sum over views. (Pinned by whole-pipeline FD in
// tests/test_oracle_grad.py.)
void ora_chain3d_exact(const ora_cfg* cfg, int64_t N, int32_t B, const ora_cam* cams,
                       const double* mean, const double* scale, const double* quat,
                       const double* freq, const int32_t* flag, const double* rec,
                       const double* rgrad, int64_t view_stride, double* g_mean,
                       double* g_scale, double* g_quat,
                       double* g_freq, double* g_phase, double* g_color, double* g_opacity) {
  const ora_cfg& c = *cfg;
  (void)rec;  // same signature as ora_chain3d
  int64_t NP = view_stride == 0 ? N : (int64_t)B * N;
  std::memset(g_mean, 0, sizeof(double) * 3 * NP);
  std::memset(g_scale, 0, sizeof(double) * 3 * NP);
  std::memset(g_quat, 0, sizeof(double) * 4 * NP);
  std::memset(g_freq, 0, sizeof(double) * 3 * NP);
  std::memset(g_phase, 0, sizeof(double) * NP);
  std::memset(g_color, 0, sizeof(double) * 3 * NP);
  std::memset(g_opacity, 0, sizeof(double) * NP);
  static const int gi[8] = {G_MUX, G_MUY, G_A, G_B, G_C, G_FX, G_FY, G_BETA};
  for (int32_t v = 0; v < B; ++v) {
    for (int64_t i = 0; i < N; ++i) {
      const int64_t o = (int64_t)v * N + i;
      if (flag[o] != 0) continue;
      const int64_t pi = (int64_t)v * view_stride + i;
      const double* g = rgrad + o * ORA_G;
      g_phase[pi] += g[G_PHI];
      for (int k = 0; k < 3; ++k) g_color[3 * pi + k] += g[G_CR + k];
      g_opacity[pi] += g[G_ALPHA];
      double prm[13];
      for (int k = 0; k < 3; ++k) prm[k] = mean[3 * pi + k];
      for (int k = 0; k < 3; ++k) prm[3 + k] = scale[3 * pi + k];
      for (int k = 0; k < 4; ++k) prm[6 + k] = quat[4 * pi + k];
      for (int k = 0; k < 3; ++k) prm[10 + k] = freq[3 * pi + k];
      double gp[13];
      for (int k = 0; k < 13; ++k) {
        const double h = 1e-6 * std::max(1.0, std::fabs(prm[k]));
        double pp[13], pm[13], rp[8], rm[8];
        std::memcpy(pp, prm, sizeof(prm));
        std::memcpy(pm, prm, sizeof(prm));
        pp[k] += h;
        pm[k] -= h;
        bool okp = exact_record(c, cams[v], pp, rp), okm = exact_record(c, cams[v], pm, rm);
        double acc = 0.0;
        if (okp && okm)
          for (int r = 0; r < 8; ++r) acc += g[gi[r]] * (rp[r] - rm[r]) / (2.0 * h);
        gp[k] = acc;
      }
      for (int k = 0; k < 3; ++k) g_mean[3 * pi + k] += gp[k];
      for (int k = 0; k < 3; ++k) g_scale[3 * pi + k] += gp[3 + k];
      for (int k = 0; k < 4; ++k) g_quat[4 * pi + k] += gp[6 + k];
      for (int k = 0; k < 3; ++k) g_freq[3 * pi + k] += gp[10 + k];
    }
  }
}

// ---------------------------------------------------------------------------
// O9 (NEXT-3): spherical-harmonic colour, PAPER.md:106 ("color attributes
// encoded by spherical harmonic coefficients c") with the 3DGS settings the
// paper keeps: real SH up to degree 3 in the 3DGS sign convention,
// colour = max(0, sum_k Y_k(d) sh_k + 1/2), d = (mu - C)/|mu - C|, C = -R^T t.
// Constants are written from their closed forms (normalisation of the real
// SH, e.g. Y_00 = 1/(2 sqrt(pi))); pinned by orthonormality on the sphere
// (tests/test_oracle_sh.py).
// ---------------------------------------------------------------------------
static void sh_basis(int deg, const double* d, double* Y) {
  const double pi = 3.14159265358979323846;
  const double x = d[0], y = d[1], z = d[2];
  const double c0 = 0.5 / std::sqrt(pi);
  const double c1 = std::sqrt(3.0 / (4.0 * pi));
  const double c2a = 0.5 * std::sqrt(15.0 / pi), c2b = 0.25 * std::sqrt(5.0 / pi),
               c2c = 0.25 * std::sqrt(15.0 / pi);
  const double c3a = 0.25 * std::sqrt(35.0 / (2.0 * pi)), c3b = 0.5 * std::sqrt(105.0 / pi),
               c3c = 0.25 * std::sqrt(21.0 / (2.0 * pi)), c3d = 0.25 * std::sqrt(7.0 / pi),
               c3e = 0.25 * std::sqrt(105.0 / pi);
  Y[0] = c0;
  if (deg < 1) return;
  Y[1] = -c1 * y;
  Y[2] = c1 * z;
  Y[3] = -c1 * x;
  if (deg < 2) return;
  Y[4] = c2a * x * y;
  Y[5] = -c2a * y * z;
  Y[6] = c2b * (2.0 * z * z - x * x - y * y);
  Y[7] = -c2a * x * z;
  Y[8] = c2c * (x * x - y * y);
  if (deg < 3) return;
  Y[9] = -c3a * y * (3.0 * x * x - y * y);
  Y[10] = c3b * x * y * z;
  Y[11] = -c3c * y * (4.0 * z * z - x * x - y * y);
  Y[12] = c3d * z * (2.0 * z * z - 3.0 * x * x - 3.0 * y * y);
  Y[13] = -c3c * x * (4.0 * z * z - x * x - y * y);
  Y[14] = c3e * z * (x * x - y * y);
  Y[15] = -c3a * x * (x * x - 3.0 * y * y);
}

void ora_sh_basis(int32_t deg, int64_t n, const double* dirs, double* out) {
  const int K = (deg + 1) * (deg + 1);
  for (int64_t i = 0; i < n; ++i) {
    double Y[16];
    sh_basis(deg, dirs + 3 * i, Y);
    for (int k = 0; k < K; ++k) out[i * K + k] = Y[k];
  }
}

static void sh_color(int deg, const ora_cam& cam, const double* mu, const double* sh,
                     double* rgb, bool* clamped) {
  double C[3], v[3];
  for (int j = 0; j < 3; ++j)
    C[j] = -(cam.R[j] * cam.t[0] + cam.R[3 + j] * cam.t[1] + cam.R[6 + j] * cam.t[2]);
  for (int j = 0; j < 3; ++j) v[j] = mu[j] - C[j];
  const double n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
  const double d[3] = {v[0] / n, v[1] / n, v[2] / n};
  double Y[16];
  sh_basis(deg, d, Y);
  const int K = (deg + 1) * (deg + 1);
  for (int ch = 0; ch < 3; ++ch) {
    double acc = 0.0;
    for (int k = 0; k < K; ++k) acc += Y[k] * sh[3 * k + ch];
    acc += 0.5;
    clamped[ch] = acc < 0.0;
    rgb[ch] = clamped[ch] ? 0.0 : acc;
  }
}

// Per (view, primitive) SH colours [B*N, 3] (the records' colour input).
void ora_sh_colors(int32_t deg, int64_t N, int32_t B, const ora_cam* cams, const double* mean,
                   const double* sh, int64_t view_stride, double* rgb) {
  const int K = (deg + 1) * (deg + 1);
  for (int32_t v = 0; v < B; ++v)
    for (int64_t i = 0; i < N; ++i) {
      const int64_t o = (int64_t)v * N + i, pi = (int64_t)v * view_stride + i;
      bool cl[3];
      sh_color(deg, cams[v], mean + 3 * pi, sh + 3 * K * pi, rgb + 3 * o, cl);
    }
}

// SH part of the chain: record colour gradients (rgrad G_CR..G_CB) ->
// dL/dsh (linear: Y_k dc where unclamped) and the view-direction term of
// dL/dmu, taken by central differences of sh_color in mu (h = 1e-6 |.|),
// ADDED to g_mean. Rows of g_sh / g_mean: param rows (view_stride 0 => summed
// over views).
void ora_sh_chain(int32_t deg, int64_t N, int32_t B, const ora_cam* cams, const double* mean,
                  const double* sh, int64_t view_stride, const int32_t* flag,
                  const double* rgrad, double* g_sh, double* g_mean) {
  const int K = (deg + 1) * (deg + 1);
  const int64_t NP = view_stride == 0 ? N : (int64_t)B * N;
  std::memset(g_sh, 0, sizeof(double) * 3 * K * NP);
  for (int32_t v = 0; v < B; ++v)
    for (int64_t i = 0; i < N; ++i) {
      const int64_t o = (int64_t)v * N + i, pi = (int64_t)v * view_stride + i;
      if (flag[o] != 0) continue;
      const double* g = rgrad + o * ORA_G;
      const double* mu = mean + 3 * pi;
      const double* shp = sh + 3 * K * pi;
      double rgb[3], C[3], v3[3];
      bool cl[3];
      sh_color(deg, cams[v], mu, shp, rgb, cl);
      for (int j = 0; j < 3; ++j)
        C[j] = -(cams[v].R[j] * cams[v].t[0] + cams[v].R[3 + j] * cams[v].t[1] +
                 cams[v].R[6 + j] * cams[v].t[2]);
      for (int j = 0; j < 3; ++j) v3[j] = mu[j] - C[j];
      const double nn = std::sqrt(v3[0] * v3[0] + v3[1] * v3[1] + v3[2] * v3[2]);
      const double d[3] = {v3[0] / nn, v3[1] / nn, v3[2] / nn};
      double Y[16];
      sh_basis(deg, d, Y);
      for (int ch = 0; ch < 3; ++ch) {
        if (cl[ch]) continue;
        for (int k = 0; k < K; ++k) g_sh[(3 * K) * pi + 3 * k + ch] += Y[k] * g[G_CR + ch];
      }
      for (int j = 0; j < 3; ++j) {
        double mp[3] = {mu[0], mu[1], mu[2]}, mm[3] = {mu[0], mu[1], mu[2]};
        const double h = 1e-6 * std::max(1.0, std::fabs(mu[j]));
        mp[j] += h;
        mm[j] -= h;
        double cp[3], cm[3];
        bool t1[3], t2[3];
        sh_color(deg, cams[v], mp, shp, cp, t1);
        sh_color(deg, cams[v], mm, shp, cm, t2);
        double acc = 0.0;
        for (int ch = 0; ch < 3; ++ch) acc += (cp[ch] - cm[ch]) / (2.0 * h) * g[G_CR + ch];
        g_mean[3 * pi + j] += acc;
      }
    }
}

// ---------------------------------------------------------------------------
// Roofline work counters (SURVEY §8(d) "How n_cand and n_ell are obtained"):
// per pixel, over the pixel's TILE LIST (the live primitives whose tile rect
// contains the pixel's tile, in the evaluation order of O4: index for SUM,
// (depth key, index) for ALPHA), counted up to and including the entry at
// which ALPHA compositing stops (Q10):
//   cand[k] : list entries processed (SUM: the whole list),
//   ell[k]  : of those, pairs passing the skip pre-test alpha*G >= thr_ell
//             (the envelope bound of R8: alpha*W >= alpha_min implies it),
//   con[k]  : contributing pairs (SUM: w >= alpha_min; ALPHA: composited),
//   amb[k]  : pairs whose log2(alpha*G) lies within 1e-5 of log2(thr_ell),
//             i.e. whose ell decision may flip under FP32 rounding.
// Plain counting on top of the O3/O4 predicates; no tiling of the evaluation.
// ---------------------------------------------------------------------------
void ora_render_counts(const ora_cfg* cfg, int64_t N, int32_t B, const double* rec,
                       const int32_t* flag, const int32_t* rect, const uint32_t* keylo,
                       double thr_ell, int64_t* cand, int64_t* ell, int64_t* con,
                       int64_t* amb) {
  const ora_cfg& c = *cfg;
  const int64_t H = c.height, W = c.width, HW = H * W;
  std::vector<std::vector<int64_t>> order(B);
  for (int32_t v = 0; v < B; ++v) {
    auto& ord = order[v];
    for (int64_t i = 0; i < N; ++i)
      if (flag[(int64_t)v * N + i] == 0) ord.push_back(i);
    if (c.alpha_blend)
      std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
        return keylo[(int64_t)v * N + a] < keylo[(int64_t)v * N + b];
      });
  }
  const double lthr = std::log2(thr_ell);
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t k = 0; k < (int64_t)B * HW; ++k) {
    const int64_t v = k / HW, rem = k % HW, yi = rem / W, xi = rem % W;
    const double px = (double)xi + 0.5, py = (double)yi + 0.5;
    const int64_t tx = xi / c.tile, ty = yi / c.tile;
    int64_t nc = 0, ne = 0, nn = 0, na = 0;
    double T = 1.0;
    for (int64_t i : order[v]) {
      const int64_t o = v * N + i;
      const int32_t* rc = rect + 4 * o;
      if (!(tx >= rc[0] && tx < rc[2] && ty >= rc[1] && ty < rc[3])) continue;
      const double* r = rec + o * ORA_P;
      ++nc;
      pair_eval e;
      eval_pair(r, px, py, e);
      const double aG = r[P_ALPHA] * e.G;
      if (aG >= thr_ell) ++ne;
      if (std::fabs(std::log2(aG) - lthr) < 1e-5) ++na;
      if (!c.alpha_blend) {
        if (e.w >= c.alpha_min) ++nn;
      } else {
        const double a = std::min(c.alpha_max, e.w);
        if (!(a >= c.alpha_min)) continue;
        const double Tn = T * (1.0 - a);
        if (Tn < c.T_min) break;
        T = Tn;
        ++nn;
      }
    }
    cand[k] = nc; ell[k] = ne; con[k] = nn; amb[k] = na;
  }
}

}  // extern "C"
