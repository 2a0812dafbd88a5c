/* ==========================================================================
 * include/wipes.h — C ABI of the B200-native WIPES rasterizer (ABI version 2)
 * ==========================================================================
 * WIPES: Wavelet-based vIsual PrimitivES, arXiv 2508.12615 (/root/reference/
 * PAPER.md). This library implements the paper's one data-parallel hot path,
 * the "fast, differentiable rasterizer" (Sec. 1; PAPER.md:215,
 * Sec. 4.1; Sec. 5): per-primitive preprocess, tile binning
 * with a (tile | depth) key radix sort, per-pixel evaluation of the wavelet
 * primitive W = G * 1/2 [1 + beta cos(f.(x - mu) + phi)] (PAPER.md:187-191,
 * Eq. 6; beta, phi: DESIGN.md R1), accumulated as the weighted sum of Eq. 4
 * or front-to-back alpha blending of Eq. 3, and
 * analytic gradients of every primitive parameter.
 *
 * Conventions for every entry point
 *  - Pointers are DEVICE pointers unless marked (host). Arrays are dense,
 *    row-major, float32 unless noted, and 16-byte aligned (else WIPES_EINVAL).
 *  - The CALLER owns every buffer. The library never allocates or frees device
 *    memory, keeps no state between calls outside `ws`, and launches all work
 *    on `stream` (a cudaStream_t; NULL = legacy default stream).
 *  - It never synchronises, except (a) wipes_preprocess when `n_dup` is
 *    non-NULL and (b) wipes_check_overflow / wipes_timing_collect.
 *  - Status codes only; nothing is thrown across the ABI. Arguments are
 *    validated BEFORE any launch. CUDA launch failures return WIPES_ECUDA with
 *    the detail in wipes_last_error() (thread-local).
 *  - Degenerate primitives are NOT errors ("signals a degenerate
 *    primitive to be skipped"): they are culled — no tiles, no contribution,
 *    zero gradient — and reported in cull_flags: 1 = camera depth outside
 *    [near, far]; 2 = det(Sigma') < det_min or non-positive variance; 3 =
 *    opacity < alpha_min; 4 = off-screen (no tile); 5 = non-finite input.
 *  - Reentrant: calls with distinct workspaces may run concurrently on
 *    distinct streams (kernel timing, when enabled, is process-global).
 * ========================================================================== */
#ifndef WIPES_H
#define WIPES_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WIPES_ABI_VERSION 4
#define WIPES_MAX_CAMERAS_PER_LAUNCH 128 /* more views are processed in chunks */
#define WIPES_GRAD_MOMENTS 12            /* see wipes_get_grad_moments */

typedef enum {
  WIPES_OK = 0,
  WIPES_EINVAL = 1,       /* bad argument; nothing launched                    */
  WIPES_ECAPACITY = 2,    /* dup total > dup_capacity (known on the host)      */
  WIPES_ECUDA = 3,        /* a CUDA call failed; see wipes_last_error()        */
  WIPES_EUNSUPPORTED = 4  /* a mode this build does not implement              */
} wipes_status;

enum { WIPES_PRIM_2D = 0, WIPES_PRIM_3D = 1 };
/* Eq. 4 weighted sum / Eq. 3 alpha blending */
enum { WIPES_BLEND_SUM = 0, WIPES_BLEND_ALPHA = 1 };
/* 2D covariance parameterisations ("Cholesky and RS") */
enum { WIPES_COV2_SIGMA = 0, WIPES_COV2_CHOLESKY = 1, WIPES_COV2_RS = 2 };
/* Eq. 7 as written (beta = 1) / exact z-marginal (NEXT-1,
 * SPEC S:193, R4): with the full ray-space covariance Sigma_hat,
 * S2 its undilated 2x2 block, sigma = Sigma_hat[0:2, 2], v = Sigma_hat_zz -
 * sigma^T S2^-1 sigma, f_hat = (J3 R)^-T f:  f' = f_hat_xy + f_hat_z S2^-1 sigma,
 * beta = exp(-1/2 f_hat_z^2 v). Tile rects, counts and depth keys are the same
 * in both modes; EXACT adds 4 bytes per (view, primitive) to the workspace. */
enum { WIPES_PROJ_PAPER = 0, WIPES_PROJ_EXACT = 1 };
enum { WIPES_COLOR_RGB = 0, WIPES_COLOR_SH = 1 };
/* Render-backward moment accumulation (R37): the per-record gradient
 * moments (sums over a record's pixels of dL/dw-weighted powers of the pixel
 * offset) are summed per lane and reduced per warp in FP32 (AUTO, F32) or with
 * FP64 lane sums, products and warp reduction (F64: removes the accumulation
 * share of the rounding error at ~1.35x the C3 render-backward time; the
 * per-pair FP32/SFU evaluation error, R23b, remains either way). */
enum { WIPES_ACCUM_AUTO = 0, WIPES_ACCUM_F32 = 1, WIPES_ACCUM_F64 = 2 };
/* tile extent: opacity-aware AABB (R7, default) / SPEC's 3-sigma square */
enum { WIPES_EXTENT_OPACITY = 0, WIPES_EXTENT_SIGMA3 = 1 };

/* Pinhole camera, (host) memory. World -> camera x_c = R x_w + t (R row-major),
 * camera axes x right, y down, z forward (the ray-space z of PAPER.md:116-122);
 * pixel (j, i) has centre (j + 0.5, i + 0.5) (R11). */
typedef struct {
  float R[9];
  float t[3];
  float fx, fy, cx, cy;   /* pixels */
  float near_z, far_z;    /* primitives with z outside [near, far] are culled */
} wipes_camera;

typedef struct {
  int32_t width, height;  /* pixels, each in [1, 16384]                        */
  int32_t tile;           /* 8, 16 or 32 (default 16)                          */
  int32_t prim;           /* WIPES_PRIM_*                                      */
  int32_t blend;          /* WIPES_BLEND_*                                     */
  int32_t cov2;           /* WIPES_COV2_* (2D only)                            */
  int32_t proj;           /* WIPES_PROJ_* (3D only)                            */
  int32_t extent;         /* WIPES_EXTENT_*                                    */
  float alpha_min;        /* skip contributions with alpha*W < alpha_min (1/255) */
  float alpha_max;        /* ALPHA: clamp a = min(alpha_max, alpha*W) (0.99)   */
  float T_min;            /* ALPHA: stop when T (1 - a) < T_min (1e-4)         */
  float dilation;         /* added to diag(Sigma') (0.3 px^2 in 3D, 0 in 2D)   */
  float cov_eps;          /* added to diag(Sigma') too (default 0)             */
  float det_min;          /* cull if det(Sigma') < det_min (1e-12)             */
  int32_t ewa_clamp;      /* 1: clamp x/z, y/z at 1.3 x half-FOV inside J      */
  float background[3];    /* ALPHA only                                        */
  int32_t deterministic;  /* 1: bitwise run-to-run deterministic backward: each
                           * warp writes its per-record moments to a slot per
                           * (intersection, footprint) and a gather sums a
                           * record's slots in a fixed order (no float atomics);
                           * the workspace grows by dup_capacity x footprints
                           * x 48 (52 with WIPES_PROJ_EXACT) bytes. */
  /* Image-space sharding: when row_mod > 1 only tile rows ty
   * with ty % row_mod == row_rem are binned and rendered (the rest of the image
   * is left unbinned: zero in SUM mode, background in ALPHA mode, no gradient).
   * Each rank of a row_mod-way split renders its rows; summing the ranks'
   * gradients gives the full-image gradient. 0 / 0 = all rows. */
  int32_t row_mod, row_rem;
  /* Colour (NEXT-3; "color attributes encoded by spherical
   * harmonic coefficients", P:380 settings "aligned with 3DGS"):
   * WIPES_COLOR_RGB reads `color` [N,3]; WIPES_COLOR_SH (3D only) evaluates
   * c = max(0, sum_k Y_k(d) sh[k] + 0.5) per (view, primitive) with
   * d = (mu - C_v) / |mu - C_v|, C_v = -R^T t the camera centre, real SH of
   * degree sh_degree in 0..3 (K = (sh_degree + 1)^2 coefficients, DESIGN.md
   * R33 for the basis and its sign convention). */
  int32_t color_mode;     /* WIPES_COLOR_*                                     */
  int32_t sh_degree;      /* 0..3 (WIPES_COLOR_SH)                             */
  int32_t grad_accum;     /* WIPES_ACCUM_* (ABI v3)                            */
} wipes_config;

/* Primitive parameters (device). Shapes, with N primitives:
 *   2D: mean [N,2] px, cov [N,3] = (sxx, sxy, syy) | (l1, l2, l3) Cholesky
 *       L = [[l1,0],[l2,l3]] | (theta, sx, sy) RS, freq [N,2] rad/px,
 *       depth [N] (ALPHA only: the compositing order key).
 *   3D: mean [N,3], scale [N,3] (activated), quat [N,4] (w,x,y,z; normalised
 *       inside), freq [N,3] rad/world-unit.
 *   both: phase [N] rad (NULL = 0), color [N,3], opacity [N] (activated).
 *   3D with WIPES_COLOR_SH: sh [N, K, 3] (coefficient-major, then RGB) instead
 *       of color.
 * view_stride (3D, counted in PRIMITIVES): view v reads row v*view_stride + i;
 * 0 = one shared set for all B views (static scene), N = per-view sets
 * (6D per-frame parameters, Eq. 8). Gradients are w.r.t. these
 * activated values; activations belong to the caller's autograd. */
typedef struct {
  const float *mean, *cov, *scale, *quat, *freq, *phase, *color, *opacity, *depth;
  int64_t view_stride;
  const float* sh;
} wipes_params;

/* Gradient outputs, same shapes as wipes_params (rows [B*N] when view_stride
 * = N). Overwritten (never accumulated into). NULL = group not written. */
typedef struct {
  float *mean, *cov, *scale, *quat, *freq, *phase, *color, *opacity, *sh;
} wipes_grads;

/* Bytes of opaque workspace for N primitives, B views and room for
 * dup_capacity (view, primitive, tile) intersections. */
size_t wipes_workspace_bytes(const wipes_config* cfg, int64_t N, int32_t B,
                             int64_t dup_capacity);

/* Step 1: per (view, primitive) preprocess — covariance
 * (2D modes / 3D EWA projection PAPER.md:122 + frequency transform :212),
 * conic, opacity-aware extent, tile rect (FP64 decisions, DESIGN.md "Pinned
 * preprocess arithmetic"), 64-byte render record, depth key; then the
 * exclusive scan of tile counts. cams: (host) [B] for 3D, NULL for 2D (B must
 * be 1). n_dup: (host) out, total intersections — when non-NULL the call
 * synchronises `stream` once; NULL keeps it sync-free (capacity protocol).
 * cull_flags: [B*N] uint8 out or NULL. */
wipes_status wipes_preprocess(const wipes_config* cfg, const wipes_params* params,
                              int64_t N, const wipes_camera* cams, int32_t B,
                              void* ws, size_t ws_bytes, int64_t dup_capacity,
                              int64_t* n_dup, uint8_t* cull_flags, void* stream);

/* Step 2 (a4-a6): duplicate each primitive once per overlapped tile under the
 * key ((view*T + tile) << 32) | depth_bits (depth_bits = 0 in SUM mode),
 * stable LSD radix sort of the significant key bits, per-tile CSR ranges.
 * Optional copies for parity tests: keys_out/vals_out [dup_capacity],
 * tile_offsets_out [B*T + 1] int32 (T = ceil(W/tile) * ceil(H/tile)).
 * If the total exceeds dup_capacity nothing past the capacity is written and
 * a device overflow flag is set (see wipes_check_overflow). */
wipes_status wipes_bin_sort(const wipes_config* cfg, int64_t N, int32_t B, void* ws,
                            size_t ws_bytes, int64_t dup_capacity, uint64_t* keys_out,
                            uint32_t* vals_out, int32_t* tile_offsets_out, void* stream);

/* Reads the device total and overflow flag; synchronises `stream`. */
wipes_status wipes_check_overflow(const void* ws, size_t ws_bytes, int64_t* n_dup,
                                  int32_t* overflowed, void* stream);

/* Copies of the preprocess artefacts for parity tests (device outputs, each
 * optional): rect [B*N,4] int32 (tx0, ty0, tx1, ty1), count [B*N] int32,
 * offsets [B*N] int64 (exclusive scan), depth_key [B*N] uint32,
 * records [B*N,16] float32 (the render record). */
wipes_status wipes_get_preprocess(const wipes_config* cfg, int64_t N, int32_t B,
                                  const void* ws, size_t ws_bytes, int64_t dup_capacity,
                                  int32_t* rect, int32_t* count, int64_t* offsets,
                                  uint32_t* depth_key, float* records, void* stream);

/* Step 3 (a7/a8): render. image [B,3,H,W] (planar); ALPHA mode also writes
 * T_final [B,H,W] and n_contrib [B,H,W] int32 (one past the tile-list index of
 * the last composited entry), both needed by wipes_render_bwd. */
wipes_status wipes_render_fwd(const wipes_config* cfg, int64_t N, int32_t B, void* ws,
                              size_t ws_bytes, int64_t dup_capacity, float* image,
                              float* T_final, int32_t* n_contrib, void* stream);

/* Step 4 (a9-a12): gradients of L given dL/dimage [B,3,H,W] w.r.t. every
 * parameter group ("explicit gradients for all parameters"):
 * per-pair analytic terms accumulated as 12 per-record moments, reduced per
 * warp with shuffles, then one atomic per (warp, record, moment) into the
 * workspace; then the preprocess chain rule (FP64) into `grads`. The same params/cams as the
 * forward call must be passed. */
wipes_status wipes_render_bwd(const wipes_config* cfg, const wipes_params* params,
                              int64_t N, const wipes_camera* cams, int32_t B, void* ws,
                              size_t ws_bytes, int64_t dup_capacity,
                              const float* dL_dimage, const float* T_final,
                              const int32_t* n_contrib, wipes_grads* grads, void* stream);

/* Step 4 in two calls, so a multi-GPU caller can overlap the gradient
 * all-reduce with the chain rule:
 * wipes_render_bwd_moments = the render backward into the workspace moments
 * (same arguments as wipes_render_bwd minus params/cams/grads); then
 * wipes_preprocess_bwd writes the parameter-gradient rows [row0, row1) —
 * primitives for a shared parameter set (view_stride = 0, or 2D), (view,
 * primitive) rows for per-frame sets — and may be called once per row chunk,
 * each chunk's rows complete when its call's work on `stream` completes.
 * wipes_render_bwd == moments + preprocess_bwd(0, rows). Rows outside
 * [row0, row1) are not written. row1 < 0 means all rows. */
wipes_status wipes_render_bwd_moments(const wipes_config* cfg, int64_t N, int32_t B, void* ws,
                                      size_t ws_bytes, int64_t dup_capacity,
                                      const float* dL_dimage, const float* T_final,
                                      const int32_t* n_contrib, void* stream);
wipes_status wipes_preprocess_bwd(const wipes_config* cfg, const wipes_params* params, int64_t N,
                                  const wipes_camera* cams, int32_t B, void* ws, size_t ws_bytes,
                                  int64_t dup_capacity, wipes_grads* grads, int64_t row0,
                                  int64_t row1, void* stream);

/* The 12 per-record gradient MOMENTS [B*N, 12] (float32) accumulated by the
 * last wipes_render_bwd, for tests and inspection. With gw = dL/dw of a valid
 * (pixel, record) pair, w = alpha W, ag = alpha G, d = pixel - mu', sums over
 * the record's pairs: M0 = gw w, M1 = gw w dx, M2 = gw w dy, M3 = gw w dx^2,
 * M4 = gw w dx dy, M5 = gw w dy^2, M6 = gw ag sin(theta), M7 = M6 dx,
 * M8 = M6 dy, M9..M11 = dL/dc (w g, or a T g in ALPHA mode). The record
 * gradients are linear in them. */
wipes_status wipes_get_grad_moments(const wipes_config* cfg, int64_t N, int32_t B,
                                    const void* ws, size_t ws_bytes, int64_t dup_capacity,
                                    float* out, void* stream);

/* Measurement only (not on the hot path): runs a counting variant of the
 * forward render kernel over the workspace of the last preprocess/bin_sort
 * and writes stats3 (device, 3 x uint64): [0] tile-method candidate pairs
 * (tile-list entries x in-image pixels, up to each pixel's termination in
 * ALPHA mode), [1] in-ellipse pairs (alpha*G >= alpha_min), [2] contributing
 * pairs (alpha*W >= alpha_min; composited in ALPHA mode). These are the
 * algorithmic work units of the render roofline. */
wipes_status wipes_render_stats(const wipes_config* cfg, int64_t N, int32_t B, void* ws,
                                size_t ws_bytes, int64_t dup_capacity, uint64_t* stats3,
                                void* stream);

/* ---- NEXT-2: the image-fitting step around the rasterizer --
 * One fitting iteration (Eq. 4 objective,
 * PAPER.md:299 "all hyperparameters were kept consistent with GSImage") is
 *   preprocess -> bin_sort -> render_fwd -> wipes_loss_l2 -> render_bwd ->
 *   wipes_adam_step,
 * all on one stream and graph-capturable (no host synchronisation: the Adam
 * step counter lives in device memory, and an optional device guard word
 * (wipes_overflow_flag) turns the update into a no-op for a step whose
 * intersections overflowed the capacity). */

/* Bytes of scratch (device) shared by wipes_loss_l2 and wipes_adam_step; zero
 * it once before first use (the calls leave their counters at zero). */
size_t wipes_train_scratch_bytes(void);

/* L2 objective, mean over the n floats (B*3*H*W) of image vs target (SPEC
 * S:336 "returns pre-update L2 loss (mean over pixels and channels)"):
 *   loss = (1/n) sum (image - target)^2   (device double, written once),
 *   dL_dimage = (2/n) (image - target)    (device float [n]).
 * The sum is reduced in FP64 in a fixed order (run-to-run deterministic).
 * image/target/dL_dimage: device [n] float32, 4-byte aligned; dL_dimage may
 * alias neither input. */
wipes_status wipes_loss_l2(const float* image, const float* target, int64_t n,
                           float* dL_dimage, double* loss, void* scratch, void* stream);

/* Parameter activations ("opacity_raw = 0 (opacity 0.5)"). */
enum { WIPES_ACT_NONE = 0, WIPES_ACT_SIGMOID = 1 };
#define WIPES_MAX_ADAM_GROUPS 8

/* One parameter group (all pointers device float32 [n]):
 * param   raw parameter theta (in/out),
 * grad    dL/d(act(theta)) as produced by wipes_render_bwd (in),
 * m, v    Adam moments (in/out; zero-initialised by the caller),
 * act     act(theta) written after the update (the rasterizer's input for the
 *         next step); NULL when activation == WIPES_ACT_NONE (the rasterizer
 *         reads param directly). */
typedef struct {
  float* param;
  const float* grad;
  float* m;
  float* v;
  float* act;
  int64_t n;
  float lr;
  int32_t activation;
} wipes_adam_group;

/* Adam (Kingma & Ba; SPEC S:321-324 AdamState, beta1 0.9, beta2 0.999,
 * eps 1e-15), one launch for all groups. With t = *step + 1:
 *   g  = grad * act'(theta)          (chain through the activation),
 *   m  = b1 m + (1 - b1) g,  v = b2 v + (1 - b2) g^2,
 *   theta -= lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps),
 *   act = act(theta),  *step = t.
 * step: device int64 (in/out). guard: device int32 or NULL — when *guard != 0
 * nothing is modified (used with wipes_overflow_flag). */
wipes_status wipes_adam_step(const wipes_adam_group* groups, int32_t n_groups, float beta1,
                             float beta2, float eps, int64_t* step, const int32_t* guard,
                             void* scratch, void* stream);

/* act = act(param) for every group with an activation (initialisation). */
wipes_status wipes_activate(const wipes_adam_group* groups, int32_t n_groups, void* stream);

/* Device address of the workspace's capacity-overflow word (int32, set by
 * wipes_preprocess when the intersections exceed dup_capacity). */
const int32_t* wipes_overflow_flag(const void* ws);

/* ---- NEXT-4: tcgen05 bf16 GEMM (building block of the deformation MLP) ----
 * D[M x N] = sum_k A(m, k) B(n, k) with bf16 operands and fp32 accumulation on
 * the 5th-generation tensor cores (tcgen05.mma, accumulator in TMEM), followed
 * by a fused epilogue. Operand layouts (device, bf16): A K-major: (m, k) at
 * A[m * lda + k]; A MN-major: (m, k) at A[k * lda + m]; B likewise with n.
 * Requirements: K, lda, ldb multiples of 8; pointers 16-byte aligned; N <= 256
 * per launch tile (larger N is tiled). split_k > 1 splits K over CTAs (only
 * with WIPES_GEMM_EPI_ATOMIC_F32). */
enum {
  WIPES_GEMM_EPI_STORE_F32 = 0,      /* C (f32) = D                           */
  WIPES_GEMM_EPI_BIAS_F32 = 1,       /* C (f32) = D + bias[n]                 */
  WIPES_GEMM_EPI_BIAS_RELU_BF16 = 2, /* C (bf16) = relu(D + bias[n])          */
  WIPES_GEMM_EPI_MASK_BF16 = 3,      /* C (bf16) = D * (mask(m, n) > 0)       */
  WIPES_GEMM_EPI_ATOMIC_F32 = 4      /* C (f32) += D (atomic)                 */
};
typedef struct {
  const void* A;
  const void* B;
  void* C;
  const float* bias;  /* [N] f32 (BIAS epilogues)                              */
  const void* mask;   /* bf16, (m, n) at mask[m * ldm + n] (MASK epilogue)      */
  int64_t M, N, K;
  int64_t lda, ldb, ldc, ldm;
  int32_t a_mn_major, b_mn_major, epilogue, split_k;
  float* colsum;      /* optional [N] f32: += column sums of the epilogue result
                         over the rows (atomic; e.g. a bias gradient), or NULL */
  int64_t split3;     /* bf16 epilogues (ABI v4): 0 = C holds bf16(v); > 0 = C
                         holds the split-bf16 triple of v (R38):
                         C[m, n] = C[m, n + split3] = hi = bf16(v),
                         C[m, n + 2 split3] = lo = bf16(v - hi), so that a
                         following GEMM over [hi | hi | lo] against weights
                         [W_hi | W_lo | W_hi] forms hi W_hi + hi W_lo + lo W_hi */
} wipes_gemm_args;
wipes_status wipes_gemm_bf16(const wipes_gemm_args* args, void* stream);

/* ---- NEXT-4: the time-conditioned deformation field (Eq. 8;
 * network of D-3DGS, Eq. 5; R34-R36) ----------------------
 * (dx, dq, ds, df) = F_theta(gamma(x), gamma(t)): positional encoding
 * gamma_L(p) = [p, sin(2^k p), cos(2^k p)]_(k<L) of the canonical centre x (Lx)
 * and the frame time t (Lt); `depth` ReLU layers of `width`, the input
 * re-concatenated after layer `skip` ([gamma, h]); a 13-output linear head.
 * Per-frame parameters: mu_t = mu + dx, q_t = q + dq, s_t = s exp(ds),
 * f_t = f + df (x enters through a stop-gradient). Every layer is a tcgen05
 * GEMM (bf16 operands rounded to nearest even, fp32 accumulation) with a fused
 * bias + ReLU epilogue; theta stays fp32 (flat layout: W_l [width, K_l]
 * row-major then b_l [width] for each layer, then W_h [13, width], b_h [13];
 * K_0 = E = 3(1+2Lx) + 1+2Lt, K_(skip+1) = E + width, else width). */
typedef struct {
  int32_t width;   /* multiple of 16, 16..256 (D-3DGS: 256) */
  int32_t depth;   /* >= 1 (D-3DGS: 8)                      */
  int32_t skip;    /* -1 (none) or 0..depth-2 (D-3DGS: 4)    */
  int32_t Lx, Lt;  /* encoding frequencies (D-3DGS: 10, 6)   */
  int32_t precision; /* ABI v4: WIPES_MLP_BF16X3 (0, default) = every operand
                      * carried as a split-bf16 pair v = hi + lo (hi = bf16(v),
                      * lo = bf16(v - hi)) and every product as hi.hi + hi.lo +
                      * lo.hi on the bf16 tensor cores (one GEMM over
                      * concatenated [hi | hi | lo] x [W_hi | W_lo | W_hi]
                      * operands, fp32 accumulation; ~2^-16 relative operands,
                      * close to the FP32 network of D-3DGS, R38);
                      * WIPES_MLP_BF16 (1) = single bf16 operands (faster, R36) */
} wipes_mlp_config;
enum { WIPES_MLP_BF16X3 = 0, WIPES_MLP_BF16 = 1 };

size_t wipes_mlp_param_count(const wipes_mlp_config* cfg);
/* Workspace for F*N rows; the forward keeps its activations there for the
 * backward of the same rows. */
size_t wipes_mlp_workspace_bytes(const wipes_mlp_config* cfg, int64_t rows);
/* Frame f, primitive i -> row f*N + i. times: (host) [F]. canon: mean, quat,
 * scale, freq [N] (+ phase, color, opacity, sh copied to the frame rows when
 * both canon and frame pointers are non-NULL); frame: the same groups, [F*N]
 * rows (device, caller-owned), ready for the rasterizer with view_stride = N.
 * train: 1 keeps every layer's activations in `ws` for wipes_mlp_backward;
 * 0 (inference) writes only the frame rows. When width is a multiple of 64,
 * depth <= 8 and F <= 128, inference runs all layers of a 128-row tile fused on
 * chip; training runs layer by layer (width 256: the 256-input hidden layers
 * use a kernel in which CTA pairs split the output columns). Deterministic:
 * fixed-order fp32 accumulation, no atomics. */
wipes_status wipes_mlp_forward(const wipes_mlp_config* cfg, const float* theta, int64_t N,
                               int32_t F, const float* times, const wipes_params* canon,
                               const wipes_params* frame, int32_t sh_coeffs, int32_t train,
                               void* ws, size_t ws_bytes, void* stream);
/* From g_frame (gradients w.r.t. the frame rows' mean, quat, scale, freq) of
 * the last wipes_mlp_forward on this workspace: g_theta [param_count] (fp32,
 * overwritten) and g_canon mean/quat/scale/freq [N] (overwritten; mean is the
 * frame sum: stop-gradient into the network). At width 256 each hidden layer
 * after the first computes its input gradient, weight gradient and the bias
 * gradient below it in one pass (per-CTA-pair partial sums, reduced in a fixed
 * order); the head, layer 0 and the encoding columns of the skip layer use
 * split-K GEMMs with fp32 atomics (run-to-run differences at rounding level). */
wipes_status wipes_mlp_backward(const wipes_mlp_config* cfg, const float* theta, int64_t N,
                                int32_t F, const wipes_params* canon, const wipes_grads* g_frame,
                                float* g_theta, const wipes_grads* g_canon, void* ws,
                                size_t ws_bytes, void* stream);

/* Instrumentation: per-kernel CUDA-event timing (process-global, not for use
 * during graph capture) and a launch counter. */
int          wipes_num_kernels(void);
const char*  wipes_kernel_name(int kernel_id);
void         wipes_timing_enable(int on);
/* Synchronises on the recorded events; fills ms[k] (summed device time) and
 * launches[k] per kernel id since the last collect, then resets. */
wipes_status wipes_timing_collect(double* ms, int64_t* launches, int n);
int64_t      wipes_launch_count(void);

const char*  wipes_status_string(wipes_status s);
const char*  wipes_last_error(void);
int          wipes_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* WIPES_H */
