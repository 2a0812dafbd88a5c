// C-ABI entry points of libwipes.so (include/wipes.h): argument validation
// before any launch, workspace carving, kernel sequencing on the caller's
// stream, optional per-kernel CUDA-event timing and a launch counter.
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

// NVTX range around each north-star ABI call (visible in nsys / ncu --nvtx;
// header-only NVTX3: a no-op unless a tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

namespace wipes {

namespace {

thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};

// ---- timing: a pool of event pairs recorded around each launch ------------
struct TimedLaunch {
  int kid;
  cudaEvent_t a, b;
};
std::mutex g_tmu;
bool g_timing = false;
std::vector<cudaEvent_t> g_pool;
std::vector<TimedLaunch> g_log;
cudaEvent_t g_pending = nullptr;

cudaEvent_t take_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

const char* kNames[K_NUM] = {
    "preprocess2d", "preprocess3d", "scan_blocks", "scan_sums", "duplicate", "radix_hist",
    "radix_scan_blocks", "radix_scan_sums", "radix_scatter", "tile_ranges", "render_fwd",
    "render_bwd", "preprocess2d_bwd", "preprocess3d_bwd", "memset", "tile_order", "loss_l2",
    "adam", "sh_bwd", "gemm_tc", "mlp_misc", "det_gather"};

wipes_status fail(wipes_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

wipes_status cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return WIPES_ECUDA;
}

bool aligned(const void* p, size_t a) { return ((uintptr_t)p % a) == 0; }

wipes_status check_cfg(const wipes_config* c, int64_t N, int32_t B) {
  if (!c) return fail(WIPES_EINVAL, "cfg is NULL");
  if (c->width < 1 || c->width > 16384 || c->height < 1 || c->height > 16384)
    return fail(WIPES_EINVAL, "width/height must be in [1, 16384]");
  if (c->tile != 8 && c->tile != 16 && c->tile != 32)
    return fail(WIPES_EINVAL, "tile must be 8, 16 or 32");
  if (c->prim != WIPES_PRIM_2D && c->prim != WIPES_PRIM_3D) return fail(WIPES_EINVAL, "prim");
  if (c->blend != WIPES_BLEND_SUM && c->blend != WIPES_BLEND_ALPHA)
    return fail(WIPES_EINVAL, "blend");
  if (c->cov2 < 0 || c->cov2 > 2) return fail(WIPES_EINVAL, "cov2");
  if (c->proj != WIPES_PROJ_PAPER && c->proj != WIPES_PROJ_EXACT) return fail(WIPES_EINVAL, "proj");
  if (c->extent != WIPES_EXTENT_OPACITY && c->extent != WIPES_EXTENT_SIGMA3)
    return fail(WIPES_EINVAL, "extent");
  if (c->color_mode != WIPES_COLOR_RGB && c->color_mode != WIPES_COLOR_SH)
    return fail(WIPES_EINVAL, "color_mode");
  if (c->color_mode == WIPES_COLOR_SH && c->prim != WIPES_PRIM_3D)
    return fail(WIPES_EINVAL, "color_mode SH needs 3D primitives");
  if (c->color_mode == WIPES_COLOR_SH && (c->sh_degree < 0 || c->sh_degree > 3))
    return fail(WIPES_EINVAL, "sh_degree must be in 0..3");
  if (c->deterministic != 0 && c->deterministic != 1) return fail(WIPES_EINVAL, "deterministic");
  if (c->grad_accum < WIPES_ACCUM_AUTO || c->grad_accum > WIPES_ACCUM_F64)
    return fail(WIPES_EINVAL, "grad_accum");
  if (!(c->alpha_min >= 0.f) || !(c->alpha_max > c->alpha_min) || !(c->alpha_max <= 1.f))
    return fail(WIPES_EINVAL, "need 0 <= alpha_min < alpha_max <= 1");
  if (!(c->T_min >= 0.f) || !(c->T_min < 1.f)) return fail(WIPES_EINVAL, "T_min");
  if (c->row_mod < 0 || (c->row_mod > 1 && (c->row_rem < 0 || c->row_rem >= c->row_mod)))
    return fail(WIPES_EINVAL, "row_mod / row_rem");
  if (N < 0 || N > ((int64_t)1 << 31) - 1) return fail(WIPES_EINVAL, "N out of range");
  if (B < 1) return fail(WIPES_EINVAL, "B must be >= 1");
  if (c->prim == WIPES_PRIM_2D && B != 1) return fail(WIPES_EINVAL, "2D primitives need B == 1");
  int64_t GX = (c->width + c->tile - 1) / c->tile, GY = (c->height + c->tile - 1) / c->tile;
  if (GX * GY * (int64_t)B >= ((int64_t)1 << 31)) return fail(WIPES_EINVAL, "B*T >= 2^31");
  return WIPES_OK;
}

wipes_status check_ws(const Layout& L, const void* ws, size_t ws_bytes, int64_t cap) {
  if (cap < 0 || cap >= ((int64_t)1 << 30)) return fail(WIPES_EINVAL, "dup_capacity must be in [0, 2^30)");
  if (!ws) return fail(WIPES_EINVAL, "ws is NULL");
  if (!aligned(ws, 256)) return fail(WIPES_EINVAL, "ws must be 256-byte aligned");
  if (ws_bytes < L.total) return fail(WIPES_EINVAL, "ws_bytes smaller than wipes_workspace_bytes");
  return WIPES_OK;
}

#define REQ(ptr, name)                                                        \
  do {                                                                        \
    if (!(ptr)) return fail(WIPES_EINVAL, std::string(name) + " is NULL");    \
    if (!aligned((ptr), 4)) return fail(WIPES_EINVAL, std::string(name) + " misaligned"); \
  } while (0)

wipes_status check_params(const wipes_config* c, const wipes_params* p, int64_t N, int32_t B) {
  if (!p) return fail(WIPES_EINVAL, "params is NULL");
  if (N == 0) return WIPES_OK;
  REQ(p->mean, "mean");
  REQ(p->freq, "freq");
  if (c->color_mode == WIPES_COLOR_SH) REQ(p->sh, "sh");
  else REQ(p->color, "color");
  REQ(p->opacity, "opacity");
  if (p->phase && !aligned(p->phase, 4)) return fail(WIPES_EINVAL, "phase misaligned");
  if (c->prim == WIPES_PRIM_2D) {
    REQ(p->cov, "cov");
    if (c->blend == WIPES_BLEND_ALPHA) REQ(p->depth, "depth (2D alpha blending)");
  } else {
    REQ(p->scale, "scale");
    REQ(p->quat, "quat");
    if (p->view_stride != 0 && p->view_stride != N)
      return fail(WIPES_EINVAL, "view_stride must be 0 or N");
    (void)B;
  }
  return WIPES_OK;
}

}  // namespace

void launch_begin(int kid, cudaStream_t s) {
  if (kid != K_MEMSET) g_launches.fetch_add(1, std::memory_order_relaxed);  // kernels only
  if (!g_timing) return;
  std::lock_guard<std::mutex> lk(g_tmu);
  g_pending = take_event();
  cudaEventRecord(g_pending, s);
  (void)kid;
}

void launch_end(int kid, cudaStream_t s) {
  if (!g_timing) return;
  std::lock_guard<std::mutex> lk(g_tmu);
  cudaEvent_t b = take_event();
  cudaEventRecord(b, s);
  g_log.push_back({kid, g_pending, b});
  g_pending = nullptr;
}

}  // namespace wipes

using namespace wipes;

extern "C" {

size_t wipes_workspace_bytes(const wipes_config* cfg, int64_t N, int32_t B, int64_t cap) {
  if (!cfg || check_cfg(cfg, N, B) != WIPES_OK) return 0;
  return make_layout(*cfg, N, B, cap).total;
}

wipes_status wipes_preprocess(const wipes_config* cfg, const wipes_params* params, int64_t N,
                              const wipes_camera* cams, int32_t B, void* ws, size_t ws_bytes,
                              int64_t dup_capacity, int64_t* n_dup, uint8_t* cull_flags,
                              void* stream) {
  NvtxRange nvtx_range("wipes_preprocess");
  wipes_status st = check_cfg(cfg, N, B);
  if (st != WIPES_OK) return st;
  st = check_params(cfg, params, N, B);
  if (st != WIPES_OK) return st;
  if (cfg->prim == WIPES_PRIM_3D && !cams) return fail(WIPES_EINVAL, "cams is NULL (3D)");
  Layout L = make_layout(*cfg, N, B, dup_capacity);
  st = check_ws(L, ws, ws_bytes, dup_capacity);
  if (st != WIPES_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  char* w = (char*)ws;
  cudaError_t e = cfg->prim == WIPES_PRIM_2D
                      ? launch_preprocess2d(*cfg, *params, L, w, cull_flags, s)
                      : launch_preprocess3d(*cfg, *params, L, cams, w, cull_flags, s);
  if (e != cudaSuccess) return cuda_fail(e, "preprocess launch");
  e = launch_scan_counts(L, w, s);
  if (e != cudaSuccess) return cuda_fail(e, "scan launch");
  if (n_dup) {
    WsHeader h;
    e = cudaMemcpyAsync(&h, w + L.hdr, sizeof(h), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "n_dup readback");
    *n_dup = h.total;
    if (h.total > dup_capacity)
      return fail(WIPES_ECAPACITY, "tile intersections exceed dup_capacity");
  }
  return WIPES_OK;
}

wipes_status wipes_bin_sort(const wipes_config* cfg, int64_t N, int32_t B, void* ws,
                            size_t ws_bytes, int64_t dup_capacity, uint64_t* keys_out,
                            uint32_t* vals_out, int32_t* tile_offsets_out, void* stream) {
  NvtxRange nvtx_range("wipes_bin_sort");
  wipes_status st = check_cfg(cfg, N, B);
  if (st != WIPES_OK) return st;
  Layout L = make_layout(*cfg, N, B, dup_capacity);
  st = check_ws(L, ws, ws_bytes, dup_capacity);
  if (st != WIPES_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  char* w = (char*)ws;
  int fb = 0;
  cudaError_t e = launch_bin_sort(*cfg, L, w, s, &fb);
  if (e != cudaSuccess) return cuda_fail(e, "bin_sort launch");
  if (keys_out && L.cap) e = launch_keys64(L, w, fb, keys_out, s);
  if (e == cudaSuccess && vals_out && L.cap) e = launch_vals_copy(L, w, fb, vals_out, s);
  if (e == cudaSuccess && tile_offsets_out)
    e = cudaMemcpyAsync(tile_offsets_out, w + L.toff, 4 * (L.BT + 1), cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return cuda_fail(e, "bin_sort copies");
  return WIPES_OK;
}

wipes_status wipes_check_overflow(const void* ws, size_t ws_bytes, int64_t* n_dup,
                                  int32_t* overflowed, void* stream) {
  if (!ws || ws_bytes < sizeof(WsHeader)) return fail(WIPES_EINVAL, "ws");
  cudaStream_t s = (cudaStream_t)stream;
  WsHeader h;
  cudaError_t e = cudaMemcpyAsync(&h, ws, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_fail(e, "check_overflow");
  if (n_dup) *n_dup = h.total;
  if (overflowed) *overflowed = h.overflow;
  return WIPES_OK;
}

wipes_status wipes_get_preprocess(const wipes_config* cfg, int64_t N, int32_t B, const void* ws,
                                  size_t ws_bytes, int64_t dup_capacity, int32_t* rect,
                                  int32_t* count, int64_t* offsets, uint32_t* depth_key,
                                  float* records, void* stream) {
  wipes_status st = check_cfg(cfg, N, B);
  if (st != WIPES_OK) return st;
  Layout L = make_layout(*cfg, N, B, dup_capacity);
  st = check_ws(L, ws, ws_bytes, dup_capacity);
  if (st != WIPES_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const char* w = (const char*)ws;
  cudaError_t e = cudaSuccess;
  if (L.BN == 0) return WIPES_OK;
  if (rect) e = cudaMemcpyAsync(rect, w + L.rect, 16 * L.BN, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && count)
    e = cudaMemcpyAsync(count, w + L.count, 4 * L.BN, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && depth_key)
    e = cudaMemcpyAsync(depth_key, w + L.dkey, 4 * L.BN, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && records)
    e = cudaMemcpyAsync(records, w + L.rec, 64 * L.BN, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && offsets) e = launch_offsets_copy(L, w, offsets, s);
  if (e != cudaSuccess) return cuda_fail(e, "get_preprocess copies");
  return WIPES_OK;
}

wipes_status wipes_render_fwd(const wipes_config* cfg, int64_t N, int32_t B, void* ws,
                              size_t ws_bytes, int64_t dup_capacity, float* image, float* T_final,
                              int32_t* n_contrib, void* stream) {
  NvtxRange nvtx_range("wipes_render_fwd");
  wipes_status st = check_cfg(cfg, N, B);
  if (st != WIPES_OK) return st;
  Layout L = make_layout(*cfg, N, B, dup_capacity);
  st = check_ws(L, ws, ws_bytes, dup_capacity);
  if (st != WIPES_OK) return st;
  if (!image || !aligned(image, 4)) return fail(WIPES_EINVAL, "image NULL or misaligned");
  if (cfg->blend == WIPES_BLEND_ALPHA && (!T_final || !n_contrib))
    return fail(WIPES_EINVAL, "ALPHA mode needs T_final and n_contrib");
  cudaError_t e = launch_render_fwd(*cfg, L, (char*)ws, final_buffer_is_b(L), image, T_final,
                                    n_contrib, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "render_fwd launch");
  return WIPES_OK;
}

static wipes_status render_bwd_moments(const wipes_config* cfg, const Layout& L, void* ws,
                                       const float* dL_dimage, const float* T_final,
                                       const int32_t* n_contrib, cudaStream_t s) {
  if (!dL_dimage || !aligned(dL_dimage, 4)) return fail(WIPES_EINVAL, "dL_dimage");
  if (cfg->blend == WIPES_BLEND_ALPHA && (!T_final || !n_contrib))
    return fail(WIPES_EINVAL, "ALPHA mode needs T_final and n_contrib");
  char* w = (char*)ws;
  cudaError_t e = cudaSuccess;
  if (L.BN > 0) {
    launch_begin(K_MEMSET, s);
    e = cudaMemsetAsync(w + L.rgrad, 0, sizeof(float) * kMoments * L.BN, s);
    if (e == cudaSuccess && L.exact) e = cudaMemsetAsync(w + L.rbeta, 0, sizeof(float) * L.BN, s);
    if (e == cudaSuccess && L.det && L.cap)
      e = cudaMemsetAsync(w + L.slotmask, 0, (size_t)L.cap * L.fps, s);
    launch_end(K_MEMSET, s);
    if (e != cudaSuccess) return cuda_fail(e, "rgrad memset");
  }
  e = launch_render_bwd(*cfg, L, w, final_buffer_is_b(L), dL_dimage, T_final, n_contrib, s);
  if (e != cudaSuccess) return cuda_fail(e, "render_bwd launch");
  if (L.det) {
    e = launch_det_gather(L, w, s);
    if (e != cudaSuccess) return cuda_fail(e, "det_gather launch");
  }
  return WIPES_OK;
}

static wipes_status preprocess_bwd(const wipes_config* cfg, const wipes_params* params,
                                   const wipes_camera* cams, const Layout& L, void* ws,
                                   wipes_grads* grads, int64_t row0, int64_t row1,
                                   cudaStream_t s) {
  if (!grads) return fail(WIPES_EINVAL, "grads is NULL");
  if (cfg->prim == WIPES_PRIM_3D && !cams) return fail(WIPES_EINVAL, "cams is NULL (3D)");
  if (row0 < 0 || (row1 >= 0 && row1 < row0)) return fail(WIPES_EINVAL, "row0 / row1");
  char* w = (char*)ws;
  cudaError_t e = cfg->prim == WIPES_PRIM_2D
                      ? launch_preprocess2d_bwd(*cfg, *params, L, w, *grads, s, row0, row1)
                      : launch_preprocess3d_bwd(*cfg, *params, L, cams, w, *grads, s, row0, row1);
  if (e != cudaSuccess) return cuda_fail(e, "preprocess_bwd launch");
  return WIPES_OK;
}

wipes_status wipes_render_bwd(const wipes_config* cfg, const wipes_params* params, int64_t N,
                              const wipes_camera* cams, int32_t B, void* ws, size_t ws_bytes,
                              int64_t dup_capacity, const float* dL_dimage, const float* T_final,
                              const int32_t* n_contrib, wipes_grads* grads, void* stream) {
  NvtxRange nvtx_range("wipes_render_bwd");
  wipes_status st = check_cfg(cfg, N, B);
  if (st != WIPES_OK) return st;
  st = check_params(cfg, params, N, B);
  if (st != WIPES_OK) return st;
  Layout L = make_layout(*cfg, N, B, dup_capacity);
  st = check_ws(L, ws, ws_bytes, dup_capacity);
  if (st != WIPES_OK) return st;
  if (!grads) return fail(WIPES_EINVAL, "grads is NULL");
  if (cfg->prim == WIPES_PRIM_3D && !cams) return fail(WIPES_EINVAL, "cams is NULL (3D)");
  cudaStream_t s = (cudaStream_t)stream;
  st = render_bwd_moments(cfg, L, ws, dL_dimage, T_final, n_contrib, s);
  if (st != WIPES_OK) return st;
  return preprocess_bwd(cfg, params, cams, L, ws, grads, 0, -1, s);
}

wipes_status wipes_render_bwd_moments(const wipes_config* cfg, int64_t N, int32_t B, void* ws,
                                      size_t ws_bytes, int64_t dup_capacity,
                                      const float* dL_dimage, const float* T_final,
                                      const int32_t* n_contrib, void* stream) {
  NvtxRange nvtx_range("wipes_render_bwd_moments");
  wipes_status st = check_cfg(cfg, N, B);
  if (st != WIPES_OK) return st;
  Layout L = make_layout(*cfg, N, B, dup_capacity);
  st = check_ws(L, ws, ws_bytes, dup_capacity);
  if (st != WIPES_OK) return st;
  return render_bwd_moments(cfg, L, ws, dL_dimage, T_final, n_contrib, (cudaStream_t)stream);
}

wipes_status wipes_preprocess_bwd(const wipes_config* cfg, const wipes_params* params, int64_t N,
                                  const wipes_camera* cams, int32_t B, void* ws, size_t ws_bytes,
                                  int64_t dup_capacity, wipes_grads* grads, int64_t row0,
                                  int64_t row1, void* stream) {
  NvtxRange nvtx_range("wipes_preprocess_bwd");
  wipes_status st = check_cfg(cfg, N, B);
  if (st != WIPES_OK) return st;
  st = check_params(cfg, params, N, B);
  if (st != WIPES_OK) return st;
  Layout L = make_layout(*cfg, N, B, dup_capacity);
  st = check_ws(L, ws, ws_bytes, dup_capacity);
  if (st != WIPES_OK) return st;
  return preprocess_bwd(cfg, params, cams, L, ws, grads, row0, row1, (cudaStream_t)stream);
}

wipes_status wipes_get_grad_moments(const wipes_config* cfg, int64_t N, int32_t B, const void* ws,
                                    size_t ws_bytes, int64_t dup_capacity, float* out,
                                    void* stream) {
  wipes_status st = check_cfg(cfg, N, B);
  if (st != WIPES_OK) return st;
  Layout L = make_layout(*cfg, N, B, dup_capacity);
  st = check_ws(L, ws, ws_bytes, dup_capacity);
  if (st != WIPES_OK) return st;
  if (!out) return fail(WIPES_EINVAL, "out is NULL");
  if (L.BN == 0) return WIPES_OK;
  cudaError_t e = cudaMemcpyAsync(out, (const char*)ws + L.rgrad, 4 * kMoments * L.BN,
                                  cudaMemcpyDeviceToDevice, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "get_grad_moments");
  return WIPES_OK;
}

wipes_status wipes_render_stats(const wipes_config* cfg, int64_t N, int32_t B, void* ws,
                                size_t ws_bytes, int64_t dup_capacity, uint64_t* stats3,
                                void* stream) {
  wipes_status st = check_cfg(cfg, N, B);
  if (st != WIPES_OK) return st;
  Layout L = make_layout(*cfg, N, B, dup_capacity);
  st = check_ws(L, ws, ws_bytes, dup_capacity);
  if (st != WIPES_OK) return st;
  if (!stats3 || !aligned(stats3, 8)) return fail(WIPES_EINVAL, "stats3");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(stats3, 0, 3 * sizeof(uint64_t), s);
  if (e == cudaSuccess)
    e = launch_render_fwd(*cfg, L, (char*)ws, final_buffer_is_b(L), nullptr, nullptr, nullptr, s,
                          (unsigned long long*)stats3);
  if (e != cudaSuccess) return cuda_fail(e, "render_stats");
  return WIPES_OK;
}

size_t wipes_train_scratch_bytes(void) { return train_scratch_bytes(); }

wipes_status wipes_loss_l2(const float* image, const float* target, int64_t n, float* dL_dimage,
                           double* loss, void* scratch, void* stream) {
  if (n < 0) return fail(WIPES_EINVAL, "n < 0");
  if (!image || !target || !dL_dimage || !loss || !scratch)
    return fail(WIPES_EINVAL, "image, target, dL_dimage, loss and scratch must be non-NULL");
  if (!aligned(image, 4) || !aligned(target, 4) || !aligned(dL_dimage, 4) || !aligned(loss, 8) ||
      !aligned(scratch, 16))
    return fail(WIPES_EINVAL, "misaligned pointer");
  if (dL_dimage == image || dL_dimage == target)
    return fail(WIPES_EINVAL, "dL_dimage aliases an input");
  cudaError_t e = launch_loss_l2(image, target, n, dL_dimage, loss, scratch, (cudaStream_t)stream);
  return e == cudaSuccess ? WIPES_OK : cuda_fail(e, "loss_l2 launch");
}

static wipes_status check_groups(const wipes_adam_group* g, int32_t ng, bool need_grad) {
  if (!g || ng < 1 || ng > WIPES_MAX_ADAM_GROUPS)
    return fail(WIPES_EINVAL, "need 1 <= n_groups <= WIPES_MAX_ADAM_GROUPS");
  for (int k = 0; k < ng; ++k) {
    if (g[k].n < 0) return fail(WIPES_EINVAL, "group n < 0");
    if (g[k].activation != WIPES_ACT_NONE && g[k].activation != WIPES_ACT_SIGMOID)
      return fail(WIPES_EINVAL, "group activation");
    if (g[k].n == 0) continue;
    if (!g[k].param || (need_grad && (!g[k].grad || !g[k].m || !g[k].v)))
      return fail(WIPES_EINVAL, "group param/grad/m/v is NULL");
    if (g[k].activation != WIPES_ACT_NONE && !g[k].act)
      return fail(WIPES_EINVAL, "group with an activation needs act");
    if (!(g[k].lr >= 0.f)) return fail(WIPES_EINVAL, "group lr must be >= 0");
  }
  return WIPES_OK;
}

wipes_status wipes_adam_step(const wipes_adam_group* groups, int32_t n_groups, float beta1,
                             float beta2, float eps, int64_t* step, const int32_t* guard,
                             void* scratch, void* stream) {
  wipes_status st = check_groups(groups, n_groups, true);
  if (st != WIPES_OK) return st;
  if (!(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f) || !(eps >= 0.f))
    return fail(WIPES_EINVAL, "need 0 <= beta1, beta2 < 1 and eps >= 0");
  if (!step || !aligned(step, 8) || !scratch || !aligned(scratch, 16))
    return fail(WIPES_EINVAL, "step/scratch NULL or misaligned");
  cudaError_t e = launch_adam(groups, n_groups, beta1, beta2, eps, step, guard, scratch, 0,
                              (cudaStream_t)stream);
  return e == cudaSuccess ? WIPES_OK : cuda_fail(e, "adam launch");
}

wipes_status wipes_activate(const wipes_adam_group* groups, int32_t n_groups, void* stream) {
  wipes_status st = check_groups(groups, n_groups, false);
  if (st != WIPES_OK) return st;
  cudaError_t e = launch_adam(groups, n_groups, 0.f, 0.f, 0.f, nullptr, nullptr, nullptr, 1,
                              (cudaStream_t)stream);
  return e == cudaSuccess ? WIPES_OK : cuda_fail(e, "activate launch");
}

const int32_t* wipes_overflow_flag(const void* ws) {
  return ws ? &((const WsHeader*)ws)->overflow : nullptr;
}

wipes_status wipes_gemm_bf16(const wipes_gemm_args* g, void* stream) {
  if (!g) return fail(WIPES_EINVAL, "args is NULL");
  if (g->M < 0 || g->N < 0 || g->K < 0) return fail(WIPES_EINVAL, "negative size");
  if (g->M == 0 || g->N == 0) return WIPES_OK;
  if (!g->A || !g->B || !g->C) return fail(WIPES_EINVAL, "A, B and C must be non-NULL");
  if (!aligned(g->A, 16) || !aligned(g->B, 16)) return fail(WIPES_EINVAL, "A/B not 16-byte aligned");
  if (g->K % 8 || g->lda % 8 || g->ldb % 8) return fail(WIPES_EINVAL, "K, lda, ldb must be multiples of 8");
  if (g->epilogue < WIPES_GEMM_EPI_STORE_F32 || g->epilogue > WIPES_GEMM_EPI_ATOMIC_F32)
    return fail(WIPES_EINVAL, "epilogue");
  if ((g->epilogue == WIPES_GEMM_EPI_BIAS_F32 || g->epilogue == WIPES_GEMM_EPI_BIAS_RELU_BF16) &&
      !g->bias)
    return fail(WIPES_EINVAL, "bias is NULL");
  if (g->epilogue == WIPES_GEMM_EPI_MASK_BF16 && !g->mask) return fail(WIPES_EINVAL, "mask is NULL");
  if (g->split3 < 0 || (g->split3 > 0 && g->epilogue != WIPES_GEMM_EPI_BIAS_RELU_BF16 &&
                        g->epilogue != WIPES_GEMM_EPI_MASK_BF16))
    return fail(WIPES_EINVAL, "split3 needs a bf16 epilogue");
  if (g->split_k > 1 && g->epilogue != WIPES_GEMM_EPI_ATOMIC_F32)
    return fail(WIPES_EINVAL, "split_k > 1 needs the atomic epilogue");
  cudaError_t e = launch_gemm(*g, (cudaStream_t)stream);
  return e == cudaSuccess ? WIPES_OK : cuda_fail(e, "gemm launch");
}

size_t wipes_mlp_param_count(const wipes_mlp_config* c) {
  if (!c || !mlp_config_valid(*c)) { fail(WIPES_EINVAL, "mlp config"); return 0; }
  return (size_t)mlp_param_count(*c);
}

size_t wipes_mlp_workspace_bytes(const wipes_mlp_config* c, int64_t rows) {
  if (!c || !mlp_config_valid(*c) || rows < 0) { fail(WIPES_EINVAL, "mlp config/rows"); return 0; }
  return mlp_workspace_bytes(*c, rows);
}

static wipes_status check_mlp(const wipes_mlp_config* c, const float* theta, int64_t N, int32_t F,
                              void* ws, size_t ws_bytes) {
  if (!c || !mlp_config_valid(*c)) return fail(WIPES_EINVAL, "mlp config");
  if (N < 0 || F < 1) return fail(WIPES_EINVAL, "need N >= 0 and F >= 1");
  if (!theta) return fail(WIPES_EINVAL, "theta is NULL");
  if (!ws || !aligned(ws, 256)) return fail(WIPES_EINVAL, "ws NULL or not 256-byte aligned");
  if (ws_bytes < mlp_workspace_bytes(*c, N * (int64_t)F))
    return fail(WIPES_EINVAL, "ws_bytes < wipes_mlp_workspace_bytes");
  return WIPES_OK;
}

wipes_status wipes_mlp_forward(const wipes_mlp_config* c, const float* theta, int64_t N, int32_t F,
                               const float* times, const wipes_params* canon,
                               const wipes_params* frame, int32_t sh_coeffs, int32_t train,
                               void* ws, size_t ws_bytes, void* stream) {
  wipes_status st = check_mlp(c, theta, N, F, ws, ws_bytes);
  if (st != WIPES_OK) return st;
  if (!times || !canon || !frame) return fail(WIPES_EINVAL, "times/canon/frame NULL");
  if (!canon->mean || !canon->quat || !canon->scale || !canon->freq || !frame->mean ||
      !frame->quat || !frame->scale || !frame->freq)
    return fail(WIPES_EINVAL, "mean/quat/scale/freq (canon and frame) must be non-NULL");
  if (sh_coeffs < 0 || sh_coeffs > 16) return fail(WIPES_EINVAL, "sh_coeffs");
  cudaError_t e = launch_mlp_forward(*c, theta, N, F, times, *canon, *frame, sh_coeffs, train,
                                     (char*)ws, (cudaStream_t)stream);
  return e == cudaSuccess ? WIPES_OK : cuda_fail(e, "mlp forward");
}

wipes_status wipes_mlp_backward(const wipes_mlp_config* c, const float* theta, int64_t N,
                                int32_t F, const wipes_params* canon, const wipes_grads* gf,
                                float* g_theta, const wipes_grads* gc, void* ws, size_t ws_bytes,
                                void* stream) {
  wipes_status st = check_mlp(c, theta, N, F, ws, ws_bytes);
  if (st != WIPES_OK) return st;
  if (!canon || !canon->scale || !gf || !gf->mean || !gf->quat || !gf->scale || !gf->freq ||
      !g_theta || !gc)
    return fail(WIPES_EINVAL, "canon.scale, g_frame groups, g_theta and g_canon are required");
  cudaError_t e = launch_mlp_backward(*c, theta, N, F, *canon, *gf, g_theta, *gc, (char*)ws,
                                      (cudaStream_t)stream);
  return e == cudaSuccess ? WIPES_OK : cuda_fail(e, "mlp backward");
}

int wipes_num_kernels(void) { return K_NUM; }

const char* wipes_kernel_name(int k) { return (k >= 0 && k < K_NUM) ? kNames[k] : "?"; }

void wipes_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_tmu);
  g_timing = on != 0;
}

wipes_status wipes_timing_collect(double* ms, int64_t* launches, int n) {
  std::lock_guard<std::mutex> lk(g_tmu);
  for (int k = 0; k < n; ++k) {
    if (ms) ms[k] = 0.0;
    if (launches) launches[k] = 0;
  }
  cudaError_t e = cudaSuccess;
  if (!g_log.empty()) e = cudaEventSynchronize(g_log.back().b);
  for (auto& t : g_log) {
    float dt = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&dt, t.a, t.b);
    if (t.kid < n) {
      if (ms) ms[t.kid] += dt;
      if (launches) launches[t.kid] += 1;
    }
    g_pool.push_back(t.a);
    g_pool.push_back(t.b);
  }
  g_log.clear();
  if (e != cudaSuccess) return cuda_fail(e, "timing_collect");
  return WIPES_OK;
}

int64_t wipes_launch_count(void) { return g_launches.load(); }

const char* wipes_status_string(wipes_status s) {
  switch (s) {
    case WIPES_OK: return "WIPES_OK";
    case WIPES_EINVAL: return "WIPES_EINVAL";
    case WIPES_ECAPACITY: return "WIPES_ECAPACITY";
    case WIPES_ECUDA: return "WIPES_ECUDA";
    case WIPES_EUNSUPPORTED: return "WIPES_EUNSUPPORTED";
  }
  return "WIPES_UNKNOWN";
}

const char* wipes_last_error(void) { return g_last_error.c_str(); }

int wipes_abi_version(void) { return WIPES_ABI_VERSION; }

}  // extern "C"
