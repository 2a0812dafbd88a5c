// Shared definitions of the WIPES CUDA library (sm_100a): workspace layout,
// render-record layout, kernel ids, launch helpers. Product code only — no
// oracle code or header is included anywhere under csrc/.
#pragma once
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cassert>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/wipes.h"

// Debug builds (-DWIPES_CHECKS, see tools/sanitize_run.py) assert every index
// the kernels derive from data before using it.
#ifdef WIPES_CHECKS
#define WCHECK(c) assert(c)
#else
#define WCHECK(c) ((void)0)
#endif

// Raise a kernel's dynamic shared-memory limit once per (call site, device):
// the attribute is per device, so a process that launches on several GPUs sets
// it on each; concurrent first calls only repeat an idempotent set.
#define WIPES_SET_SMEM_ONCE(kernel, bytes)                                           \
  do {                                                                               \
    static std::atomic<unsigned long long> wipes_smem_mask_{0};                      \
    int wipes_dev_ = 0;                                                              \
    cudaGetDevice(&wipes_dev_);                                                      \
    const unsigned long long wipes_bit_ = 1ull << (wipes_dev_ & 63);                 \
    if (!(wipes_smem_mask_.load(std::memory_order_acquire) & wipes_bit_)) {          \
      cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (bytes)); \
      wipes_smem_mask_.fetch_or(wipes_bit_, std::memory_order_release);              \
    }                                                                                \
  } while (0)

namespace wipes {

constexpr int kRecGrads = 13;                  // record-gradient slots (FP64, in registers)
constexpr int kMoments = WIPES_GRAD_MOMENTS;   // 12 per-record gradient moments (HBM)
constexpr int kScanBlock = 256;                // threads per scan block
constexpr int kScanItems = 8;                  // items per thread
constexpr int kScanTile = kScanBlock * kScanItems;
constexpr int kRadixBits = 8;
#ifndef WIPES_SORT_RTS_TILES
#define WIPES_SORT_RTS_TILES 1024  // sorts of at least this many 2048-key tiles: reduce-then-scan
#endif
// The threshold, overridable at run time (environment WIPES_SORT_RTS_TILES) so
// the tests can run either sort mode at any size.
inline int64_t sort_rts_tiles() {
  const char* e = getenv("WIPES_SORT_RTS_TILES");
  return (e && *e) ? atoll(e) : (int64_t)WIPES_SORT_RTS_TILES;
}
constexpr int kSortThreads = 256;              // onesweep CTA (one digit per thread)
#ifndef WIPES_SORT_ITEMS
#define WIPES_SORT_ITEMS 8
#endif
constexpr int kSortItems = WIPES_SORT_ITEMS;   // keys per thread per tile
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr int kMaxPasses = 8;
constexpr int32_t kWsMagic = 0x57495053;       // "WIPS"

// Record-gradient slot order (matches the oracle's documented layout, written
// independently): mu'x, mu'y, a, b, c, f'x, f'y, phi, beta, cr, cg, cb, alpha.
enum { RG_MUX = 0, RG_MUY, RG_A, RG_B, RG_C, RG_FX, RG_FY, RG_PHI, RG_BETA, RG_CR, RG_CG,
       RG_CB, RG_ALPHA };

// 64-byte render record (4 x float4), one per (view, primitive):
//  r0 = {ax, ay, mu'x - ax, mu'y - ay}  (ax, ay) = integer anchor floor(mu') as float
//  r1 = {A, B, C, log2(alpha)}          A,B,C = -1/2 log2(e) (a, 2b, c), conic (a,b;b,c)
//  r2 = {f'x, f'y, phi, beta/2}
//  r3 = {c_r, c_g, c_b, half2(rx, ry)}  (rx, ry) = opacity-extent half widths (fp16,
//                                       rounded up), only for conservative sub-tile culling
// The candidate test needs r0, r1 only (two broadcast LDS.128).
constexpr int kBuckets = 32;  // tile-cost buckets (log2 of the list length)
constexpr int kQueues = 4;    // work queues: render fwd, render bwd, stats, spare

struct WsHeader {
  int64_t total;       // number of (view, primitive, tile) intersections
  int32_t overflow;    // 1 if total > capacity
  int32_t magic;
  int64_t N, cap, bytes;
  int32_t B, pad;
  // persistent-kernel work queues (self-resetting: the last CTA zeroes them)
  int32_t work[kQueues], done[kQueues];
  // longest-first tile order: per-bucket counts and fill pointers (zeroed by
  // the count scan of every preprocess)
  int32_t bcount[kBuckets], bfill[kBuckets];
  // last-block arrival counters of the fused binning kernels (count scan,
  // ALPHA order scan, tile ranges); zeroed by preprocess, self-resetting
  int32_t arrive[4];
};
static_assert(sizeof(WsHeader) <= 512, "header must fit its slot");

struct Layout {
  int64_t N = 0, BN = 0, cap = 0, BT = 0, T = 0;
  int32_t B = 0, GX = 0, GY = 0;
  int32_t hi_bits = 0, passes = 0, pre_passes = 0;  // dup-sort / depth-presort passes
  int32_t pre_seg = 0;  // depth presort segmented by view (reduce-then-scan, no view pass)
  int32_t tile_seg = 0;  // ALPHA tile sort segmented by view (per-view tile ids: fewer passes)
  int64_t tile_bound = 0;  // tiles of a view-segmented tile sort (upper bound)
  int32_t alpha = 0;
  int32_t exact = 0;       // 3D exact z-integration: extra beta moment per record
  int32_t det = 0;         // deterministic backward: per-(dup, footprint) moment slots
  int32_t fps = 1;         // warp footprints per tile (render work items per tile)
  int32_t slotw = 0;       // floats per slot (12 moments [+ beta])
  int64_t nblk_scan = 0;   // blocks of the count scan
  int64_t sort_tiles = 0;  // onesweep tiles of kSortTile keys
  size_t hdr = 0, rect = 0, count = 0, flag = 0, dkey = 0, rec = 0, loc_off = 0,
         blk_sum = 0, keysA = 0, keysB = 0, valsA = 0, valsB = 0, pkA = 0, pkB = 0, pvA = 0,
         pvB = 0, cnt2 = 0, loc2 = 0, blk2 = 0, sort_hist = 0, sort_status = 0, sort_loc = 0,
         sort_blk = 0, vseg_off = 0, vseg_tiles = 0, vseg_map = 0, toff = 0,
         order = 0, rgrad = 0, rbeta = 0, rdc = 0, prevals = 0, slots = 0, slotmask = 0, total = 0;
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Image-space sharding: first tile row >= y0 with ty % mod == rem, and the
// number of such rows in [y0, y1).
__host__ __device__ inline int band_first_row(int y0, int mod, int rem) {
  return y0 + (((rem - y0) % mod) + mod) % mod;
}
__host__ __device__ inline int rows_in_band(int y0, int y1, int mod, int rem) {
  const int f = band_first_row(y0, mod, rem);
  return f < y1 ? (y1 - 1 - f) / mod + 1 : 0;
}

inline Layout make_layout(const wipes_config& c, int64_t N, int32_t B, int64_t cap) {
  Layout L;
  L.N = N; L.B = B; L.BN = N * (int64_t)B; L.cap = cap < 0 ? 0 : cap;
  L.GX = (c.width + c.tile - 1) / c.tile;
  L.GY = (c.height + c.tile - 1) / c.tile;
  L.T = (int64_t)L.GX * L.GY;
  L.BT = L.T * B;
  int hb = 0;
  while (((int64_t)1 << hb) < L.BT) ++hb;
  L.hi_bits = hb;
  // dups are keyed by the 32-bit (view*T + tile) id alone: SUM lists are in
  // index order by emission; ALPHA emits in (view, depth, index) order after a
  // depth presort of the (view, primitive) records (4 depth-byte passes + the
  // view bytes), so only the tile bits are sorted per dup.
  L.alpha = c.blend == WIPES_BLEND_ALPHA;
  L.passes = (hb + kRadixBits - 1) / kRadixBits;
  int vb = 0;
  while (((int64_t)1 << vb) < B) ++vb;
  // large presorts run segmented by view (each view's records sorted among
  // themselves, tiles inside one view): the 4 depth-byte passes keep the views
  // in order, so no view pass; small ones sort (view, depth) as one key
  const int64_t seg_tiles = (N + kSortTile - 1) / kSortTile;
  L.pre_seg = L.alpha && (int64_t)B * seg_tiles >= sort_rts_tiles();
  L.pre_passes = L.alpha ? (L.pre_seg ? 4 : 4 + (vb + kRadixBits - 1) / kRadixBits) : 0;
  const int64_t sort_n = L.cap > L.BN ? L.cap : L.BN;
  L.sort_tiles = (sort_n + kSortTile - 1) / kSortTile;
  if (L.pre_seg && (int64_t)B * seg_tiles > L.sort_tiles) L.sort_tiles = (int64_t)B * seg_tiles;
  // ALPHA dups are emitted view-major (presorted order), so sorting each view's
  // dups by the view-local tile id (key - view*T) keeps the views in order: when
  // that id needs fewer radix passes than (view*T + tile), the tile sort runs
  // segmented by view (reduce-then-scan; C4: 13 instead of 20 bits, 2 passes)
  {
    int tb = 0;
    while (((int64_t)1 << tb) < L.T) ++tb;
    const int seg_passes = (tb + kRadixBits - 1) / kRadixBits;
    L.tile_bound = (L.cap + kSortTile - 1) / kSortTile + B;
    L.tile_seg = L.alpha && B > 1 && seg_passes < L.passes && L.tile_bound >= sort_rts_tiles();
    if (L.tile_seg) {
      L.passes = seg_passes;
      if (L.tile_bound > L.sort_tiles) L.sort_tiles = L.tile_bound;
    }
  }
  L.nblk_scan = (L.BN + kScanTile - 1) / kScanTile;
  if (L.nblk_scan < 1) L.nblk_scan = 1;
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
  L.hdr = take(512);
  L.rect = take(sizeof(int4) * L.BN);
  L.count = take(sizeof(int32_t) * L.BN);
  L.flag = take(sizeof(uint8_t) * L.BN);
  L.dkey = take(sizeof(uint32_t) * L.BN);
  L.rec = take(64 * L.BN);
  L.loc_off = take(sizeof(int64_t) * L.BN);
  L.blk_sum = take(sizeof(int64_t) * (L.nblk_scan + 1));
  L.keysA = take(sizeof(uint32_t) * L.cap);
  L.keysB = take(sizeof(uint32_t) * L.cap);
  L.valsA = take(sizeof(uint32_t) * L.cap);
  L.valsB = take(sizeof(uint32_t) * L.cap);
  const int64_t pn = L.alpha ? L.BN : 0;
  L.pkA = take(sizeof(uint32_t) * pn);
  L.pkB = take(sizeof(uint32_t) * pn);
  L.pvA = take(sizeof(uint32_t) * pn);
  L.pvB = take(sizeof(uint32_t) * pn);
  L.cnt2 = take(sizeof(int32_t) * pn);
  L.loc2 = take(sizeof(int64_t) * pn);
  L.blk2 = take(sizeof(int64_t) * (L.alpha ? L.nblk_scan + 1 : 0));
  L.sort_hist = take(sizeof(uint32_t) * (kMaxPasses * 256 + kMaxPasses));
  L.sort_status = take(sizeof(uint32_t) * 256 * (L.sort_tiles > 0 ? L.sort_tiles : 1));
  // reduce-then-scan passes (large sorts): the digit-major tile counts reuse
  // sort_status; their flat exclusive scan goes to sort_loc / sort_blk
  {
    const int64_t ent = 256 * (L.sort_tiles > 0 ? L.sort_tiles : 1);
    L.sort_loc = take(sizeof(int64_t) * ent);
    L.sort_blk = take(sizeof(int64_t) * ((ent + kScanTile - 1) / kScanTile + 1));
  }
  L.vseg_off = take(sizeof(int64_t) * (L.tile_seg ? B + 1 : 0));
  L.vseg_tiles = take(sizeof(int64_t) * (L.tile_seg ? B + 1 : 0));
  L.vseg_map = take(sizeof(int32_t) * (L.tile_seg ? L.tile_bound : 0));
  L.toff = take(sizeof(int32_t) * (L.BT + 1));
  L.order = take(sizeof(int32_t) * (L.BT + 1));
  L.rgrad = take(sizeof(float) * kMoments * L.BN);
  L.exact = c.prim == WIPES_PRIM_3D && c.proj == WIPES_PROJ_EXACT;
  L.rbeta = take(sizeof(float) * (L.exact ? L.BN : 0));
  // SH colour: the records' colour gradients, compacted for the SH backward
  const bool sh = c.prim == WIPES_PRIM_3D && c.color_mode == WIPES_COLOR_SH;
  L.rdc = take(sizeof(float) * 3 * (sh ? L.BN : 0));
  // Deterministic backward (cfg.deterministic): the sorted values are dup
  // indices j (prevals[j] = primitive), the render backward writes each
  // warp's per-record moments to slot (j, footprint) and a gather sums a
  // record's slots in a fixed order (no float atomics).
  L.det = c.deterministic != 0;
  L.fps = (c.tile / 8) * (c.tile >= 16 ? c.tile / 16 : 1);
  L.slotw = kMoments + (L.exact ? 1 : 0);
  L.prevals = take(sizeof(uint32_t) * (L.det ? L.cap : 0));
  L.slots = take(sizeof(float) * (L.det ? (size_t)L.cap * L.fps * L.slotw : 0));
  // one byte per slot: written this frame (only the mask is cleared per frame,
  // and the gather reads only marked slots; plain byte stores, no atomics)
  L.slotmask = take(L.det ? (size_t)L.cap * L.fps : 0);
  L.total = o;
  return L;
}

// Kernel ids for the timing instrumentation (wipes_kernel_name).
enum KernelId {
  K_PRE2D = 0, K_PRE3D, K_SCAN_BLOCKS, K_SCAN_SUMS, K_DUPLICATE, K_RADIX_HIST,
  K_RADIX_SCAN_BLOCKS, K_RADIX_SCAN_SUMS, K_RADIX_SCATTER, K_TILE_RANGES, K_RENDER_FWD,
  K_RENDER_BWD, K_PRE2D_BWD, K_PRE3D_BWD, K_MEMSET, K_TILE_ORDER, K_LOSS, K_ADAM, K_SH_BWD, K_GEMM, K_MLP_MISC, K_DET_GATHER, K_NUM
};

// Camera block passed BY VALUE as a kernel parameter (no H2D copy; graph
// capturable). 18 floats per camera: R[9], t[3], fx, fy, cx, cy, near, far.
struct CamBlock {
  float v[WIPES_MAX_CAMERAS_PER_LAUNCH][18];
  int32_t nv;    // cameras in this block
  int32_t v0;    // first view index of this block
};

// ---- host-side launch bookkeeping (defined in abi.cu) ----------------------
void launch_begin(int kid, cudaStream_t s);
void launch_end(int kid, cudaStream_t s);

// ---- launchers (defined in the .cu files) ----------------------------------
size_t train_scratch_bytes();
cudaError_t launch_gemm(const wipes_gemm_args& g, cudaStream_t s);
cudaError_t launch_det_gather(const Layout& L, char* ws, cudaStream_t s);
cudaError_t launch_vals_copy(const Layout& L, const char* ws, int final_in_b, uint32_t* out,
                             cudaStream_t s);
// Description of one fused deformation-MLP forward (mlp_fused.cu).
struct MlpFusedDesc {
  int32_t W, D, skip, Lx, Lt, E8, catw, train, shc, F;
  int64_t N, M;
  const float* times;  // (host) [F]
  const float* theta;
  int64_t thb[32], thbh;
  wipes_params canon, frame;
  float* out;
  const __nv_bfloat16* wbf[32];
  int32_t Kp[32];
  const __nv_bfloat16* whbf;
  __nv_bfloat16* h[32];
  __nv_bfloat16* cat;
};
bool launch_mlp_fused_fwd(const MlpFusedDesc& d, cudaStream_t s, cudaError_t* err);
// One hidden layer's backward in one pass (mlp_fused.cu): dz_(l-1) = (dz W) * (act > 0)
// and the partial sums of dW = dz^T act and db_(l-1) = colsum(dz_(l-1)) per CTA group.
struct MlpBwdDesc {
  int32_t W;                   // width (the fused path takes W == 256)
  int64_t M;                   // rows
  const __nv_bfloat16* dz;     // [M, W] dL/dz_l
  const __nv_bfloat16* act;    // [M, W] (pitch act_ld) input of layer l = h_(l-1), also the ReLU mask
  const __nv_bfloat16* wl;     // [W, W] (pitch w_ld) bf16 weights of layer l (out x in)
  int64_t act_ld, w_ld;
  __nv_bfloat16* dzo;          // [M, W] dL/dz_(l-1)
  float* wpart;                // [groups, W, W] partial dW (rows: out, cols: in)
  float* bpart;                // [groups * 4, W] partial colsums of dz_(l-1)
  int32_t max_groups;
};
constexpr int kMlpBwdMaxGroups = 128;
// One hidden layer's forward (mlp_fused.cu): out = relu(x W^T + b) in bf16, x [M, 256]
// (pitch x_ld), W [256, 256] bf16 (out x in), b fp32 [256], out pitch out_ld.
struct MlpFwdLayerDesc {
  int32_t W;
  int64_t M, x_ld, out_ld;
  const __nv_bfloat16* x;
  const __nv_bfloat16* w;
  const float* bias;
  __nv_bfloat16* out;
};
// returns false when outside the envelope (W != 256 or unaligned operands)
bool launch_mlp_fwd_layer(const MlpFwdLayerDesc& d, cudaStream_t s, cudaError_t* err);
// Head backward into the last hidden layer (mlp_fused.cu): dz = (dout Wh) * (h > 0),
// dout [M, 16] bf16, Wh [16, 256] bf16, h [M, 256] (pitch h_ld); per-group partial
// column sums of dz in bpart [groups * 2, 256]. Returns the number of groups, 0 when
// outside the envelope.
struct MlpHeadBwdDesc {
  int64_t M, h_ld;
  const __nv_bfloat16* dout;
  const __nv_bfloat16* wh;
  const __nv_bfloat16* h;
  __nv_bfloat16* dz;
  float* bpart;
  int32_t W, max_groups;
};
int launch_mlp_head_bwd(const MlpHeadBwdDesc& d, cudaStream_t s, cudaError_t* err);
// returns the number of groups (partials) launched, or 0 when outside the envelope
int launch_mlp_bwd_layer(const MlpBwdDesc& d, cudaStream_t s, cudaError_t* err);
bool mlp_config_valid(const wipes_mlp_config& c);
int64_t mlp_param_count(const wipes_mlp_config& c);
size_t mlp_workspace_bytes(const wipes_mlp_config& c, int64_t rows);
cudaError_t launch_mlp_forward(const wipes_mlp_config& c, const float* theta, int64_t N,
                               int32_t F, const float* times, const wipes_params& canon,
                               const wipes_params& frame, int32_t sh_coeffs, int32_t train,
                               char* ws, cudaStream_t s);
cudaError_t launch_mlp_backward(const wipes_mlp_config& c, const float* theta, int64_t N,
                                int32_t F, const wipes_params& canon, const wipes_grads& gfr,
                                float* g_theta, const wipes_grads& gcan, char* ws,
                                cudaStream_t s);
cudaError_t launch_loss_l2(const float* img, const float* tgt, int64_t n, float* grad,
                           double* loss, void* scratch, cudaStream_t s);
cudaError_t launch_adam(const wipes_adam_group* groups, int ng, float b1, float b2, float eps,
                        int64_t* step, const int32_t* guard, void* scratch, int activate_only,
                        cudaStream_t s);
cudaError_t launch_preprocess2d(const wipes_config& c, const wipes_params& p, const Layout& L,
                                char* ws, uint8_t* cull_flags, cudaStream_t s);
cudaError_t launch_preprocess3d(const wipes_config& c, const wipes_params& p, const Layout& L,
                                const wipes_camera* cams, char* ws, uint8_t* cull_flags,
                                cudaStream_t s);
cudaError_t launch_scan_counts(const Layout& L, char* ws, cudaStream_t s);
// Flat exclusive scan of n int32 values: out[i] = loc[i] + blk[i / kScanTile]
// (one launch; `arrive` a zeroed, self-resetting counter in the header).
cudaError_t launch_flat_scan(const int32_t* in, int64_t n, int64_t* loc, int64_t* blk,
                             int32_t* arrive, cudaStream_t s);
// Variable-length sort segments (the view-segmented ALPHA tile sort): segment
// v holds keys [off[v], off[v+1]) and tiles [tiles[v], tiles[v+1]); map[t] is
// tile t's segment (nseg past the last); digits come from key - v * T.
struct VSeg {
  const int64_t* off;
  const int64_t* tiles;
  const int32_t* map;
  int32_t nseg;
  uint32_t T;
  int64_t tile_bound;
};
template <typename K>
cudaError_t launch_sort(const Layout& L, char* ws, K* kA, uint32_t* vA, K* kB, uint32_t* vB,
                        const int* shifts, int npass, int64_t n_fixed, int64_t cap,
                        cudaStream_t s, uint32_t vdiv = 1, uint32_t vmask = 0,
                        bool hist_ready = false, int64_t seg_len = 0,
                        const VSeg* vseg = nullptr);
cudaError_t launch_keys64(const Layout& L, const char* ws, int final_in_b, uint64_t* out,
                          cudaStream_t s);
cudaError_t launch_offsets_copy(const Layout& L, const char* ws, int64_t* out, cudaStream_t s);
cudaError_t launch_bin_sort(const wipes_config& c, const Layout& L, char* ws, cudaStream_t s,
                            int* final_in_b);
cudaError_t launch_render_fwd(const wipes_config& c, const Layout& L, char* ws, int final_in_b,
                              float* image, float* T_final, int32_t* n_contrib,
                              cudaStream_t s, unsigned long long* stats = nullptr);
cudaError_t launch_render_bwd(const wipes_config& c, const Layout& L, char* ws, int final_in_b,
                              const float* dLdC, const float* T_final,
                              const int32_t* n_contrib, cudaStream_t s);
// Parameter rows [row0, row1) (row1 < 0: all): primitives (2D, view_stride 0)
// or (view, primitive) rows (per-frame parameter sets).
cudaError_t launch_preprocess2d_bwd(const wipes_config& c, const wipes_params& p,
                                    const Layout& L, char* ws, const wipes_grads& g,
                                    cudaStream_t s, int64_t row0 = 0, int64_t row1 = -1);
cudaError_t launch_preprocess3d_bwd(const wipes_config& c, const wipes_params& p,
                                    const Layout& L, const wipes_camera* cams, char* ws,
                                    const wipes_grads& g, cudaStream_t s, int64_t row0 = 0,
                                    int64_t row1 = -1);

inline int final_buffer_is_b(const Layout& L) { return L.passes & 1; }



}  // namespace wipes
