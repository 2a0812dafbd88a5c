// Tile binning: exclusive scan of per-(view, primitive)
// tile counts, duplication under the 64-bit key ((view*T + tile) << 32 |
// depth bits), a stable LSD radix sort over the significant key bits only,
// and per-tile CSR ranges. PAPER.md:64 ("an efficient GPU sorting algorithm").
//
// The radix sort itself is the onesweep implementation in sort.cu.
#include "common.cuh"

namespace wipes {

namespace {

__device__ __forceinline__ int64_t clamp_n(const WsHeader* h, int64_t cap) {
  int64_t t = h->total;
  return t < cap ? t : cap;
}

// ---------------------------------------------------------------- scan ----
// Exclusive scan of nblk block sums in place by one block of NT threads.
// Optionally publishes the grand total and the capacity-overflow flag into
// the workspace header and resets its per-frame scheduling state. The sums
// may have been written by other blocks of the same grid: they are read
// through L2 (ld.global.cg).
template <int NT, typename T>
__device__ __forceinline__ void scan_sums_block(T* blk, int64_t nblk, WsHeader* hdr, int64_t cap) {
  static_assert(sizeof(T) == 8, "64-bit block sums");
  constexpr int NW = NT / 32;
  __shared__ T wt[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t per = (nblk + NT - 1) / NT;
  const int64_t b0 = (int64_t)tid * per;
  T s = 0;
  for (int64_t k = 0; k < per; ++k)
    if (b0 + k < nblk) s += (T)__ldcg((const long long*)blk + b0 + k);
  T inc = s;
  for (int off = 1; off < 32; off <<= 1) {
    T t = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += t;
  }
  if (lane == 31) wt[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T t = lane < NW ? wt[lane] : (T)0;
    T ti = t;
    for (int off = 1; off < 32; off <<= 1) {
      T u = __shfl_up_sync(0xffffffffu, ti, off);
      if (lane >= off) ti += u;
    }
    if (lane < NW) wt[lane] = ti - t;
    if (lane == 31 && hdr) {
      hdr->total = (int64_t)ti;
      hdr->overflow = (int64_t)ti > cap ? 1 : 0;
    }
  }
  if (hdr && wid == 1) {  // reset the per-frame scheduling state
    hdr->bcount[lane] = 0;
    hdr->bfill[lane] = 0;
    if (lane < kQueues) { hdr->work[lane] = 0; hdr->done[lane] = 0; }
    if (lane >= 1 && lane < 4) hdr->arrive[lane] = 0;
  }
  __syncthreads();
  T run = wt[wid] + inc - s;
  for (int64_t k = 0; k < per; ++k)
    if (b0 + k < nblk) {
      T v = (T)__ldcg((const long long*)blk + b0 + k);
      blk[b0 + k] = run;
      run += v;
    }
}

// Single-launch exclusive scan: every block scans its kScanTile items and
// publishes its sum; the last block to arrive (counter `arrive`) scans the
// block sums. Consumers add loc[i] + blk[i / kScanTile].
template <typename TIn, typename TOut>
__global__ void __launch_bounds__(kScanBlock) k_scan(const TIn* in, int64_t n, TOut* loc,
                                                    TOut* blk_sum, int32_t* arrive,
                                                    WsHeader* hdr, int64_t cap) {
  __shared__ TOut warp_tot[kScanBlock / 32];
  __shared__ int is_last;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)tid * kScanItems;
  static_assert(sizeof(TIn) == 4 && sizeof(TOut) == 8 && kScanItems == 8, "vector path");
  TOut v[kScanItems];
  TOut s = 0;
  const bool whole = base + kScanItems <= n;  // a thread's 8 items: two 16-byte loads
  if (whole) {
    const int4 a0 = reinterpret_cast<const int4*>(in + base)[0];
    const int4 a1 = reinterpret_cast<const int4*>(in + base)[1];
    v[0] = (TOut)a0.x; v[1] = (TOut)a0.y; v[2] = (TOut)a0.z; v[3] = (TOut)a0.w;
    v[4] = (TOut)a1.x; v[5] = (TOut)a1.y; v[6] = (TOut)a1.z; v[7] = (TOut)a1.w;
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) v[k] = base + k < n ? (TOut)in[base + k] : (TOut)0;
  }
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) s += v[k];
  // inclusive warp scan of thread sums
  TOut inc = s;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    TOut t = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += t;
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    TOut t = lane < kScanBlock / 32 ? warp_tot[lane] : (TOut)0;
    TOut ti = t;
#pragma unroll
    for (int off = 1; off < kScanBlock / 32; off <<= 1) {
      TOut u = __shfl_up_sync(0xffffffffu, ti, off);
      if (lane >= off) ti += u;
    }
    if (lane < kScanBlock / 32) warp_tot[lane] = ti - t;  // exclusive
    if (lane == kScanBlock / 32 - 1) {
      blk_sum[blockIdx.x] = ti;
      __threadfence();  // the sum is visible before this block counts as arrived
    }
  }
  __syncthreads();
  if (tid == 0) is_last = atomicAdd(arrive, 1) == (int)gridDim.x - 1;
  TOut r[kScanItems];
  r[0] = warp_tot[wid] + inc - s;
#pragma unroll
  for (int k = 1; k < kScanItems; ++k) r[k] = r[k - 1] + v[k - 1];
  if (whole) {  // four 16-byte stores
    longlong2* o = reinterpret_cast<longlong2*>(loc + base);
#pragma unroll
    for (int k = 0; k < kScanItems / 2; ++k)
      o[k] = make_longlong2((long long)r[2 * k], (long long)r[2 * k + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
      if (base + k < n) loc[base + k] = r[k];
  }
  __syncthreads();
  if (is_last) {
    __threadfence();
    scan_sums_block<kScanBlock>(blk_sum, gridDim.x, hdr, cap);
    if (tid == 0) *arrive = 0;  // self-resetting for the next scan of this workspace
  }
}

// ----------------------------------------------------------- duplicate ----
// Each (view, primitive) record with n tiles writes n pairs (key = view*T +
// tile, value = primitive) at its offset, row-major over its rect. SUM walks
// records in index order; ALPHA walks them in the depth-presorted order
// `order` with offsets scanned in that order, so each tile's list comes out in
// (depth, index) order and only the tile bits need sorting.
struct DupArgs {
  const int4* rect;
  const int32_t* count;
  const int32_t* count_sorted;  // ALPHA: count[order[j]] (k_gather_counts)
  const uint32_t* order;  // ALPHA: presorted (view, primitive) ids; SUM: nullptr
  const int64_t* loc;
  const int64_t* blk;
  int64_t BN, N, T, cap;
  int32_t GX, row_mod, row_rem;
  uint32_t* keys;
  uint32_t* vals;
  uint32_t* prevals;  // deterministic mode: vals[j] = j, prevals[j] = primitive
  uint32_t* ghist;    // non-null: also build the radix histogram of the npass
  int32_t npass;      //   8-bit tile-key digits (sort.cu's k_sort_hist, fused)
};

// Adds a block's shared histogram into the global one (after the whole block
// has counted: every warp, including those past the records, reaches here).
__device__ __forceinline__ void flush_hist(const DupArgs& a, uint32_t (*hist)[256]) {
  __syncthreads();
  for (int i = threadIdx.x; i < a.npass * 256; i += blockDim.x) {
    const uint32_t c = (&hist[0][0])[i];
    if (c) atomicAdd(a.ghist + i, c);
  }
}

// Warp-cooperative emission: the 32 records of a warp own one contiguous
// output range (their offsets are consecutive in the scan), so the warp
// writes it lane-strided — every store instruction covers 32 consecutive
// pairs — finding each pair's record by a binary search over the lanes'
// start offsets and its tile from the record's rect.
template <bool HIST>
__global__ void __launch_bounds__(256) k_duplicate(DupArgs a) {
  __shared__ uint32_t hist[HIST ? kMaxPasses : 1][256];
  if (HIST) {
    for (int i = threadIdx.x; i < kMaxPasses * 256; i += blockDim.x) (&hist[0][0])[i] = 0;
    __syncthreads();
  }
  const int64_t j0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  constexpr unsigned kFullMask = 0xffffffffu;
  int32_t n = 0;
  int64_t start = INT64_MAX;  // beyond BN: never owns a pair
  int4 r = make_int4(0, 0, 0, 0);
  uint32_t vt = 0, ival = 0;
  int ty0 = 0, wdt = 1;
  if (j0 < a.BN) {
    const int64_t o = a.order ? (int64_t)a.order[j0] : j0;
    WCHECK(o >= 0 && o < a.BN);
    n = a.order ? a.count_sorted[j0] : a.count[o];  // ALPHA: the gathered counts (coalesced)
    start = a.loc[j0] + a.blk[j0 / kScanTile];
    const int64_t v = o / a.N;
    ival = (uint32_t)(o - v * a.N);
    vt = (uint32_t)(v * a.T);
    if (n > 0) {
      r = a.rect[o];
      ty0 = a.row_mod > 1 ? band_first_row(r.y, a.row_mod, a.row_rem) : r.y;
      wdt = r.z - r.x;
    }
  }
  // (break: the whole warp is beyond the records; it still reaches the flush)
  do {
    if (j0 - lane >= a.BN) break;
    // the warp's output range [S, E) (lane 0 is always a valid record)
    const int64_t S = __shfl_sync(kFullMask, start, 0);
    int64_t E = j0 < a.BN ? start + n : 0;
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      const int64_t t = __shfl_xor_sync(kFullMask, E, off);
      E = t > E ? t : E;
    }
    const int dty = a.row_mod > 1 ? a.row_mod : 1;
    for (int64_t j = S + lane; j - lane < E; j += 32) {
      const bool live = j < E;
      // owner = the last lane with start <= j (starts are non-decreasing; a
      // zero-count lane shares its start with the next lane, which owns it)
      int owner = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const int64_t sv = __shfl_sync(kFullMask, start, owner + step);
        if (sv <= j) owner += step;
      }
      const int64_t so = __shfl_sync(kFullMask, start, owner);
      const int ox = __shfl_sync(kFullMask, r.x, owner);
      const int ow = __shfl_sync(kFullMask, wdt, owner);
      const int oty = __shfl_sync(kFullMask, ty0, owner);
      const uint32_t ovt = __shfl_sync(kFullMask, vt, owner);
      const uint32_t oi = __shfl_sync(kFullMask, ival, owner);
      const bool emit = live && j < a.cap;
      uint32_t key = 0;
      if (emit) {
        const int t = (int)(j - so);
        const int row = t / ow, col = t - row * ow;
        WCHECK(t >= 0 && col >= 0 && col < ow && ox + col < a.GX);
        key = ovt + (uint32_t)(oty + row * dty) * (uint32_t)a.GX + (uint32_t)(ox + col);
        a.keys[j] = key;
        if (a.prevals) {
          a.vals[j] = (uint32_t)j;
          a.prevals[j] = oi;
        } else {
          a.vals[j] = oi;
        }
      }
      if (HIST) {
        // low digit: mostly distinct across the lanes (consecutive tiles);
        // higher digits: few distinct values, so one add per distinct digit
        if (emit) atomicAdd(&hist[0][key & 255u], 1u);
        for (int p = 1; p < a.npass; ++p) {
          const uint32_t d = emit ? (key >> (8 * p)) & 255u : 256u;
          const uint32_t peers = __match_any_sync(kFullMask, d);
          if (emit && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&hist[p][d], (uint32_t)__popc(peers));
        }
      }
    }
  } while (0);
  if (HIST) flush_hist(a, hist);
}

// ALPHA depth presort inputs: key = orderable depth bits, value = o = view*N +
// primitive (the view digits of the last passes are taken from value / N).
__global__ void __launch_bounds__(256) k_presort_keys(const uint32_t* dkey, int64_t BN,
                                                      uint32_t* pk, uint32_t* pv) {
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= BN) return;
  pk[o] = dkey[o];
  pv[o] = (uint32_t)o;
}

__global__ void __launch_bounds__(256) k_gather_counts(const uint32_t* order, const int32_t* count,
                                                       int64_t BN, int32_t* out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < BN) out[j] = count[order[j]];
}

// --------------------------------------------------------- tile ranges ----
// 64-bit (tile << 32 | depth bits) keys of the sorted pairs, for parity copies.
__global__ void __launch_bounds__(256) k_keys64(const uint32_t* keys, const uint32_t* vals,
                                                const uint32_t* prevals, const uint32_t* dkey,
                                                const WsHeader* hdr, int64_t cap, int64_t N,
                                                int64_t T, int32_t alpha, uint64_t* out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= clamp_n(hdr, cap)) return;
  const uint32_t k = keys[j];
  const uint32_t i = prevals ? prevals[vals[j]] : vals[j];  // primitive of entry j
  const uint64_t lo = alpha ? (uint64_t)dkey[(int64_t)(k / T) * N + i] : 0ull;
  out[j] = ((uint64_t)k << 32) | lo;
}

// Longest-first tile order for the persistent render kernels: tiles are
// bucketed by floor(log2(list length)) + 1 (0 for empty tiles) and laid out in
// descending bucket order (order within a bucket is arbitrary: it affects only
// the processing order, never a result).
__device__ __forceinline__ int tile_bucket(const int32_t* toff, int64_t u) {
  const int len = toff[u + 1] - toff[u];
  return len > 0 ? 32 - __clz(len) : 0;
}

__global__ void __launch_bounds__(256) k_tile_order_hist(const int32_t* toff, int64_t BT,
                                                         WsHeader* hdr) {
  __shared__ int32_t h[kBuckets];
  if (threadIdx.x < kBuckets) h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u < BT) atomicAdd(&h[tile_bucket(toff, u)], 1);
  __syncthreads();
  if (threadIdx.x < kBuckets && h[threadIdx.x]) atomicAdd(&hdr->bcount[threadIdx.x], h[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_tile_order_place(const int32_t* toff, int64_t BT,
                                                          WsHeader* hdr, int32_t* order) {
  __shared__ int32_t base[kBuckets], h[kBuckets];
  const int tid = threadIdx.x;
  if (tid < kBuckets) h[tid] = 0;
  __syncthreads();
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + tid;
  int b = 0, r = 0;
  if (u < BT) {
    b = tile_bucket(toff, u);
    r = atomicAdd(&h[b], 1);
  }
  __syncthreads();
  if (tid < kBuckets) {
    int off = 0;  // start of bucket tid in descending-bucket order
    for (int k = kBuckets - 1; k > tid; --k) off += hdr->bcount[k];
    base[tid] = h[tid] ? off + atomicAdd(&hdr->bfill[tid], h[tid]) : 0;
  }
  __syncthreads();
  if (u < BT) order[base[b] + r] = (int32_t)u;
}

#ifndef WIPES_DUP_HIST_MAXB
#define WIPES_DUP_HIST_MAXB 2048  // duplicate grids up to this size build the sort histogram
#endif
#ifndef WIPES_ORDER_FUSE_MAX
#define WIPES_ORDER_FUSE_MAX 8192  // up to this many tiles, the last ranges block orders them
#endif

// Per-tile CSR ranges from the sorted keys: entry i writes toff[u] = i for
// every tile u in (key[i-1], key[i]] (entry n closes the list with BT). Each
// thread takes four consecutive entries (one 16-byte key load). With `order`
// set (small BT), the last block to finish also builds the longest-first tile
// order in shared memory, saving the two tile-order launches.
__global__ void __launch_bounds__(256) k_tile_ranges(const uint32_t* keys, WsHeader* hdr,
                                                     int64_t cap, int64_t BT, int32_t* toff,
                                                     int32_t* order) {
  __shared__ int is_last;
  __shared__ int32_t h[kBuckets], base[kBuckets];
  const int tid = threadIdx.x;
  const int64_t i0 = 4 * ((int64_t)blockIdx.x * blockDim.x + tid);
  const int64_t n = clamp_n(hdr, cap);
  if (i0 <= n) {
    uint32_t k[4];
    if (i0 + 4 <= n) {
      const uint4 v = *reinterpret_cast<const uint4*>(keys + i0);
      k[0] = v.x; k[1] = v.y; k[2] = v.z; k[3] = v.w;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) k[e] = i0 + e < n ? keys[i0 + e] : 0u;
    }
    int64_t tp = i0 == 0 ? -1 : (int64_t)keys[i0 - 1];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t i = i0 + e;
      if (i > n) break;
      int64_t tc = i == n ? BT : (int64_t)k[e];
      if (tc > BT) tc = BT;
      WCHECK(tp >= -1 && tc <= BT && tp <= tc);
      for (int64_t u = tp + 1; u <= tc; ++u) toff[u] = (int32_t)i;
      tp = tc;
    }
  }
  if (!order) return;
  __threadfence();  // this thread's ranges are visible before the block arrives
  __syncthreads();
  if (tid == 0) is_last = atomicAdd(&hdr->arrive[2], 1) == (int)gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  if (tid < kBuckets) h[tid] = 0;
  // the whole CSR array into shared memory first: every load in flight at once
  // (the two passes below then read shared memory instead of two dependent L2
  // round trips per iteration)
  __shared__ int32_t s_toff[WIPES_ORDER_FUSE_MAX + 1];
#pragma unroll 8
  for (int u = tid; u <= (int)BT; u += 256) s_toff[u] = __ldcg(toff + u);
  __syncthreads();
  for (int u = tid; u < (int)BT; u += 256) {
    const int len = s_toff[u + 1] - s_toff[u];
    atomicAdd(&h[len > 0 ? 32 - __clz(len) : 0], 1);
  }
  __syncthreads();
  if (tid < kBuckets) {
    int off = 0;  // start of bucket tid in descending-bucket order
    for (int k = kBuckets - 1; k > tid; --k) off += h[k];
    base[tid] = off;
  }
  __syncthreads();
  for (int u = tid; u < (int)BT; u += 256) {
    const int len = s_toff[u + 1] - s_toff[u];
    order[atomicAdd(&base[len > 0 ? 32 - __clz(len) : 0], 1)] = (int32_t)u;
  }
  if (tid == 0) hdr->arrive[2] = 0;  // self-resetting (bin_sort may run again)
}

// View segments of the ALPHA tile sort (Layout::tile_seg): dups are emitted in
// presorted (view, depth) order, view v's records at presorted positions
// [v N, (v + 1) N), so view v's dups start at the scanned offset of position
// v N (clipped to the stored count). One block: off[0..B], and tiles[0..B] =
// the exclusive prefix of each view's 2048-key tiles.
__global__ void __launch_bounds__(1024) k_vseg_tables(const int64_t* loc, const int64_t* blk,
                                                      const WsHeader* hdr, int64_t cap, int64_t N,
                                                      int B, int64_t* off, int64_t* tiles) {
  __shared__ int64_t wsum[32];
  __shared__ int64_t carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t n = clamp_n(hdr, cap);
  for (int v = tid; v <= B; v += blockDim.x) {
    int64_t o = n;
    if (v < B) {
      const int64_t p = (int64_t)v * N;
      o = loc[p] + blk[p / kScanTile];
      if (o > n) o = n;
    }
    off[v] = o;
  }
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int v0 = 0; v0 <= B; v0 += blockDim.x) {
    const int v = v0 + tid;
    const int64_t c = v < B ? (off[v + 1] - off[v] + kSortTile - 1) / kSortTile : 0;
    int64_t inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t t = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += t;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      int64_t t = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
      int64_t ti = t;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int64_t u = __shfl_up_sync(0xffffffffu, ti, d);
        if (lane >= d) ti += u;
      }
      wsum[lane] = ti - t;
    }
    __syncthreads();
    if (v <= B) tiles[v] = carry + wsum[wid] + inc - c;
    __syncthreads();
    if (tid == (int)blockDim.x - 1) carry += wsum[wid] + inc;
    __syncthreads();
  }
}

// Segment of every tile of the view-segmented sort (B past the last one).
__global__ void k_vseg_map(const int64_t* tiles, int B, int64_t bound, int32_t* map) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= bound) return;
  int lo = 0, hi = B;  // tiles[lo] <= t < tiles[hi] (tiles[B] = total)
  if (t >= tiles[B]) {
    map[t] = B;
    return;
  }
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (tiles[mid] <= t) lo = mid; else hi = mid;
  }
  map[t] = lo;
}

__global__ void k_offsets(const int64_t* loc, const int64_t* blk, int64_t BN, int64_t* out) {
  int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (o < BN) out[o] = loc[o] + blk[o / kScanTile];
}

}  // namespace

cudaError_t launch_keys64(const Layout& L, const char* ws, int final_in_b, uint64_t* out,
                          cudaStream_t s) {
  if (L.cap == 0) return cudaSuccess;
  k_keys64<<<(unsigned)((L.cap + 255) / 256), 256, 0, s>>>(
      (const uint32_t*)(ws + (final_in_b ? L.keysB : L.keysA)),
      (const uint32_t*)(ws + (final_in_b ? L.valsB : L.valsA)),
      L.det ? (const uint32_t*)(ws + L.prevals) : nullptr, (const uint32_t*)(ws + L.dkey),
      (const WsHeader*)(ws + L.hdr), L.cap, L.N, L.T, L.alpha, out);
  return cudaGetLastError();
}

cudaError_t launch_offsets_copy(const Layout& L, const char* ws, int64_t* out, cudaStream_t s) {
  if (L.BN == 0) return cudaSuccess;
  k_offsets<<<(unsigned)((L.BN + 255) / 256), 256, 0, s>>>(
      (const int64_t*)(ws + L.loc_off), (const int64_t*)(ws + L.blk_sum), L.BN, out);
  return cudaGetLastError();
}

cudaError_t launch_scan_counts(const Layout& L, char* ws, cudaStream_t s) {
  WsHeader* hdr = (WsHeader*)(ws + L.hdr);
  if (L.BN == 0) {  // no preprocess launch zeroed the arrival counter
    cudaError_t e = cudaMemsetAsync(hdr->arrive, 0, sizeof(hdr->arrive), s);
    if (e != cudaSuccess) return e;
  }
  launch_begin(K_SCAN_BLOCKS, s);
  k_scan<int32_t, int64_t><<<(unsigned)L.nblk_scan, kScanBlock, 0, s>>>(
      (const int32_t*)(ws + L.count), L.BN, (int64_t*)(ws + L.loc_off),
      (int64_t*)(ws + L.blk_sum), &hdr->arrive[0], hdr, L.cap);
  launch_end(K_SCAN_BLOCKS, s);
  return cudaGetLastError();
}

cudaError_t launch_flat_scan(const int32_t* in, int64_t n, int64_t* loc, int64_t* blk,
                             int32_t* arrive, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const unsigned g = (unsigned)((n + kScanTile - 1) / kScanTile);
  k_scan<int32_t, int64_t><<<g, kScanBlock, 0, s>>>(in, n, loc, blk, arrive, nullptr, 0);
  return cudaGetLastError();
}

cudaError_t launch_bin_sort(const wipes_config& c, const Layout& L, char* ws, cudaStream_t s,
                            int* final_in_b) {
  WsHeader* hdr = (WsHeader*)(ws + L.hdr);
  uint32_t* kA = (uint32_t*)(ws + L.keysA);
  uint32_t* kB = (uint32_t*)(ws + L.keysB);
  uint32_t* vA = (uint32_t*)(ws + L.valsA);
  uint32_t* vB = (uint32_t*)(ws + L.valsB);
  *final_in_b = final_buffer_is_b(L);
  if (L.cap > 0 && L.BN > 0) {
    const unsigned gBN = (unsigned)((L.BN + 255) / 256);
    const uint32_t* order = nullptr;
    const int64_t* loc = (const int64_t*)(ws + L.loc_off);
    const int64_t* blk = (const int64_t*)(ws + L.blk_sum);
    cudaError_t e;
    if (L.alpha) {
      // depth presort of the (view, primitive) records, then offsets in that order
      uint32_t* pkA = (uint32_t*)(ws + L.pkA);
      uint32_t* pkB = (uint32_t*)(ws + L.pkB);
      uint32_t* pvA = (uint32_t*)(ws + L.pvA);
      uint32_t* pvB = (uint32_t*)(ws + L.pvB);
      launch_begin(K_DUPLICATE, s);
      k_presort_keys<<<gBN, 256, 0, s>>>((const uint32_t*)(ws + L.dkey), L.BN, pkA, pvA);
      launch_end(K_DUPLICATE, s);
      // 4 depth-byte passes on the key, then (unsegmented) the view bytes of
      // value / N; segmented by view, the depth passes alone
      int shifts[kMaxPasses];
      uint32_t vmask = 0;
      for (int p = 0; p < L.pre_passes; ++p) {
        shifts[p] = p < 4 ? 8 * p : 8 * (p - 4);
        if (p >= 4) vmask |= 1u << p;
      }
      e = launch_sort<uint32_t>(L, ws, pkA, pvA, pkB, pvB, shifts, L.pre_passes, L.BN, L.BN, s,
                                (uint32_t)L.N, vmask, false, L.pre_seg ? L.N : 0);
      if (e != cudaSuccess) return e;
      order = (L.pre_passes & 1) ? pvB : pvA;
      launch_begin(K_DUPLICATE, s);
      k_gather_counts<<<gBN, 256, 0, s>>>(order, (const int32_t*)(ws + L.count), L.BN,
                                          (int32_t*)(ws + L.cnt2));
      launch_end(K_DUPLICATE, s);
      launch_begin(K_SCAN_BLOCKS, s);
      k_scan<int32_t, int64_t><<<(unsigned)L.nblk_scan, kScanBlock, 0, s>>>(
          (const int32_t*)(ws + L.cnt2), L.BN, (int64_t*)(ws + L.loc2), (int64_t*)(ws + L.blk2),
          &hdr->arrive[1], nullptr, 0);
      launch_end(K_SCAN_BLOCKS, s);
      loc = (const int64_t*)(ws + L.loc2);
      blk = (const int64_t*)(ws + L.blk2);
    }
    DupArgs d;
    d.rect = (const int4*)(ws + L.rect);
    d.count = (const int32_t*)(ws + L.count);
    d.count_sorted = (const int32_t*)(ws + L.cnt2);
    d.order = order;
    d.loc = loc;
    d.blk = blk;
    d.BN = L.BN; d.N = L.N; d.T = L.T; d.cap = L.cap;
    d.GX = L.GX;
    d.row_mod = c.row_mod; d.row_rem = c.row_rem;
    d.keys = kA; d.vals = vA;
    d.prevals = L.det ? (uint32_t*)(ws + L.prevals) : nullptr;
    // small grids build the tile-key histogram while emitting (one launch
    // less); large ones leave it to k_sort_hist (fewer global atomics)
    const bool fuse_hist = L.passes > 0 && gBN <= WIPES_DUP_HIST_MAXB;
    d.ghist = (uint32_t*)(ws + L.sort_hist);
    d.npass = L.passes;
    launch_begin(K_DUPLICATE, s);
    if (fuse_hist) {
      e = cudaMemsetAsync(d.ghist, 0, sizeof(uint32_t) * (kMaxPasses * 256 + kMaxPasses), s);
      if (e != cudaSuccess) return e;
      k_duplicate<true><<<gBN, 256, 0, s>>>(d);
    } else {
      k_duplicate<false><<<gBN, 256, 0, s>>>(d);
    }
    launch_end(K_DUPLICATE, s);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // stable LSD passes over the (view*T + tile) bits only; view-segmented
    // (ALPHA, Layout::tile_seg): over the view-local tile bits
    int shifts[kMaxPasses];
    for (int p = 0; p < L.passes; ++p) shifts[p] = 8 * p;
    if (L.tile_seg) {
      VSeg vs;
      vs.off = (const int64_t*)(ws + L.vseg_off);
      vs.tiles = (const int64_t*)(ws + L.vseg_tiles);
      vs.map = (const int32_t*)(ws + L.vseg_map);
      vs.nseg = L.B;
      vs.T = (uint32_t)L.T;
      vs.tile_bound = L.tile_bound;
      launch_begin(K_RADIX_HIST, s);
      k_vseg_tables<<<1, 1024, 0, s>>>(loc, blk, hdr, L.cap, L.N, L.B, (int64_t*)(ws + L.vseg_off),
                                      (int64_t*)(ws + L.vseg_tiles));
      k_vseg_map<<<(unsigned)((L.tile_bound + 255) / 256), 256, 0, s>>>(
          (const int64_t*)(ws + L.vseg_tiles), L.B, L.tile_bound, (int32_t*)(ws + L.vseg_map));
      launch_end(K_RADIX_HIST, s);
      e = launch_sort<uint32_t>(L, ws, kA, vA, kB, vB, shifts, L.passes, -1, L.cap, s, 1, 0,
                                fuse_hist, 0, &vs);
    } else {
      e = launch_sort<uint32_t>(L, ws, kA, vA, kB, vB, shifts, L.passes, -1, L.cap, s, 1, 0,
                                fuse_hist);
    }
    if (e != cudaSuccess) return e;
  }
  const uint32_t* kf = *final_in_b ? kB : kA;
  const bool fuse_order = L.BT > 0 && L.BT <= WIPES_ORDER_FUSE_MAX;
  launch_begin(K_TILE_RANGES, s);
  k_tile_ranges<<<(unsigned)((L.cap + 1 + 1023) / 1024), 256, 0, s>>>(
      kf, hdr, L.cap, L.BT, (int32_t*)(ws + L.toff), fuse_order ? (int32_t*)(ws + L.order) : nullptr);
  launch_end(K_TILE_RANGES, s);
  if (L.BT > 0 && !fuse_order) {
    const unsigned g = (unsigned)((L.BT + 255) / 256);
    // bucket counters must start at zero for every ordering (bin_sort may run
    // more than once per preprocess)
    cudaMemsetAsync(hdr->bcount, 0, sizeof(hdr->bcount) + sizeof(hdr->bfill), s);
    launch_begin(K_TILE_ORDER, s);
    k_tile_order_hist<<<g, 256, 0, s>>>((const int32_t*)(ws + L.toff), L.BT, hdr);
    launch_end(K_TILE_ORDER, s);
    launch_begin(K_TILE_ORDER, s);
    k_tile_order_place<<<g, 256, 0, s>>>((const int32_t*)(ws + L.toff), L.BT, hdr,
                                         (int32_t*)(ws + L.order));
    launch_end(K_TILE_ORDER, s);
  }
  return cudaGetLastError();
}

// Sorted values as primitive ids (deterministic mode stores dup indices).
__global__ void k_vals_copy(const uint32_t* vals, const uint32_t* prevals, const WsHeader* hdr,
                            int64_t cap, uint32_t* out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cap) return;
  const int64_t n = hdr->total < cap ? hdr->total : cap;  // entries past the total are unset
  out[j] = (prevals && j < n) ? prevals[vals[j]] : vals[j];
}

cudaError_t launch_vals_copy(const Layout& L, const char* ws, int final_in_b, uint32_t* out,
                             cudaStream_t s) {
  if (L.cap == 0) return cudaSuccess;
  const uint32_t* v = (const uint32_t*)(ws + (final_in_b ? L.valsB : L.valsA));
  k_vals_copy<<<(unsigned)((L.cap + 255) / 256), 256, 0, s>>>(
      v, L.det ? (const uint32_t*)(ws + L.prevals) : nullptr, (const WsHeader*)(ws + L.hdr),
      L.cap, out);
  return cudaGetLastError();
}

// Deterministic backward, second half: the record at emission position j0
// sums the moment slots of its dups [start, start + count) over the warp
// footprints in a fixed order (dups past the capacity were never rendered).
__global__ void __launch_bounds__(128) k_det_gather(const int32_t* count, const uint32_t* order,
                                                    const int64_t* loc, const int64_t* blk,
                                                    int64_t BN, int64_t cap, int fps, int slotw,
                                                    const float* slots, const uint8_t* mask,
                                                    float* mom, float* mom_beta) {
  const int64_t j0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j0 >= BN) return;
  const int64_t o = order ? (int64_t)order[j0] : j0;
  const int32_t n = count[o];
  const int64_t start = loc[j0] + blk[j0 / kScanTile];
  float acc[kMoments + 1];
  for (int k = 0; k <= kMoments; ++k) acc[k] = 0.f;
  const int64_t end = start + n < cap ? start + n : cap;
  if (slotw == kMoments) {  // 48-byte slots: 3 float4 loads each (16-byte aligned)
    const float4* sl = reinterpret_cast<const float4*>(slots) + start * fps * 3;
    for (int64_t q = 0; q < (end - start) * fps; ++q, sl += 3) {
      const int64_t si = start * fps + q;
      if (!mask[si]) continue;  // slot not written this frame
      const float4 a = __ldg(sl), b = __ldg(sl + 1), c = __ldg(sl + 2);
      acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
      acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
      acc[8] += c.x; acc[9] += c.y; acc[10] += c.z; acc[11] += c.w;
    }
  } else {
    for (int64_t j = start; j < end; ++j)
      for (int f = 0; f < fps; ++f) {
        const int64_t si = j * fps + f;
        if (!mask[si]) continue;  // slot not written this frame
        const float* sl = slots + si * slotw;
        for (int k = 0; k < slotw; ++k) acc[k] += sl[k];
      }
  }
  for (int k = 0; k < kMoments; ++k) mom[o * kMoments + k] = acc[k];
  if (mom_beta) mom_beta[o] = acc[kMoments];
}

cudaError_t launch_det_gather(const Layout& L, char* ws, cudaStream_t s) {
  if (L.BN == 0) return cudaSuccess;
  const bool pre = L.alpha;  // ALPHA emits in the depth-presorted order
  const uint32_t* order = pre ? ((L.pre_passes & 1) ? (const uint32_t*)(ws + L.pvB)
                                                    : (const uint32_t*)(ws + L.pvA))
                              : nullptr;
  const int64_t* loc = (const int64_t*)(ws + (pre ? L.loc2 : L.loc_off));
  const int64_t* blk = (const int64_t*)(ws + (pre ? L.blk2 : L.blk_sum));
  launch_begin(K_DET_GATHER, s);
  k_det_gather<<<(unsigned)((L.BN + 127) / 128), 128, 0, s>>>(
      (const int32_t*)(ws + L.count), order, loc, blk, L.BN, L.cap, L.fps, L.slotw,
      (const float*)(ws + L.slots), (const uint8_t*)(ws + L.slotmask), (float*)(ws + L.rgrad),
      L.exact ? (float*)(ws + L.rbeta) : nullptr);
  launch_end(K_DET_GATHER, s);
  return cudaGetLastError();
}

}  // namespace wipes
