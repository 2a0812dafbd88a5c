// Onesweep LSD radix sort of (key, uint32 value) pairs, key = uint32 or
// uint64, over selected 8-bit digits ("an
// efficient GPU sorting algorithm"), hand-written for sm_100a (no CUB):
//
//  1. k_sort_hist  : one read of the keys builds the global 256-bin histogram
//                    of EVERY pass at once (shared-memory atomics, then one
//                    global atomic per (block, pass, digit)).
//  2. k_sort_pass  : one launch per digit. Each CTA takes the next tile of
//                    kSortTile keys (tile id from an atomic counter, so tiles
//                    are assigned in launch order), ranks them stably in shared
//                    memory (warp-striped layout, lanes with equal digits found
//                    by 9 ballots per step),
//                    publishes its per-digit counts, resolves its per-digit
//                    global offsets by DECOUPLED LOOK-BACK over the preceding
//                    tiles, stages the pairs in shared memory in sorted order
//                    and writes them out with coalesced runs.
//
// Per pass the keys/values are read once and written once — the HBM floor of
// an LSD pass. Stability: within a tile the rank follows input order
// (warp-major, then step, then lane); across tiles the look-back prefix
// follows tile order.
#include "common.cuh"

namespace wipes {

namespace {

constexpr int kWarps = kSortThreads / 32;
#ifndef WIPES_SORT_LOOKBACK
#define WIPES_SORT_LOOKBACK 4
#endif
constexpr int kLookBack = WIPES_SORT_LOOKBACK;
#ifndef WIPES_SORT_BACKOFF
#define WIPES_SORT_BACKOFF 64  // ns: keeps spinning warps off the issue slots
#endif
constexpr uint32_t kFlagAgg = 1u << 30, kFlagInc = 2u << 30, kValMask = (1u << 30) - 1;

template <typename K>
struct SortArgs {
  const K* kin;
  const uint32_t* vin;
  K* kout;
  uint32_t* vout;
  const WsHeader* hdr;
  int64_t n_fixed;     // >= 0: number of keys; < 0: min(hdr->total, cap)
  int64_t cap;
  uint32_t* ghist;     // [kMaxPasses][256]
  uint32_t* counter;   // [kMaxPasses] tile counters
  uint32_t* status;    // [tiles][256] look-back words of this pass
  int32_t shifts[kMaxPasses];
  int32_t npass, pass, shift;
  uint32_t vdiv, vmask;  // pass p with bit p of vmask: digit of (value / vdiv), not of key
  // reduce-then-scan passes: digit-major tile counts [256][tiles] and their
  // flat exclusive scan (offset of digit d of tile t = loc[i] + blk[i / kScanTile])
  uint32_t* rts_cnt;
  const int64_t* rts_loc;
  const int64_t* rts_blk;
  int64_t tiles;
  // segmented reduce-then-scan (ALPHA presort: one segment per view): keys
  // [s seg_len, (s + 1) seg_len) sort among themselves; tiles never straddle a
  // segment (seg_tiles per segment) and the counts are laid out
  // (segment, digit, tile), so the flat scan keeps the segments in order.
  // seg_len = 0: one segment of n keys.
  int64_t seg_len, seg_tiles;
  VSeg vs;  // variable-length segments (vs.map non-null), else unused
};

// Key range [base, end) of a tile, its segment (variable segments: nseg for a
// tile past the last one; else 0) and the count index of its digit d.
template <typename K, bool VS>
__device__ __forceinline__ int tile_span(const SortArgs<K>& a, int64_t tile, int64_t n,
                                         int64_t& base, int64_t& end) {
  int sg = 0;
  if constexpr (VS) {
    sg = a.vs.map[tile];
    if (sg >= a.vs.nseg) {
      base = end = 0;
      return sg;
    }
    base = a.vs.off[sg] + (tile - a.vs.tiles[sg]) * kSortTile;
    end = base + kSortTile;
    const int64_t se = a.vs.off[sg + 1];
    if (end > se) end = se;
  } else if (a.seg_len > 0) {
    const int64_t g = tile / a.seg_tiles, lt = tile - g * a.seg_tiles;
    base = g * a.seg_len + lt * kSortTile;
    end = base + kSortTile;
    const int64_t se = (g + 1) * a.seg_len;
    if (end > se) end = se;
  } else {
    base = tile * kSortTile;
    end = base + kSortTile;
  }
  if (end > n) end = n;
  return sg;
}
template <typename K, bool VS>
__device__ __forceinline__ int64_t count_index(const SortArgs<K>& a, int64_t tile, int d, int sg) {
  if constexpr (VS) {
    if (sg >= a.vs.nseg) return tile * 256 + d;  // past the segments: zero counts
    const int64_t t0 = a.vs.tiles[sg], nt = a.vs.tiles[sg + 1] - t0;
    return t0 * 256 + (int64_t)d * nt + (tile - t0);
  }
  if (a.seg_len > 0) {
    const int64_t sg = tile / a.seg_tiles, lt = tile - sg * a.seg_tiles;
    return (sg * 256 + d) * a.seg_tiles + lt;
  }
  return (int64_t)d * a.tiles + tile;
}

template <typename K>
__device__ __forceinline__ int64_t n_keys(const SortArgs<K>& a) {
  if (a.n_fixed >= 0) return a.n_fixed;
  const int64_t t = a.hdr->total;
  return t < a.cap ? t : a.cap;
}

#ifndef WIPES_HIST_KEYS
#define WIPES_HIST_KEYS 1024  // keys per histogram block (C2: 1.5 us faster than 4096)
#endif
#ifndef WIPES_HIST_MAXB
#define WIPES_HIST_MAXB 1184  // 148 SMs x 8 blocks
#endif
#ifndef WIPES_HIST_UNROLL
#define WIPES_HIST_UNROLL 4   // independent key loads in flight per thread
#endif

// Shared-memory histogram add of one digit per lane (d = 256: no key). When
// the whole warp holds one digit (the high digits of tile keys, whose runs
// are long), one add of 32 instead of 32 conflicting atomics.
__device__ __forceinline__ void warp_hist_add(uint32_t* h, uint32_t d) {
  const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
  if (__all_sync(0xffffffffu, d == d0)) {
    if ((threadIdx.x & 31) == 0 && d0 < 256u) atomicAdd(&h[d0], 32u);
  } else if (d < 256u) {
    atomicAdd(&h[d], 1u);
  }
}

template <typename K>
__global__ void __launch_bounds__(256) k_sort_hist(SortArgs<K> a) {
  __shared__ uint32_t h[kMaxPasses][256];
  for (int i = threadIdx.x; i < kMaxPasses * 256; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const int64_t n = n_keys(a);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // warp-uniform trip count (the warp's first index decides), so every lane
  // reaches the warp-wide match below
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 - lane < n;
       i0 += WIPES_HIST_UNROLL * stride) {
    // the loads of the group first (independent), then the shared-memory adds
    K k[WIPES_HIST_UNROLL];
    uint32_t vq[WIPES_HIST_UNROLL];
#pragma unroll
    for (int u = 0; u < WIPES_HIST_UNROLL; ++u) {
      const int64_t i = i0 + u * stride;
      k[u] = i < n ? a.kin[i] : (K)0;
      vq[u] = (a.vmask && i < n) ? a.vin[i] / a.vdiv : 0u;
    }
#pragma unroll
    for (int u = 0; u < WIPES_HIST_UNROLL; ++u) {
      const bool valid = i0 + u * stride < n;
#pragma unroll
      for (int p = 0; p < kMaxPasses; ++p)
        if (p < a.npass) {
          const uint32_t bin = (((a.vmask >> p) & 1u) ? (vq[u] >> a.shifts[p])
                                                      : (uint32_t)(k[u] >> a.shifts[p])) & 255u;
          if (valid) atomicAdd(&h[p][bin], 1u);  // (warp_hist_add measured slower here)
        }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < a.npass * 256; i += blockDim.x) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(a.ghist + i, c);
  }
}

#ifndef WIPES_SORT_RANK
#define WIPES_SORT_RANK 1  // lanes with equal digits: 0 = 8 ballots, 1 = shared atomicOr masks
#endif

template <typename K>
struct SortSmem {
  K keys[kSortTile];
  uint32_t vals[kSortTile];
  uint32_t wcnt[kWarps][256];  // per-warp running counts, then warp-exclusive prefixes
  uint32_t thist[256];         // tile digit histogram (published before the ranking)
  uint32_t gofs[256];          // global output offset of the tile's first key per digit
#if WIPES_SORT_RANK == 1
  uint32_t match[2][kWarps][260];  // per-warp lane masks of each digit, 257 used (double-buffered)
#endif
  uint32_t tile;
};

#ifndef WIPES_SORT_MINB
#define WIPES_SORT_MINB 4
#endif

#ifndef WIPES_SORT_LOOKBACK2
#define WIPES_SORT_LOOKBACK2 4  // larger later windows measured slower (C3 scatter 0.88 ms at 4, 0.90 at 8, 0.96 at 16, 1.05 at 32)
#endif
constexpr int kLookBack2 = WIPES_SORT_LOOKBACK2;

// One look-back round of W predecessors (t, t - 1, ...; before tile 0 reads as
// an inclusive 0): adds their values in tile order up to the first inclusive
// word (returns true) or the first unpublished one (advances t and sp past the
// aggregates used, backing off if none was).
// Look-back status words: relaxed GPU-scope accesses (flag and value share one
// word, so no ordering beyond the word itself is needed).
__device__ __forceinline__ uint32_t ld_status(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int W>
__device__ __forceinline__ bool lookback_round(const uint32_t*& sp, int& t,
                                               uint32_t& prefix) {
  uint32_t s[W];
#pragma unroll
  for (int j = 0; j < W; ++j) s[j] = t - j >= 0 ? ld_status(sp - 256 * j) : kFlagInc;
  int used = 0;
  bool stop = false;
#pragma unroll
  for (int j = 0; j < W; ++j) {
    const uint32_t f = s[j] & ~kValMask;
    if (stop || used < j || f == 0u) continue;  // unpublished: re-read from here
    prefix += s[j] & kValMask;
    ++used;
    stop = f == kFlagInc;
  }
  if (stop) return true;
  if (used == 0) __nanosleep(WIPES_SORT_BACKOFF);  // predecessor unpublished: back off
  t -= used;
  sp -= 256 * used;
  return false;
}

// Reduce-then-scan, reduce step: the digit histogram of every tile, written
// digit-major so one flat exclusive scan turns it into each (digit, tile)'s
// global output offset (no look-back). Tiles past the data write zeros.
template <typename K, bool VS>
__global__ void __launch_bounds__(kSortThreads) k_sort_up(SortArgs<K> a) {
  __shared__ uint32_t h[256];
  const int tid = threadIdx.x;
  const int64_t n = n_keys(a);
  h[tid] = 0;  // kSortThreads == 256
  __syncthreads();
  int64_t base, end;
  const int sg = tile_span<K, VS>(a, blockIdx.x, n, base, end);
  const K ksub = VS ? (K)sg * (K)a.vs.T : (K)0;  // view-local tile ids
  const bool vp = (a.vmask >> a.pass) & 1u;
  uint32_t dg[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {  // the loads first (independent)
    const int64_t idx = base + i * kSortThreads + tid;
    dg[i] = 256u;
    if (idx < end)
      dg[i] = (vp ? (a.vin[idx] / a.vdiv) >> a.shift : (uint32_t)((a.kin[idx] - ksub) >> a.shift)) &
              255u;
  }
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) warp_hist_add(h, dg[i]);
  __syncthreads();
  a.rts_cnt[count_index<K, VS>(a, blockIdx.x, tid, sg)] = h[tid];
}

template <typename K, bool RTS, bool VS>
__global__ void __launch_bounds__(kSortThreads, WIPES_SORT_MINB) k_sort_pass(SortArgs<K> a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem<K>& sm = *reinterpret_cast<SortSmem<K>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t n = n_keys(a);
  if (RTS) {
    if (tid == 0) sm.tile = blockIdx.x;  // offsets come from the scan: any tile order
  } else {
    if (tid == 0) sm.tile = atomicAdd(a.counter + a.pass, 1u);
  }
  __syncthreads();
  const uint32_t tile = sm.tile;
  int64_t base, end;  // this tile's keys (onesweep: end = min(base + tile, n))
  const int sg = tile_span<K, VS>(a, tile, n, base, end);
  if (base >= end) return;  // beyond the data: nobody waits on this tile
  const K ksub = VS ? (K)sg * (K)a.vs.T : (K)0;  // view-local tile ids
  const int shift = a.shift;
  const bool vp = (a.vmask >> a.pass) & 1u;
  const uint32_t lt = (1u << lane) - 1u;
  // ---- load (warp-striped) and rank stably within the tile ----------------
  K key[kSortItems];
  uint32_t val[kSortItems];
  uint32_t dig[kSortItems], rank[kSortItems];
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t idx = base + (int64_t)wid * (32 * kSortItems) + i * 32 + lane;
    const bool valid = idx < end;
    key[i] = valid ? a.kin[idx] : (K)0;
    val[i] = valid ? a.vin[idx] : 0u;
  }
  // zero the counters (16-byte stores) while the key loads are in flight
  {
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    uint4* w4 = reinterpret_cast<uint4*>(&sm.wcnt[0][0]);
    for (int i = tid; i < kWarps * 256 / 4; i += kSortThreads) w4[i] = z;
#if WIPES_SORT_RANK == 1
    uint4* m4 = reinterpret_cast<uint4*>(&sm.match[0][0][0]);
    for (int i = tid; i < 2 * kWarps * 260 / 4; i += kSortThreads) m4[i] = z;
#endif
    sm.thist[tid] = 0;  // kSortThreads == 256
  }
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const int64_t idx = base + (int64_t)wid * (32 * kSortItems) + i * 32 + lane;
    const uint32_t src = vp ? (val[i] / a.vdiv) >> shift : (uint32_t)((key[i] - ksub) >> shift);
    dig[i] = idx < end ? (src & 255u) : 256u;
  }
  __syncthreads();
  // tile histogram first, so the aggregate is published before the ranking
  // and the successors' look-back rarely has to wait for it
  uint32_t* st = a.status;
  if (!RTS) {  // (reduce-then-scan has its offsets already)
#pragma unroll
    for (int i = 0; i < kSortItems; ++i)
      if (dig[i] < 256u) atomicAdd(&sm.thist[dig[i]], 1u);
    __syncthreads();
    st_status(st + (int64_t)tile * 256 + tid, kFlagAgg | sm.thist[tid]);
  }
  // only the last tile has invalid slots (digit 256): full tiles match 8 bits
  const bool full_tile = base + kSortTile <= end;
#if WIPES_SORT_RANK == 1
  (void)full_tile;
  // lanes with the same digit: every lane ORs its bit into its digit's mask
  // (warp-private shared words) and, after a warp barrier, reads the mask back.
  // The digit's first lane (the leader) advances the warp's running count after
  // a second barrier, and clears its mask one step later (two buffers: the
  // clear falls between the next step's barriers, after every lane has read the
  // mask and before the buffer's next use).
  uint32_t prev_d = 256u;
  bool prev_lead = false;
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t d = dig[i];
    uint32_t* mrow = sm.match[i & 1][wid];
    atomicOr(&mrow[d], 1u << lane);
    __syncwarp();
    if (prev_lead) sm.match[(i + 1) & 1][wid][prev_d] = 0u;  // step i - 1's mask
    const uint32_t peers = *(volatile uint32_t*)&mrow[d];
    const uint32_t before = d < 256u ? sm.wcnt[wid][d] : 0u;
    rank[i] = (d << 16) | (before + __popc(peers & lt));  // digit | rank (< 2^16)
    const bool lead = (peers & lt) == 0;
    __syncwarp();
    if (lead && d < 256u) sm.wcnt[wid][d] = before + __popc(peers);
    prev_d = d;
    prev_lead = lead;
  }
#else
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t d = dig[i];
#ifdef WIPES_SORT_MATCH
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
#else
    // lanes with the same digit: AND over the digit bits (bit 8 marks an
    // invalid slot) of the matching ballots — cheaper than MATCH.ANY
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? bb : ~bb;
    }
    if (!full_tile) {
      const uint32_t bb = __ballot_sync(0xffffffffu, d >> 8);
      peers &= (d >> 8) ? bb : ~bb;
    }
#endif
    const uint32_t before = d < 256u ? sm.wcnt[wid][d] : 0u;
    rank[i] = (d << 16) | (before + __popc(peers & lt));  // digit | rank (< 2^16)
    __syncwarp();
    if (d < 256u && (peers & lt) == 0) sm.wcnt[wid][d] = before + __popc(peers);
    __syncwarp();
  }
#endif
  __syncthreads();
  // ---- per digit (thread tid = digit): warp prefixes, tile count ---------
  const int d = tid;  // kSortThreads == 256
  uint32_t cnt = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const uint32_t c = sm.wcnt[w][d];
    sm.wcnt[w][d] = cnt;
    cnt += c;
  }
  if constexpr (RTS) {
    // the scanned digit-major counts give the tile's global digit offsets
    const int64_t e = count_index<K, VS>(a, tile, d, sg);
    const uint32_t go = (uint32_t)(a.rts_loc[e] + a.rts_blk[e / kScanTile]);
    uint32_t incl_b = cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t tb = __shfl_up_sync(0xffffffffu, incl_b, off);
      if (lane >= off) incl_b += tb;
    }
    __shared__ uint32_t wb2[kWarps];
    if (lane == 31) wb2[wid] = incl_b;
    __syncthreads();
    uint32_t ob = 0;
    for (int w = 0; w < wid; ++w) ob += wb2[w];
    const uint32_t bx = ob + incl_b - cnt;
    // fold the tile-local digit base into the warp prefixes (staging: one load)
    // and keep gofs - bexcl (write-out: one load; uint32 wrap-around exact)
#pragma unroll
    for (int w = 0; w < kWarps; ++w) sm.wcnt[w][d] += bx;
    sm.gofs[d] = go - bx;
    __syncthreads();
  } else {
  // look back for the exclusive prefix (the aggregate was published above)
  uint32_t prefix = 0;
#ifdef WIPES_SORT_LB1
  for (int64_t t = (int64_t)tile - 1; t >= 0;) {
    const uint32_t s = ld_status(st + t * 256 + d);
    const uint32_t f = s & ~kValMask;
    if (f == 0u) continue;  // not yet published: spin
    prefix += s & kValMask;
    if (f == kFlagInc) break;
    --t;
  }
#else
  // look back over the predecessors: kLookBack status words per first round,
  // kLookBack2 per later round (the first wave of CTAs starts together, so its
  // tiles walk back across hundreds of aggregates; later tiles mostly find an
  // inclusive prefix one or two tiles back). The words of a round are loaded
  // together (independent loads), then consumed in tile order. 32-bit tile
  // index and one running pointer.
  {
    int t = (int)tile - 1;
    const uint32_t* sp = st + (int64_t)t * 256 + d;
    if (t >= 0 && !lookback_round<kLookBack>(sp, t, prefix))
      while (!lookback_round<kLookBack2>(sp, t, prefix)) {
      }
  }
#endif
  // flag and value share one 32-bit word: no fence needed between publishes
  st_status(st + (int64_t)tile * 256 + d, kFlagInc | (prefix + cnt));
  // global digit base = exclusive scan of the pass histogram (block scan)
  const uint32_t gh = a.ghist[a.pass * 256 + d];
  uint32_t incl_g = gh, incl_b = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t tg = __shfl_up_sync(0xffffffffu, incl_g, off);
    const uint32_t tb = __shfl_up_sync(0xffffffffu, incl_b, off);
    if (lane >= off) { incl_g += tg; incl_b += tb; }
  }
  __shared__ uint32_t wg[kWarps], wb[kWarps];
  if (lane == 31) { wg[wid] = incl_g; wb[wid] = incl_b; }
  __syncthreads();
  uint32_t og = 0, ob = 0;
  for (int w = 0; w < wid; ++w) { og += wg[w]; ob += wb[w]; }
  const uint32_t excl_g = og + incl_g - gh, excl_b = ob + incl_b - cnt;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) sm.wcnt[w][d] += excl_b;
  sm.gofs[d] = excl_g + prefix - excl_b;
  __syncthreads();
  }
  // ---- stage in tile-sorted order, then coalesced write-out -----------------
  // 32-bit keys: (key, value) staged as one 8-byte word (one scattered store
  // and one load per pair instead of two each)
  constexpr bool kPair = sizeof(K) == 4;
  uint2* const kv = reinterpret_cast<uint2*>(sm.keys);  // spans keys + vals (16 KB)
#pragma unroll
  for (int i = 0; i < kSortItems; ++i) {
    const uint32_t dd = rank[i] >> 16;
    if (dd < 256u) {
      const uint32_t loc = sm.wcnt[wid][dd] + (rank[i] & 0xffffu);
      WCHECK(loc < (uint32_t)kSortTile);
      if constexpr (kPair) {
        kv[loc] = make_uint2((uint32_t)key[i], val[i]);
      } else {
        sm.keys[loc] = key[i];
        sm.vals[loc] = val[i];
      }
    }
  }
  __syncthreads();
  const int64_t rem = end - base;
  const int tn = rem < kSortTile ? (int)rem : kSortTile;
  for (int j = tid; j < tn; j += kSortThreads) {
    K k;
    uint32_t v;
    if constexpr (kPair) {
      const uint2 p = kv[j];
      k = (K)p.x;
      v = p.y;
    } else {
      k = sm.keys[j];
      v = sm.vals[j];
    }
    const uint32_t dd = (vp ? (v / a.vdiv) >> shift : (uint32_t)((k - ksub) >> shift)) & 255u;
    const int64_t pos = (int64_t)(uint32_t)(sm.gofs[dd] + (uint32_t)j);
    WCHECK(pos >= 0 && pos < n);
    a.kout[pos] = k;
    a.vout[pos] = v;
  }
}

}  // namespace

template <typename K>
cudaError_t launch_sort(const Layout& L, char* ws, K* kA, uint32_t* vA, K* kB, uint32_t* vB,
                        const int* shifts, int npass, int64_t n_fixed, int64_t cap,
                        cudaStream_t s, uint32_t vdiv, uint32_t vmask, bool hist_ready,
                        int64_t seg_len, const VSeg* vseg) {
  if (npass == 0 || cap == 0) return cudaSuccess;
  WIPES_SET_SMEM_ONCE((k_sort_pass<K, false, false>), (int)sizeof(SortSmem<K>));
  WIPES_SET_SMEM_ONCE((k_sort_pass<K, true, false>), (int)sizeof(SortSmem<K>));
  WIPES_SET_SMEM_ONCE((k_sort_pass<K, true, true>), (int)sizeof(SortSmem<K>));
  SortArgs<K> a;
  a.hdr = (const WsHeader*)(ws + L.hdr);
  a.n_fixed = n_fixed;
  a.cap = cap;
  a.ghist = (uint32_t*)(ws + L.sort_hist);
  a.counter = a.ghist + kMaxPasses * 256;
  a.status = (uint32_t*)(ws + L.sort_status);
  a.npass = npass;
  a.vdiv = vdiv ? vdiv : 1u;
  a.vmask = vmask;
  for (int p = 0; p < kMaxPasses; ++p) a.shifts[p] = p < npass ? shifts[p] : 0;
  // segmented (n_fixed keys in segments of seg_len): tiles never straddle one
  a.seg_len = seg_len > 0 ? seg_len : 0;
  a.seg_tiles = seg_len > 0 ? (seg_len + kSortTile - 1) / kSortTile : 0;
  a.vs = vseg ? *vseg : VSeg{nullptr, nullptr, nullptr, 0, 0u, 0};
  const int64_t tiles = vseg ? vseg->tile_bound
                             : seg_len > 0 ? (n_fixed / seg_len) * a.seg_tiles
                                           : (cap + kSortTile - 1) / kSortTile;
  // large sorts: reduce-then-scan passes (no look-back chain across the
  // hundreds of tiles in flight); small ones: onesweep (one launch per pass).
  // Segmented sorts are reduce-then-scan only (Layout::pre_seg).
  const bool rts = vseg || seg_len > 0 || tiles >= sort_rts_tiles();
  if (seg_len > 0 && (n_fixed % seg_len != 0 || tiles > L.sort_tiles)) return cudaErrorInvalidValue;
  if (vseg && tiles > L.sort_tiles) return cudaErrorInvalidValue;
  a.tiles = tiles;
  a.rts_cnt = a.status;
  a.rts_loc = (const int64_t*)(ws + L.sort_loc);
  a.rts_blk = (const int64_t*)(ws + L.sort_blk);
  int32_t* arrive = &((WsHeader*)(ws + L.hdr))->arrive[3];
  cudaError_t e = cudaSuccess;
  a.kin = kA; a.vin = vA; a.pass = 0; a.shift = 0;
  if (!hist_ready && !rts) {  // else the producer zeroed ghist + counters and built the histogram
    e = cudaMemsetAsync(a.ghist, 0, sizeof(uint32_t) * (kMaxPasses * 256 + kMaxPasses), s);
    if (e != cudaSuccess) return e;
    const int64_t hist_blocks = (cap + WIPES_HIST_KEYS - 1) / WIPES_HIST_KEYS;
    launch_begin(K_RADIX_HIST, s);
    k_sort_hist<K><<<(unsigned)(hist_blocks < WIPES_HIST_MAXB ? (hist_blocks > 0 ? hist_blocks : 1)
                                                                : WIPES_HIST_MAXB),
                     256, 0, s>>>(a);
    launch_end(K_RADIX_HIST, s);
  }
  for (int p = 0; p < npass; ++p) {
    const bool from_a = (p & 1) == 0;
    a.kin = from_a ? kA : kB; a.vin = from_a ? vA : vB;
    a.kout = from_a ? kB : kA; a.vout = from_a ? vB : vA;
    a.pass = p;
    a.shift = shifts[p];
    if (rts) {
      launch_begin(K_RADIX_HIST, s);
      if (vseg)
        k_sort_up<K, true><<<(unsigned)tiles, kSortThreads, 0, s>>>(a);
      else
        k_sort_up<K, false><<<(unsigned)tiles, kSortThreads, 0, s>>>(a);
      e = launch_flat_scan((const int32_t*)a.rts_cnt, 256 * tiles, (int64_t*)a.rts_loc,
                           (int64_t*)a.rts_blk, arrive, s);
      launch_end(K_RADIX_HIST, s);
      if (e != cudaSuccess) return e;
      launch_begin(K_RADIX_SCATTER, s);
      if (vseg)
        k_sort_pass<K, true, true><<<(unsigned)tiles, kSortThreads, sizeof(SortSmem<K>), s>>>(a);
      else
        k_sort_pass<K, true, false><<<(unsigned)tiles, kSortThreads, sizeof(SortSmem<K>), s>>>(a);
      launch_end(K_RADIX_SCATTER, s);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      continue;
    }
    e = cudaMemsetAsync(a.status, 0, sizeof(uint32_t) * 256 * (size_t)tiles, s);
    if (e != cudaSuccess) return e;
    launch_begin(K_RADIX_SCATTER, s);
    k_sort_pass<K, false, false><<<(unsigned)tiles, kSortThreads, sizeof(SortSmem<K>), s>>>(a);
    launch_end(K_RADIX_SCATTER, s);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

template cudaError_t launch_sort<uint32_t>(const Layout&, char*, uint32_t*, uint32_t*,
                                           uint32_t*, uint32_t*, const int*, int, int64_t,
                                           int64_t, cudaStream_t, uint32_t, uint32_t, bool,
                                           int64_t, const VSeg*);
template cudaError_t launch_sort<uint64_t>(const Layout&, char*, uint64_t*, uint32_t*,
                                           uint64_t*, uint32_t*, const int*, int, int64_t,
                                           int64_t, cudaStream_t, uint32_t, uint32_t, bool,
                                           int64_t, const VSeg*);

size_t sort_smem_bytes64() { return sizeof(SortSmem<uint64_t>); }

}  // namespace wipes
