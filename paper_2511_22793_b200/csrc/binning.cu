// K3: per-tile depth sort.  Replaces the np.lexsort depth order
// (rasterizer.py:82-87) restricted to each of rasterizer._tile_lists
// (rasterizer.py:115-145).
//
// This is the second half of an MSD radix sort on the composite key
// (tile, depth, index):
//   digit 1 (tile) -- counting sort, done by K2 (preprocess.cu): every
//     preprocess CTA stages its pairs as one contiguous segment per touched
//     tile (the azimuth-seam duplicate included: a tile covered by both
//     column segments gets two entries, rasterizer.py:139-141);
//   digits 2.. (depth, index) -- one CTA per tile gathers the tile's
//     segments into shared memory and sorts them by the packed key
//     (coarse_depth32 << 32 | index).  coarse_depth32 is the monotone
//     truncation (bits(depth) - bits(0.05)) >> 24; runs that tie on it are
//     re-ordered by the full f64 bit pattern, so the final order is exactly
//     np.lexsort((idx, depth)) restricted to the tile.
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"

namespace gs {

long long* dbg_rows(int which);

struct SortArgs {
  uint64_t* pairs;
  int* tile_start;
  const uint64_t* key;
  int* counters;
  const int* tile_count;
  int* ready;  // [ntiles] queue of sorted tiles, tile + 1 (the frame's tile_cursor, zeroed by K2)
  const int2* seg;
  const uint64_t* stage;
  int64_t seg_stride;
  uint64_t* sort_tmp;  // [pair_capacity] scratch for lists beyond shared memory
  int* inv;          // deterministic frames: [n][ntiles] list positions
  const int4* rect;  // tile rectangles (K2)
  int ntx;
  int ntiles;
  long long* dbg;  // experiments: per-CTA phase clocks (GSPARC_SORT_DBG)
  int long_bits;   // bucket bits of the long-list path
};

// Ascending-only bitonic network on n elements (virtual +inf padding up to
// the next power of two never moves, so no padding is stored).
template <bool SHARED>
__device__ void bitonic_sort(uint64_t* a, int n) {
  int np2 = 1, lg = 0;
  while (np2 < n) {
    np2 <<= 1;
    ++lg;
  }
  for (int lk = 1; lk <= lg; ++lk) {
    const int k = 1 << lk;
    // first step of the merge: compare i with its mirror in the k-block
    for (int p = threadIdx.x; p < np2 / 2; p += blockDim.x) {
      const int blk = p >> (lk - 1), off = p & ((k >> 1) - 1);
      int i = blk * k + off;
      int j = blk * k + (k - 1 - off);
      if (j < n) {
        uint64_t x = a[i], y = a[j];
        if (y < x) {
          a[i] = y;
          a[j] = x;
        }
      }
    }
    __syncthreads();
    for (int ls = lk - 2; ls >= 0; --ls) {
      const int s = 1 << ls;
      for (int p = threadIdx.x; p < np2 / 2; p += blockDim.x) {
        const int blk = p >> ls, off = p & (s - 1);
        int i = (blk << (ls + 1)) + off;
        int j = i + s;
        if (j < n) {
          uint64_t x = a[i], y = a[j];
          if (y < x) {
            a[i] = y;
            a[j] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Re-order runs that tie on the sort key (coarse depth, reduced by `shift`
// relative to `cmin`) by the full f64 key, then the source index.
__device__ __forceinline__ uint32_t sort_digits(uint64_t v, uint32_t cmin, int shift) {
  return ((uint32_t)(v >> 32) - cmin) >> shift;
}
__device__ void fix_coarse_ties(uint64_t* a, int n, const uint64_t* key, uint32_t cmin = 0,
                                int shift = 0) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    uint32_t cj = sort_digits(a[j], cmin, shift);
    bool head = (j == 0) || (sort_digits(a[j - 1], cmin, shift) != cj);
    if (!head || j + 1 >= n || sort_digits(a[j + 1], cmin, shift) != cj) continue;
    int e = j + 1;
    while (e < n && sort_digits(a[e], cmin, shift) == cj) ++e;
    // insertion sort a[j..e) by (key64[idx], idx)
    for (int p = j + 1; p < e; ++p) {
      uint64_t v = a[p];
      uint32_t vi = (uint32_t)v;
      uint64_t vk = key[vi];
      int q = p - 1;
      while (q >= j) {
        uint32_t qi = (uint32_t)a[q];
        uint64_t qk = key[qi];
        if (qk > vk || (qk == vk && qi > vi)) {
          a[q + 1] = a[q];
          --q;
        } else {
          break;
        }
      }
      a[q + 1] = v;
    }
  }
}

// Block LSD radix sort of one tile's packed keys (coarse_depth32 << 32 |
// index) in shared memory on the tile-relative key
//     d = (coarse - cmin) >> shift   (at most 24 significant bits)
// in 8-bit digits, only as many passes as d has bytes.  Elements are ranked
// warp by warp in list order (warp-striped: key i = 256 w + 32 e + lane) with
// __match_any_sync peers, so every pass is stable; elements that tie on d are
// put in exact (full key, index) order by fix_coarse_ties afterwards.
constexpr int RS_T = 1024;
constexpr int RS_W = RS_T / 32;
constexpr int RS_E = 8;
constexpr int RS_CAP = RS_T * RS_E;  // 8192 keys per tile in shared memory
constexpr int BK_BITS = 13;          // bucket pass: top 13 bits of the key
constexpr int BK_N = 1 << BK_BITS;
constexpr int BK_BIG = 64;           // larger buckets -> LSD radix fallback
constexpr int BK_BIG_G = 256;        // long lists: larger buckets -> bitonic fallback
constexpr int SEG_MAX = 4096;        // staged segments per tile gathered in parallel

__device__ uint64_t* block_radix_sort(uint64_t* src, uint64_t* dst, int* cnt, int n,
                                      uint32_t cmin, int shift, int npass) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int pass = 0; pass < npass; ++pass) {
    const int sh = 8 * pass;
    int* wc = cnt + warp * 256;
    for (int d = lane; d < 256; d += 32) wc[d] = 0;
    __syncwarp();
    int rank[RS_E];
    int dig[RS_E];
    const int wbase = warp * 32 * RS_E;
    // all peer masks first (independent MATCH latencies overlap), then the
    // per-warp digit counters in element order (stable)
    unsigned peers[RS_E];
#pragma unroll
    for (int e = 0; e < RS_E; ++e) {
      const int i = wbase + e * 32 + lane;
      const bool valid = i < n;
      const int d = valid ? (int)((sort_digits(src[valid ? i : 0], cmin, shift) >> sh) & 0xFF) : 0;
      peers[e] = __match_any_sync(0xffffffffu, valid ? d : 0x1000 + lane);
      dig[e] = valid ? d : -1;
    }
#pragma unroll
    for (int e = 0; e < RS_E; ++e) {
      const int d = dig[e];
      const int leader = __ffs(peers[e]) - 1;
      int old = 0;
      if (d >= 0 && lane == leader) {
        old = wc[d];
        wc[d] = old + __popc(peers[e]);
      }
      old = __shfl_sync(0xffffffffu, old, leader);
      rank[e] = old + __popc(peers[e] & lt);
      __syncwarp();
    }
    __syncthreads();
    // offsets: digit-major, warp-minor
    if (tid < 256) {
      int run = 0;
      for (int w = 0; w < RS_W; ++w) {
        const int c = cnt[w * 256 + tid];
        cnt[w * 256 + tid] = run;
        run += c;
      }
      cnt[RS_W * 256 + tid] = run;  // digit total
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scan of the 256 digit totals (8 per lane)
      int loc[8];
      int sum = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        loc[k] = sum;
        sum += cnt[RS_W * 256 + tid * 8 + k];
      }
      int inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      const int ex = inc - sum;
#pragma unroll
      for (int k = 0; k < 8; ++k) cnt[RS_W * 256 + 256 + tid * 8 + k] = ex + loc[k];
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < RS_E; ++e) {
      const int i = wbase + e * 32 + lane;
      if (i < n) {
        const int d = dig[e];
        dst[cnt[RS_W * 256 + 256 + d] + cnt[warp * 256 + d] + rank[e]] = src[i];
      }
    }
    __syncthreads();
    uint64_t* t = src;
    src = dst;
    dst = t;
  }
  return src;  // buffer holding the result
}

// In-place exclusive scan of c[0 .. PER * RS_T) (PER consecutive counts per
// thread); c[PER * RS_T] = total.  Ends with a barrier.
template <int PER>
__device__ void scan_counts(int* c) {
  int sum = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) sum += c[threadIdx.x * PER + k];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  __shared__ int s_ws[RS_W];
  if (lane == 31) s_ws[wid] = inc;
  __syncthreads();
  int x = s_ws[lane];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += u;
  }
  int run = inc - sum + __shfl_sync(0xffffffffu, x - s_ws[lane], wid);
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int v = c[threadIdx.x * PER + k];
    c[threadIdx.x * PER + k] = run;
    run += v;
  }
  if (threadIdx.x == RS_T - 1) c[PER * RS_T] = run;
  __syncthreads();
}

// One bucket pass of K3 on keys a[0..n) (shared or global memory): bcnt holds
// the BK_N bucket counts on entry; exclusive scan -> bucket starts, scatter
// a -> b by bucket, then every key is ranked inside its (small) bucket by
// (coarse32, index) and written back to a in sorted order.  Ends with the
// CTA's writes to a visible to the CTA.
__device__ void bucket_pass(uint64_t* a, uint64_t* b, int* bcnt, int* bcur, int n,
                            uint32_t cmin, int bshift, long long* dbg = nullptr,
                            long long t_dbg0 = 0) {
  // exclusive scan of the bucket counts (BK_N / blockDim per thread)
  constexpr int PER = BK_N / RS_T;
  int loc[PER];
  int sum = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    loc[k] = sum;
    sum += bcnt[threadIdx.x * PER + k];
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  __shared__ int s_wsum[RS_W];
  if (lane == 31) s_wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    int x = s_wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += u;
    }
    s_wsum[lane] = x;
  }
  __syncthreads();
  const int base0 = inc - sum + (wid > 0 ? s_wsum[wid - 1] : 0);
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int st0 = base0 + loc[k];
    bcur[threadIdx.x * PER + k] = st0;
    bcnt[threadIdx.x * PER + k] = st0;  // bucket start
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const uint64_t v = a[j];
    const int bk = (int)(((uint32_t)(v >> 32) - cmin) >> bshift);
    b[atomicAdd(bcur + bk, 1)] = v;
  }
  __syncthreads();
  if (dbg && threadIdx.x == 0) *dbg = clock64() - t_dbg0;
  // every key's rank inside its bucket: one pass over the (small)
  // bucket per key, all keys in parallel; written to a in sorted order
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const uint64_t v = b[j];
    const int bk = (int)(((uint32_t)(v >> 32) - cmin) >> bshift);
    const int lo = bcnt[bk], hi = bcur[bk];
    int rank = lo;
    for (int i = lo; i < hi; ++i) {
      const uint64_t u = b[i];
      rank += (u < v) || (u == v && i < j);  // equal keys: seam duplicates
    }
    a[rank] = v;
  }
  __syncthreads();
}

// K3 for lists longer than shared memory: one bucket pass on the top GB bits
// of the tile-relative coarse key with the keys in L2 (the list g and a
// scratch slice tmp of the same offsets) and 2^GB bucket cursors in shared
// memory, then whole-bucket windows of <= WCAP keys ranked in shared memory;
// a bucket of >= BK_BIG_G keys falls back to a bitonic sort.
template <int GB>
__device__ void sort_long_list(const SortArgs& A, uint64_t* s_keys, uint64_t* g, int n, int s,
                               uint32_t cmin, uint32_t cmax, long long t_dbg0) {
  constexpr int GN = 1 << GB, WCAP = GB > BK_BITS + 1 ? RS_CAP / 2 : RS_CAP;
  uint64_t* wa = s_keys;
  uint64_t* wb = s_keys + WCAP;
  int* cur = (int*)(s_keys + 2 * WCAP);  // [GN + 1]: counts, then starts, then ends
  const uint32_t span = cmax - cmin;
  const int bits = span ? 32 - __clz(span) : 0;
  const int bshift = bits > GB ? bits - GB : 0;
  __shared__ int s_gbig;
  if (threadIdx.x == 0) s_gbig = 0;
  for (int q = threadIdx.x; q < GN; q += blockDim.x) cur[q] = 0;
  __syncthreads();
  // RS_E keys' loads in flight per thread, then their counter atomics
  for (int j0 = threadIdx.x; j0 < n; j0 += RS_CAP) {
    uint64_t v[RS_E];
#pragma unroll
    for (int e = 0; e < RS_E; ++e) {
      const int j = j0 + e * RS_T;
      v[e] = j < n ? __ldcg(g + j) : 0;
    }
#pragma unroll
    for (int e = 0; e < RS_E; ++e) {
      if (j0 + e * RS_T < n) {
        const int bk = (int)(((uint32_t)(v[e] >> 32) - cmin) >> bshift);
        if (atomicAdd(cur + bk, 1) == BK_BIG_G) s_gbig = 1;
      }
    }
  }
  __syncthreads();
  if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 3] = clock64() - t_dbg0;
  if (s_gbig || !A.sort_tmp) {
    bitonic_sort<false>(g, n);  // in place in global memory (L2 resident)
    __syncthreads();
    fix_coarse_ties(g, n, A.key);
    __syncthreads();
    return;
  }
  uint64_t* tmp = A.sort_tmp + s;
  scan_counts<GN / RS_T>(cur);  // cur = bucket starts
  for (int j0 = threadIdx.x; j0 < n; j0 += RS_CAP) {  // scatter by bucket
    uint64_t v[RS_E];
#pragma unroll
    for (int e = 0; e < RS_E; ++e) {
      const int j = j0 + e * RS_T;
      v[e] = j < n ? __ldcg(g + j) : 0;
    }
#pragma unroll
    for (int e = 0; e < RS_E; ++e) {
      if (j0 + e * RS_T < n) {
        const int bk = (int)(((uint32_t)(v[e] >> 32) - cmin) >> bshift);
        tmp[atomicAdd(cur + bk, 1)] = v[e];
      }
    }
  }
  __syncthreads();  // cur = bucket ends (bucket b starts at cur[b - 1])
  if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 4] = clock64() - t_dbg0;
  for (int w0 = 0; w0 < n;) {
    // window end: the last bucket end <= w0 + WCAP (a bucket holds fewer
    // than BK_BIG_G < WCAP keys, so the window is not empty)
    int w1 = n;
    if (w0 + WCAP < n) {
      int b = -1;
#pragma unroll
      for (int step = GN / 2; step >= 1; step >>= 1)
        if (cur[b + step] <= w0 + WCAP) b += step;
      w1 = cur[b];
    }
    const int len = w1 - w0;
#pragma unroll
    for (int e = 0; e < WCAP / RS_T; ++e) {
      const int j = threadIdx.x + e * RS_T;
      if (j < len) wa[j] = __ldcg(tmp + w0 + j);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < len; j += blockDim.x) {
      const uint64_t v = wa[j];
      const int bk = (int)(((uint32_t)(v >> 32) - cmin) >> bshift);
      const int lo = (bk ? cur[bk - 1] : 0) - w0, hi = cur[bk] - w0;
      int rank = lo;
      for (int i = lo; i < hi; ++i) {
        const uint64_t u = wa[i];
        rank += (u < v) || (u == v && i < j);  // equal keys: seam duplicates
      }
      wb[rank] = v;
    }
    __syncthreads();
    fix_coarse_ties(wb, len, A.key);  // a coarse-key run lies inside one bucket
    __syncthreads();
    for (int j = threadIdx.x; j < len; j += blockDim.x) g[w0 + j] = wb[j];
    __syncthreads();
    w0 = w1;
  }
  if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 5] = clock64() - t_dbg0;
}

// Gather each tile's staged segments, sort them by (coarse depth, index),
// fix coarse ties by the full f64 key and write the tile's list.
__global__ void __launch_bounds__(RS_T) k_tile_sort(SortArgs A) {
  const long long t_dbg0 = clock64();
  if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 14] = gtimer();
  pdl_trigger();  // pass A may be scheduled now; it waits on A.ready per tile
  // launched as a dependent of K2: every histogram and segment is written
  // once K2's grid has completed
  pdl_wait();
  if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 0] = clock64() - t_dbg0;
  extern __shared__ uint64_t s_keys[];  // 2 * RS_CAP keys + counters
  __shared__ int s_pos, s_ovf;
  __shared__ int s_w[2][RS_W];
  __shared__ uint32_t s_mm[2];
  const int t = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned full = 0xffffffffu;
  // every global read of the prologue is issued before the first wait: the
  // overflow flag, this tile's count and the counts before it (its list
  // offset), and the staged-segment descriptors.  Warp w takes segments
  // [w S, w S + S), S = ceil(nseg / 32): lane l holds segment w S + 32 k + l.
  const int nseg = (int)A.seg_stride;  // one slot per preprocess CTA (length 0: empty)
  const int2* sg = A.seg + (int64_t)t * A.seg_stride;
  const bool seg_fast = nseg <= SEG_MAX;
  const int S = (nseg + 31) >> 5;
  if (tid == 0) {
    s_ovf = __ldcg(A.counters + GSPARC_CNT_OVERFLOW);
    s_pos = 0;
    s_mm[0] = 0xFFFFFFFFu;
    s_mm[1] = 0u;
  }
  const int n = __ldcg(A.tile_count + t);
  int pre_t = 0;
  for (int i = tid; i < t; i += RS_T) pre_t += __ldcg(A.tile_count + i);
  int2 d[SEG_MAX / RS_T];
#pragma unroll
  for (int k = 0; k < SEG_MAX / RS_T; ++k) {
    const int r = 32 * k + lane, j = warp * S + r;
    d[k] = seg_fast && r < S && j < nseg ? __ldcg(sg + j) : make_int2(0, 0);
  }
  // segment positions inside the tile's list: scan in (warp, k, lane) order
  int rowpre[SEG_MAX / RS_T];
  int wtot = 0;
#pragma unroll
  for (int k = 0; k < SEG_MAX / RS_T; ++k) {
    int inc = d[k].y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(full, inc, o);
      if (lane >= o) inc += u;
    }
    rowpre[k] = wtot + inc - d[k].y;
    wtot += __shfl_sync(full, inc, 31);
  }
  pre_t = __reduce_add_sync(full, pre_t);
  if (lane == 0) {
    s_w[0][warp] = wtot;
    s_w[1][warp] = pre_t;
  }
  __syncthreads();
  const int s = __reduce_add_sync(full, s_w[1][lane]);  // tile_start[t]
  int wbase = s_w[0][lane];
  {
    int inc = wbase;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(full, inc, o);
      if (lane >= o) inc += u;
    }
    wbase = __shfl_sync(full, inc - wbase, warp);
  }
  if (A.dbg && tid == 0) A.dbg[blockIdx.x * 16 + 1] = clock64() - t_dbg0;
  if (s_ovf) {
    // the staged pairs are incomplete: no list, but the tile is still
    // published so that pass-A CTAs waiting on the queue see the overflow
    // (K2 has completed, so the flag is final) and exit
    if (tid == 0) {
      A.tile_start[t] = s;
      A.tile_start[t + 1] = s + n;
      __threadfence();
      const int q = atomicAdd(A.counters + GSPARC_CNT_SORTED, 1);
      flag_release(A.ready + q, t + 1);
    }
    return;
  }
  uint64_t* g = A.pairs + s;
  uint32_t lo = 0xFFFFFFFFu, hi = 0u;
  if (seg_fast) {
    // segment table in shared memory (the bucket counters' space, unused
    // until the histogram): offset, length, list position
    int* s_soff = (int*)(s_keys + 2 * RS_CAP);
    int* s_slen = s_soff + SEG_MAX;
    int* s_spre = s_slen + SEG_MAX;
    const int mybase = wbase;
#pragma unroll
    for (int k = 0; k < SEG_MAX / RS_T; ++k) {
      const int r = 32 * k + lane, j = warp * S + r;
      if (r < S && j < nseg) {
        s_soff[j] = d[k].x;
        s_slen[j] = d[k].y;
        s_spre[j] = mybase + rowpre[k];
      }
    }
    __syncthreads();
    // windows of RS_CAP keys (one for lists that fit shared memory, else
    // written to the list in L2): warp w gathers the window's keys
    // [32 per w, 32 per (w + 1)), lane l the keys 32 e + l of that block, so
    // every load instruction reads consecutive keys; a lane binary-searches
    // the segment positions for its first key and walks forward from there.
    // All of a thread's loads are in flight together.
    for (int w0 = 0; w0 < n; w0 += RS_CAP) {
      const int nw = min(n - w0, RS_CAP);
      const int per = (nw + RS_T - 1) / RS_T;  // <= RS_E
      const int j0 = w0 + warp * 32 * per + lane, jend = w0 + nw;
      uint64_t v[RS_E];
      if (j0 < jend) {
        int l = 0;  // last segment with position <= j0
        for (int step = 1 << (31 - __clz(nseg)); step >= 1; step >>= 1)
          if (l + step < nseg && s_spre[l + step] <= j0) l += step;
        int sbeg = s_spre[l], send = sbeg + s_slen[l], soff = s_soff[l];
#pragma unroll
        for (int e = 0; e < RS_E; ++e) {
          const int j = j0 + 32 * e;
          v[e] = 0;
          if (e < per && j < jend) {
            while (j >= send) {  // segment holding key j
              ++l;
              sbeg = s_spre[l];
              send = sbeg + s_slen[l];
              soff = s_soff[l];
            }
            v[e] = __ldcg(A.stage + soff + (j - sbeg));
          }
        }
#pragma unroll
        for (int e = 0; e < RS_E; ++e) {
          const int j = j0 + 32 * e;
          if (e < per && j < jend) {
            if (n <= RS_CAP)
              s_keys[j] = v[e];
            else
              g[j] = v[e];
            const uint32_t c = (uint32_t)(v[e] >> 32);
            lo = min(lo, c);
            hi = max(hi, c);
          }
        }
      }
    }
    if (A.dbg && tid == 0) A.dbg[blockIdx.x * 16 + 9] = clock64() - t_dbg0;
  } else {  // one thread per staged segment (any order, the sort is total)
    uint64_t* dst = n <= RS_CAP ? s_keys : g;
    for (int j = tid; j < nseg; j += blockDim.x) {
      const int2 dj = __ldcg(sg + j);
      const int p = atomicAdd(&s_pos, dj.y);
      const uint64_t* src = A.stage + dj.x;
      for (int k = 0; k < dj.y; ++k) {
        const uint64_t x = __ldcg(src + k);
        dst[p + k] = x;
        const uint32_t c = (uint32_t)(x >> 32);
        lo = min(lo, c);
        hi = max(hi, c);
      }
    }
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&s_mm[0], lo);
    atomicMax(&s_mm[1], hi);
  }
  __syncthreads();
  if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 2] = clock64() - t_dbg0;
  if (n > 1 && n <= RS_CAP) {
    uint64_t* a = s_keys;
    uint64_t* b = s_keys + RS_CAP;
    int* cnt = (int*)(s_keys + 2 * RS_CAP);
    const uint32_t cmin = s_mm[0], span = s_mm[1] - s_mm[0];
    const int bits = span ? 32 - __clz(span) : 0;
    // one bucket pass on the top 13 bits of the tile-relative coarse key
    // (shared-memory atomics; order inside a bucket is fixed next), then
    // every key is ranked by (coarse32, index) inside its bucket and runs
    // tying on coarse32 are put in exact (f64 key, index) order
    const int bshift = bits > BK_BITS ? bits - BK_BITS : 0;
    int* bcnt = cnt;              // [BK_N]
    int* bcur = cnt + BK_N;       // [BK_N]
    __shared__ int s_bmax;
    if (threadIdx.x == 0) s_bmax = 0;
    for (int t = threadIdx.x; t < BK_N; t += blockDim.x) bcnt[t] = 0;
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const int bk = (int)(((uint32_t)(a[j] >> 32) - cmin) >> bshift);
      const int c = atomicAdd(bcnt + bk, 1);
      if (c == BK_BIG) atomicMax(&s_bmax, c);
    }
    __syncthreads();
    if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 3] = clock64() - t_dbg0;
    uint64_t* r;
    if (s_bmax < BK_BIG) {
      bucket_pass(a, b, bcnt, bcur, n, cmin, bshift, A.dbg ? A.dbg + blockIdx.x * 16 + 4 : nullptr, t_dbg0);
      __syncthreads();
      if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 5] = clock64() - t_dbg0;
      r = a;
      fix_coarse_ties(r, n, A.key);
    } else {  // a heavily populated bucket: stable LSD radix passes
      const int shift = bits > 24 ? bits - 24 : 0;
      const int npass = (bits - shift + 7) / 8;  // 0..3
      r = block_radix_sort(a, b, cnt, n, cmin, shift, npass);
      fix_coarse_ties(r, n, A.key, cmin, shift);
    }
    __syncthreads();
    if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 7] = clock64() - t_dbg0;
    for (int j = threadIdx.x; j < n; j += blockDim.x) g[j] = r[j];
  } else if (n == 1) {
    if (threadIdx.x == 0) g[0] = s_keys[0];
  } else if (n > RS_CAP) {
    if (threadIdx.x == 0) atomicAdd(A.counters + GSPARC_CNT_BIGTILE, 1);
    // (2^15 + 1 cursors fit behind two half windows: 64 + 128 KB)
    if (A.long_bits == 15)
      sort_long_list<15>(A, s_keys, g, n, s, s_mm[0], s_mm[1], t_dbg0);
    else if (A.long_bits == 14)
      sort_long_list<14>(A, s_keys, g, n, s, s_mm[0], s_mm[1], t_dbg0);
    else
      sort_long_list<13>(A, s_keys, g, n, s, s_mm[0], s_mm[1], t_dbg0);
  }
  if (A.inv) {  // deterministic backward: list position of (Gaussian, tile slot)
    __syncthreads();
    const int ty = t / A.ntx, tx = t - ty * A.ntx;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const uint64_t v = g[j];
      if (j > 0 && g[j - 1] == v) continue;  // second copy of a seam duplicate
      const uint32_t idx = (uint32_t)v;
      const int4 rc = __ldg(A.rect + idx);
      const int y0 = rc.x & 0xffff, a0 = rc.y & 0xffff, a1 = rc.y >> 16, b1 = rc.z >> 16;
      const int na = a1 - a0 + 1, nbo = b1 >= 0 ? min(b1, a0 - 1) + 1 : 0;
      const int slot = (ty - y0) * (na + nbo) + (tx >= a0 && tx <= a1 ? tx - a0 : na + tx);
      // slot < rows * (na + nbo) <= nty * ntx: the table has ntiles slots
      // per Gaussian (capi.cu gsparc_plan_frame), so no slot is dropped
      A.inv[(int64_t)idx * A.ntiles + slot] = s + j;
    }
  }
  // publish the tile: its bounds (same values CTA 0 wrote) and list, then
  // its id in the next slot of the K3 -> K4a queue (pass A's CTAs take
  // tiles in the order their sorts finish)
  __syncthreads();
  if (threadIdx.x == 0) {
    A.tile_start[t] = s;
    A.tile_start[t + 1] = s + n;
    __threadfence();
    const int q = atomicAdd(A.counters + GSPARC_CNT_SORTED, 1);
    flag_release(A.ready + q, t + 1);
  }
  if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 15] = gtimer();
}

int launch_bin_tiles(const gsparc_frame_layout& L, char* frame, cudaStream_t st, bool dependent) {
  SortArgs A;
  A.pairs = (uint64_t*)(frame + L.off_pairs);
  A.tile_start = (int*)(frame + L.off_tile_start);
  A.key = (const uint64_t*)(frame + L.off_key);
  A.counters = (int*)(frame + L.off_counters);
  A.tile_count = (const int*)(frame + L.off_tile_count);
  A.ready = (int*)(frame + L.off_tile_cursor);
  A.seg = (const int2*)(frame + L.off_seg);
  A.stage = (const uint64_t*)(frame + L.off_stage);
  A.seg_stride = L.seg_stride;
  A.inv = L.with_backward == 2 ? (int*)(frame + L.off_det_inv) : nullptr;
  A.sort_tmp = (uint64_t*)(frame + L.off_sort_tmp);
  A.rect = (const int4*)(frame + L.off_rect);
  A.ntx = L.ntx;
  A.ntiles = L.ntiles;
  A.dbg = nullptr;
  A.long_bits = experiment_env("GSPARC_SORT_LBITS") ? atoi(experiment_env("GSPARC_SORT_LBITS")) : 14;
  if (experiment_env("GSPARC_SORT_DBG")) A.dbg = dbg_rows(0);  // experiments only
  const size_t cnt_ints =
      (size_t)max(RS_W * 256 + 512, 2 * BK_N + 1);
  const size_t smem_sort = 2 * RS_CAP * sizeof(uint64_t) + sizeof(int) * cnt_ints;
  static_assert(2 * RS_CAP * sizeof(uint64_t) + sizeof(int) * (2 * BK_N + 1) <= 227 * 1024,
                "k_tile_sort shared memory");
  static size_t attr_set = 0;
  if (attr_set < smem_sort) {
    cudaFuncSetAttribute(k_tile_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_sort);
    attr_set = smem_sort;
  }
  // dependent launch behind K2 on the lazy render path (config 3: -0.5 us);
  // ahead of the full MLP (config 1) it measured 5 us slower, so there the
  // sort is an ordinary launch (griddepcontrol.wait then returns at once)
  static const bool pdl_env = !getenv("GSPARC_NO_PDL") && !experiment_env("GSPARC_NO_PDL_K3");
  const bool pdl = pdl_env && dependent;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(L.ntiles);
  cfg.blockDim = dim3(RS_T);
  cfg.dynamicSmemBytes = smem_sort;
  cfg.stream = st;
  if (pdl) {  // K2 triggers at its start; this launch then waits for it on the device
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  cudaLaunchKernelEx(&cfg, k_tile_sort, A);
  return check_launch("k_tile_sort");
}

}  // namespace gs
