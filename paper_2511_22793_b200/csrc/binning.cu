// K3: tile binning and per-tile depth sort.  Replaces the np.lexsort depth
// order (rasterizer.py:82-87) and rasterizer._tile_lists
// (rasterizer.py:115-145).
//
// This is an MSD radix sort on the composite key (tile, depth, index):
//   digit 1 (tile) -- counting sort: per-tile counts come from K2, an
//     exclusive scan gives the tile ranges, every Gaussian is scattered into
//     the buckets of the tiles its footprint covers (the azimuth-seam
//     duplicate included: a tile covered by both column segments gets two
//     entries, rasterizer.py:139-141);
//   digits 2.. (depth, index) -- every bucket is sorted in shared memory by
//     the packed key (coarse_depth32 << 32 | index).  coarse_depth32 is the
//     monotone truncation (bits(depth) - bits(0.05)) >> 24; runs that tie on
//     it are re-ordered by the full f64 bit pattern, so the final order is
//     exactly np.lexsort((idx, depth)) restricted to the tile.
#include "common.cuh"
#include "kernels.cuh"

namespace gs {

struct BinArgs {
  const uint64_t* key;
  const int4* rect;
  const int* tile_count;
  int* tile_cursor;
  int* tile_start;
  int* counters;
  uint64_t* pairs;
  int64_t capacity;
  int64_t n;
  int ntx, ntiles;
};

__device__ __forceinline__ uint32_t coarse_key(uint64_t k) {
  return (uint32_t)((k - DEPTH_KEY_BASE) >> COARSE_SHIFT);
}

// Block-wide exclusive scan of `in[0..n)` into `out[0..n]` (out[n] = total),
// any n, blockDim multiple of 32.  Uses `tmp` of blockDim/32+1 ints.
__device__ void block_exclusive_scan(const int* in, int* out, int n, int* tmp) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (n + nt - 1) / nt;
  const int beg = min(n, tid * per), end = min(n, beg + per);
  int local = 0;
  for (int k = beg; k < end; ++k) local += in[k];
  // inclusive warp scan of `local`
  int lane = tid & 31, warp = tid >> 5;
  int v = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  if (lane == 31) tmp[warp] = v;
  __syncthreads();
  if (warp == 0) {
    int nw = nt >> 5;
    int w = lane < nw ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += u;
    }
    if (lane < nw) tmp[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  int run = v - local + (warp > 0 ? tmp[warp - 1] : 0);
  for (int k = beg; k < end; ++k) {
    out[k] = run;
    run += in[k];
  }
  if (tid == nt - 1) out[n] = run;
  __syncthreads();
}

__device__ __forceinline__ void unpack_rect(int4 r, int& y0, int& y1, int& a0, int& a1, int& b0,
                                            int& b1) {
  y0 = r.x & 0xffff;
  y1 = r.x >> 16;
  a0 = r.y & 0xffff;
  a1 = r.y >> 16;
  b0 = r.z & 0xffff;
  b1 = r.z >> 16;
}

__global__ void __launch_bounds__(256) k_bin(BinArgs A) {
  extern __shared__ int sm[];
  const int T = A.ntiles;
  int* s_start = sm;             // T+1
  int* s_cnt = s_start + T + 1;  // T
  int* s_base = s_cnt + T;       // T
  int* s_tmp = s_base + T;       // 33
  block_exclusive_scan(A.tile_count, s_start, T, s_tmp);
  const int total = s_start[T];
  if (blockIdx.x == 0) {
    for (int t = threadIdx.x; t <= T; t += blockDim.x) A.tile_start[t] = s_start[t];
    if (threadIdx.x == 0 && total > A.capacity) A.counters[GSPARC_CNT_OVERFLOW] = 1;
  }
  if (total > A.capacity) return;  // host reports the overflow
  for (int t = threadIdx.x; t < T; t += blockDim.x) s_cnt[t] = 0;
  __syncthreads();

  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t k = (i < A.n) ? A.key[i] : ~0ULL;
  const bool kept = k != ~0ULL;
  int y0 = 0, y1 = -1, a0 = 0, a1 = -1, b0 = 0, b1 = -1;
  if (kept) {
    unpack_rect(A.rect[i], y0, y1, a0, a1, b0, b1);
    for (int ty = y0; ty <= y1; ++ty) {
      for (int tx = a0; tx <= a1; ++tx) atomicAdd(s_cnt + ty * A.ntx + tx, 1);
      for (int tx = b0; tx <= b1; ++tx) atomicAdd(s_cnt + ty * A.ntx + tx, 1);
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    int c = s_cnt[t];
    s_base[t] = c ? s_start[t] + atomicAdd(A.tile_cursor + t, c) : 0;
    s_cnt[t] = 0;
  }
  __syncthreads();
  if (kept) {
    const uint64_t packed = ((uint64_t)coarse_key(k) << 32) | (uint32_t)i;
    for (int ty = y0; ty <= y1; ++ty) {
      for (int tx = a0; tx <= a1; ++tx) {
        int t = ty * A.ntx + tx;
        A.pairs[s_base[t] + atomicAdd(s_cnt + t, 1)] = packed;
      }
      for (int tx = b0; tx <= b1; ++tx) {
        int t = ty * A.ntx + tx;
        A.pairs[s_base[t] + atomicAdd(s_cnt + t, 1)] = packed;
      }
    }
  }
}

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

// Register bitonic sort of up to 8192 keys per CTA (1024 threads x 8 keys,
// blocked layout i = 8*tid + e).  Compare-exchange partners at index
// distance < 8 are in the same thread, < 256 in the same warp (shuffles),
// larger go through shared memory.  All comparators put the minimum at the
// lower index (ascending-only network), so the virtual +inf padding never
// moves and is never stored.
constexpr int RB_E = 8;
constexpr int RB_T = 1024;
constexpr int RB_CAP = RB_E * RB_T;

__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src);
  const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}

// in-thread compare-exchange of x[e] with x[e ^ D] (D compile time)
template <int D>
__device__ __forceinline__ void cx_local(uint64_t (&x)[RB_E]) {
#pragma unroll
  for (int e = 0; e < RB_E; ++e) {
    if ((e ^ D) > e) {
      const uint64_t a = x[e], b = x[e ^ D];
      x[e] = a < b ? a : b;
      x[e ^ D] = a < b ? b : a;
    }
  }
}

// cross-thread step: partner thread t ^ tm; MIRROR pairs element e with the
// partner's 7 - e (first merge step), otherwise with the partner's e.
template <bool MIRROR>
__device__ __forceinline__ void cx_remote(uint64_t (&x)[RB_E], uint64_t* sm, int tm,
                                          bool lo_half) {
  const int t = threadIdx.x;
  uint64_t y[RB_E];
  if (tm < 32) {
#pragma unroll
    for (int e = 0; e < RB_E; ++e) y[e] = shfl64(x[MIRROR ? RB_E - 1 - e : e], (t & 31) ^ tm);
  } else {
    __syncthreads();
#pragma unroll
    for (int e = 0; e < RB_E; ++e) sm[t * RB_E + e] = x[e];
    __syncthreads();
    const int pt = t ^ tm;
#pragma unroll
    for (int e = 0; e < RB_E; ++e) y[e] = sm[pt * RB_E + (MIRROR ? RB_E - 1 - e : e)];
  }
#pragma unroll
  for (int e = 0; e < RB_E; ++e) {
    const uint64_t a = x[e], b = y[e];
    x[e] = lo_half ? (a < b ? a : b) : (a < b ? b : a);
  }
}

__device__ void reg_bitonic(uint64_t (&x)[RB_E], uint64_t* sm, int np2) {
  const int t = threadIdx.x;
  // k = 2, 4, 8: entirely inside the thread (mirror + cleaners)
  cx_local<1>(x);
  cx_local<3>(x);
  cx_local<1>(x);
  cx_local<7>(x);
  cx_local<2>(x);
  cx_local<1>(x);
  for (int k = 16; k <= np2; k <<= 1) {
    cx_remote<true>(x, sm, (k - 1) >> 3, (t & (k >> 4)) == 0);
    for (int s = k >> 2; s >= RB_E; s >>= 1) cx_remote<false>(x, sm, s >> 3, (t & (s >> 3)) == 0);
    cx_local<4>(x);
    cx_local<2>(x);
    cx_local<1>(x);
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

// Sort each tile's bucket by (coarse depth, index), fix coarse ties by the
// full f64 key, then stage the f32 raster record of every entry in list
// order (pair_rec) so the raster streams records instead of gathering them.
__global__ void __launch_bounds__(RS_T) k_tile_sort(uint64_t* pairs, const int* tile_start,
                                                    const uint64_t* key, int* counters,
                                                    const float4* rec32, float4* pair_rec,
                                                    int /*unused*/) {
  extern __shared__ uint64_t s_keys[];  // 2 * RS_CAP keys + counters
  if (counters[GSPARC_CNT_OVERFLOW]) return;
  const int t = blockIdx.x;
  const int s = tile_start[t], n = tile_start[t + 1] - s;
  uint64_t* g = pairs + s;
  if (n > 1 && n <= RS_CAP) {
    uint64_t* a = s_keys;
    uint64_t* b = s_keys + RS_CAP;
    int* cnt = (int*)(s_keys + 2 * RS_CAP);
    __shared__ uint32_t s_mm[2];
    if (threadIdx.x == 0) {
      s_mm[0] = 0xFFFFFFFFu;
      s_mm[1] = 0u;
    }
    __syncthreads();
    uint32_t lo = 0xFFFFFFFFu, hi = 0u;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const uint64_t v = g[j];
      a[j] = v;
      const uint32_t c = (uint32_t)(v >> 32);
      lo = min(lo, c);
      hi = max(hi, c);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&s_mm[0], lo);
      atomicMax(&s_mm[1], hi);
    }
    __syncthreads();
    const uint32_t cmin = s_mm[0], span = s_mm[1] - s_mm[0];
    const int bits = span ? 32 - __clz(span) : 0;
    // one bucket pass on the top 13 bits of the tile-relative coarse key
    // (shared-memory atomics; order inside a bucket is fixed next), then
    // every bucket is insertion-sorted by (coarse32, index) and runs tying
    // on coarse32 are put in exact (f64 key, index) order
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
    uint64_t* r;
    if (s_bmax < BK_BIG) {
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
      for (int bk = threadIdx.x; bk < BK_N; bk += blockDim.x) {
        const int lo = bcnt[bk], hi = bcur[bk];
        for (int p = lo + 1; p < hi; ++p) {  // insertion sort, buckets are small
          const uint64_t v = b[p];
          int q = p - 1;
          while (q >= lo && b[q] > v) {
            b[q + 1] = b[q];
            --q;
          }
          b[q + 1] = v;
        }
      }
      __syncthreads();
      r = b;
      fix_coarse_ties(r, n, key);
    } else {  // a heavily populated bucket: stable LSD radix passes
      const int shift = bits > 24 ? bits - 24 : 0;
      const int npass = (bits - shift + 7) / 8;  // 0..3
      r = block_radix_sort(a, b, cnt, n, cmin, shift, npass);
      fix_coarse_ties(r, n, key, cmin, shift);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) g[j] = r[j];
  } else if (n > RS_CAP) {
    if (threadIdx.x == 0) atomicAdd(counters + GSPARC_CNT_BIGTILE, 1);
    bitonic_sort<false>(g, n);  // in place in global memory (L2 resident)
    fix_coarse_ties(g, n, key);
    __syncthreads();
  }
  if (pair_rec) {
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const uint32_t idx = (uint32_t)g[j];
      const float4 a4 = __ldg(rec32 + 2 * idx), b4 = __ldg(rec32 + 2 * idx + 1);
      pair_rec[2 * (size_t)(s + j)] = a4;
      pair_rec[2 * (size_t)(s + j) + 1] = make_float4(b4.x, b4.y, __int_as_float((int)idx), 0.f);
    }
  }
}

int launch_bin_tiles(const gsparc_frame_layout& L, char* frame, cudaStream_t st) {
  BinArgs A;
  A.key = (const uint64_t*)(frame + L.off_key);
  A.rect = (const int4*)(frame + L.off_rect);
  A.tile_count = (const int*)(frame + L.off_tile_count);
  A.tile_cursor = (int*)(frame + L.off_tile_cursor);
  A.tile_start = (int*)(frame + L.off_tile_start);
  A.counters = (int*)(frame + L.off_counters);
  A.pairs = (uint64_t*)(frame + L.off_pairs);
  A.capacity = L.pair_capacity;
  A.n = L.n;
  A.ntx = L.ntx;
  A.ntiles = L.ntiles;
  if (cudaMemsetAsync(A.tile_cursor, 0, sizeof(int) * L.ntiles, st) != cudaSuccess)
    return check_launch("bin memset");
  int blocks = (int)((L.n + 255) / 256);
  if (blocks < 1) blocks = 1;
  size_t smem = sizeof(int) * (3 * (size_t)L.ntiles + 1 + 40);
  k_bin<<<blocks, 256, smem, st>>>(A);
  GS_TRY(check_launch("k_bin"));
  const size_t smem_sort =
      2 * RS_CAP * sizeof(uint64_t) + sizeof(int) * (size_t)max(RS_W * 256 + 512, 2 * BK_N);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_tile_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_sort);
    attr_set = true;
  }
  int idx_bits = 8;
  while (idx_bits < 32 && ((int64_t)1 << idx_bits) < L.n) idx_bits += 8;
  float4* pair_rec = nullptr;  // the f32 raster gathers rrec by index
  k_tile_sort<<<L.ntiles, RS_T, smem_sort, st>>>(A.pairs, A.tile_start, A.key, A.counters,
                                           (const float4*)(frame + L.off_rec32), pair_rec,
                                           idx_bits);
  return check_launch("k_tile_sort");
}

}  // namespace gs
