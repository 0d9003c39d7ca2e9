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

// Re-order runs that tie on the coarse 32-bit depth by the full f64 key.
__device__ void fix_coarse_ties(uint64_t* a, int n, const uint64_t* key) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    uint32_t cj = (uint32_t)(a[j] >> 32);
    bool head = (j == 0) || ((uint32_t)(a[j - 1] >> 32) != cj);
    if (!head || j + 1 >= n || (uint32_t)(a[j + 1] >> 32) != cj) continue;
    int e = j + 1;
    while (e < n && (uint32_t)(a[e] >> 32) == cj) ++e;
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

__global__ void __launch_bounds__(1024) k_tile_sort(uint64_t* pairs, const int* tile_start,
                                                    const uint64_t* key, int* counters, int cap) {
  extern __shared__ uint64_t s_pairs[];
  if (counters[GSPARC_CNT_OVERFLOW]) return;
  const int t = blockIdx.x;
  const int s = tile_start[t], n = tile_start[t + 1] - s;
  if (n <= 1) return;
  uint64_t* g = pairs + s;
  if (n <= cap) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) s_pairs[j] = g[j];
    __syncthreads();
    bitonic_sort<true>(s_pairs, n);
    fix_coarse_ties(s_pairs, n, key);
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x) g[j] = s_pairs[j];
  } else {
    if (threadIdx.x == 0) atomicAdd(counters + GSPARC_CNT_BIGTILE, 1);
    bitonic_sort<false>(g, n);  // in place in global memory (L2 resident)
    fix_coarse_ties(g, n, key);
  }
}

constexpr int SORT_SMEM_CAP = 16384;  // 128 KiB of u64 per tile in smem

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
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_tile_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         SORT_SMEM_CAP * (int)sizeof(uint64_t));
    attr_set = true;
  }
  k_tile_sort<<<L.ntiles, 1024, SORT_SMEM_CAP * sizeof(uint64_t), st>>>(
      A.pairs, A.tile_start, A.key, A.counters, SORT_SMEM_CAP);
  return check_launch("k_tile_sort");
}

}  // namespace gs
