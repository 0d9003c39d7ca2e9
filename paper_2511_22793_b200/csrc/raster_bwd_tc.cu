// K5 (f32 frames, 16 <= Cp <= 64 channels = batched TX x C): the backward of
// the compositing with both channel contractions on the tensor cores.
// Replaces the per-tile loop of rasterizer.rasterize_backward
// (rasterizer.py:286-326), batched over transmitters (Cp = B*C columns).
//
// For a half tile (128 pixels, lane = pixel) and a batch of 32 list entries
// (back to front), the two contractions over channels are GEMMs:
//   UC[p, j] = sum_c u[p, c] coef[j, c]        (u = dL/dimg; needed by the
//              scan: d alpha = T_b uc - suffix / (1 - alpha))
//   GC[c, j] = sum_p u[p, c] wgt[p, j]         (dL/dcoef, the rows K6 reads)
// run as tcgen05.mma kind::tf32 with the 3xTF32 split (hi.hi + hi.lo +
// lo.hi, f32 accumulate in TMEM, ~2^-21 relative):
//   GEMM 1: D1[128 px, 32] = U[128 px, Kp] . Coef^T     A = U in TMEM (ts),
//           B = the batch's coef rows, K-major SWIZZLE_128B in shared memory
//   GEMM 2: D2[128 ch, 32] = U^T[128 ch, 128 px] . W    A = U^T, K-major
//           SW128 in shared memory (rows >= 64 read the next K block: finite
//           data, their accumulator rows are never read); B = the batch's
//           weights T_b alpha written by the scan threads, K-major SW128.
// Only the sequential back-to-front scan (alpha, T, the suffix sum, the
// geometric gradients of rasterizer.py:302-321) stays on the CUDA cores.
//
// Warp roles (320 threads, one CTA per half tile):
//   0-3  scan: pixel per lane (TMEM lane quadrant = warp), 32 entries per
//        batch fully unrolled; warp-reduced geometric gradients
//   4-5, 8-9  GEMM-2 epilogue: lane = channel, 16 entries each per tcgen05.ld
//   6    loader: the batch's list entries, raster records and coef rows
//        (split hi/lo, swizzled) one batch ahead
//   7    MMA issuer (one thread): GEMM 1 of batch b+1 before GEMM 2 of b
// Accumulation into gcoef / ggeo: atomics, or (deterministic frames) the
// per-(list entry, half tile) partials k_bwd_reduce sums in a fixed order
// (nsub = 2).
#include "common.cuh"
#include "kernels.cuh"

namespace gs {

namespace {

constexpr int TC_NB = 32;           // entries per batch (GEMM N)
constexpr int TC_KMAX = 64;         // channels (GEMM-1 K) supported
constexpr int TC_NS = 4;            // coef / record stages (loader runs ahead)
constexpr int K5_CCAP = 768;        // chunks per half tile for the compacted walk (else list walk)
constexpr uint32_t TC_TMEM_COLS = 256;
// TMEM columns: U hi [0,64) | U lo [64,128) | D1 x2 [128,192) | D2 x2 [192,256)
constexpr uint32_t COL_UHI = 0, COL_ULO = 64, COL_D1 = 128, COL_D2 = 192;

// shared memory (bytes, from a 1024-aligned base)
constexpr int COEF_PLANE = 2 * 4096;          // 2 K blocks x 32 rows x 128 B
constexpr int COEF_STAGE = 2 * COEF_PLANE;    // hi | lo
constexpr int UT_KB = 8192;                   // 64 channel rows x 128 B per 32-px block
constexpr int UT_PLANE = 4 * UT_KB + UT_KB;   // 4 K blocks + pad (rows 64..127 of the last)
constexpr int W_PLANE = 4 * 4096;             // 4 K blocks x 32 entry rows x 128 B
constexpr int W_STAGE = 2 * W_PLANE;
constexpr int OFF_COEF = 0;
constexpr int OFF_UT = OFF_COEF + TC_NS * COEF_STAGE;
constexpr int OFF_W = OFF_UT + 2 * UT_PLANE;
constexpr int SMEM_TC = OFF_W + 2 * W_STAGE + 1024;  // + alignment slack

struct TcShared {
  float4 fr[TC_NS][TC_NB][3];        // raster records per coef stage (+ conic, sigma)
  int idx[TC_NS][TC_NB];             // source index | bit 31: first copy of a seam duplicate
  float red[2][TC_NB][4][6];     // per scan warp geometric partial sums
  int cs[K5_CCAP + 1];           // compacted walk: used entries before each chunk
  uint64_t coef_full[TC_NS], stage_empty[TC_NS], d1_full[2], d1_empty[2];
  uint64_t w_full[2], w_empty[2], d2_full[2], d2_empty[2], red_full[2], red_empty[2];
  uint32_t tmem;
};

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   su32(b))
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra W_%=;\n\t}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// helper warps (loader, MMA issue, epilogue) wait with a sleeping back-off:
// a spinning helper would take issue slots from the scan warp sharing its
// scheduler
__device__ __forceinline__ void bar_wait_sleep(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(100);
  }
}
__device__ __forceinline__ void tc_commit(uint64_t* b) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          su32(b))
      : "memory");
}
// K-major SWIZZLE_128B descriptor: 128 B rows, 8-row atoms 1024 B apart
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = __uint_as_float(r[k]);
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = __uint_as_float(r[k]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]));
}
// shared-window stores by 32-bit shared address (the 1024-aligned dynamic
// base is computed through an integer, which would otherwise make every
// store a generic 64-bit ST)
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void sts_v2(uint32_t a, float x, float y) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(x), "f"(y) : "memory");
}
__device__ __forceinline__ void sts_v4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
// byte offset of element (row r, k) in a K-major SW128 block of 32-bit data
__device__ __forceinline__ uint32_t sw128_off(int r, int k) {
  return (uint32_t)((r >> 3) * 1024 + (r & 7) * 128 + ((((k >> 2) ^ r) & 7) << 4) + (k & 3) * 4);
}

}  // namespace

struct BwdTcArgs {
  const uint64_t* pairs;
  const int* tile_start;
  const int* wstop;
  const float4* rrec;
  const float* coef;   // [n, Cp]
  const float* dL;     // [B, h, w, C]
  const float* T_final;
  const int* last;
  float* gcoef;        // [n, Cp]
  float* ggeo;         // [n, 8]
  float* dgc;          // deterministic partials [pairs][2][Cp]
  float* dgg;          // [pairs][2][1][6]
  const int* counters;
  int Cp, C, Kp;
  int w, h, ntx;
  int det;
  int lpt;  // longest-first CTA order
  // compacted walk (non-deterministic frames): pass A's chunk entries of the
  // half tile and their used bits
  const uint32_t* ch_used;
  const uint32_t* ch_idx;
  const int* ch_pos;
  const int* ch_n;
  int compact;
};

__global__ void __launch_bounds__(320, 1) k_raster_bwd_tc(BwdTcArgs A) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ TcShared S;
  if (A.counters[GSPARC_CNT_OVERFLOW]) return;
  int cta = blockIdx.x;
  if (A.lpt) {
    // longest-first: CTAs are dispatched in blockIdx order, so block k takes
    // the half tile with the k-th most entries to visit (ties by index);
    // one CTA per SM, and the heavy half tiles no longer end the grid
    __shared__ int s_item;
    int* s_nv = (int*)sm;  // [gridDim.x], before any staging
    const int nitem = gridDim.x;
    for (int i = threadIdx.x; i < nitem; i += blockDim.x) {
      const int t = i >> 1, hf = i & 1;
      int nv = 0;
      if ((t / A.ntx) * TILE + hf * 8 < A.h) {
#pragma unroll
        for (int q = 0; q < 4; ++q) nv = max(nv, A.wstop[t * 8 + hf * 4 + q]);
      }
      s_nv[i] = nv;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nitem; i += blockDim.x) {
      const int v = s_nv[i];
      int rank = 0;
      for (int j = 0; j < nitem; ++j) {
        const int u = s_nv[j];
        rank += (u > v) || (u == v && j < i);
      }
      if (rank == (int)blockIdx.x) s_item = i;
    }
    __syncthreads();
    cta = s_item;
  }
  const int tile = cta >> 1, half = cta & 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tx_ = tile % A.ntx, ty = tile / A.ntx;
  const int x0 = tx_ * TILE, y0 = ty * TILE + half * 8;
  if (y0 >= A.h) return;
  const int start = A.tile_start[tile], tile_end = A.tile_start[tile + 1];
  int nvisit = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) nvisit = max(nvisit, A.wstop[tile * 8 + half * 4 + q]);
  if (nvisit == 0) return;
  // Compacted walk (non-deterministic frames): only the entries that some
  // pixel of this half tile included (pass A's ch_used bits, list order) can
  // have a nonzero term -- an entry no pixel included has alpha under the cut
  // or lies past every pixel's last included entry, so its scan terms, its
  // weights (GEMM-2 column) and its gradients are all zero, and T / suffix
  // pass it unchanged (rcp(1 - 0) = 1, fma(0, u, s) = s): skipping it is
  // exact.  Batches are then 32 used entries; the deterministic mode keeps
  // the list walk (its partial slots are indexed by list position).
  int nwork = nvisit, cnch = 0;
  int64_t cslot0 = 0;
  bool cmp = false;
  if (A.compact) {
    cnch = A.ch_n[cta];
    if (cnch <= K5_CCAP) {
      cslot0 = 2 * (((int64_t)start + 31 * (int64_t)tile) >> 5) +
               (int64_t)half * ((tile_end - start + 31) >> 5);
      if (warp == 0) {
        int run = 0;
        for (int c0 = 0; c0 < cnch; c0 += 32) {
          const int c = c0 + lane;
          const int v = c < cnch ? __popc(__ldcg(A.ch_used + cslot0 + c)) : 0;
          int inc = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
          }
          if (c < cnch) S.cs[c] = run + inc - v;
          run += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) S.cs[cnch] = run;
      }
      __syncthreads();
      nwork = S.cs[cnch];
      cmp = true;
      if (nwork == 0) return;
    }
  }
  // e-th used entry of the half tile (list order): source index, and its
  // list position from the tile's start in rel
  auto centry = [&](int e, int& rel) -> int {
    int lo = 0, hi = cnch;  // cs[lo] <= e < cs[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (S.cs[mid] <= e) lo = mid;
      else hi = mid;
    }
    uint32_t m = __ldcg(A.ch_used + cslot0 + lo);
    int r = e - S.cs[lo], k = 0;  // position of the r-th set bit of m
#pragma unroll
    for (int wdt = 16; wdt >= 1; wdt >>= 1) {
      const int cnt = __popc(m & ((1u << wdt) - 1u));
      if (r >= cnt) {
        r -= cnt;
        k += wdt;
        m >>= wdt;
      }
    }
    const int64_t o = (cslot0 + lo) * 32 + k;
    rel = __ldcg(A.ch_pos + o);
    return (int)__ldcg(A.ch_idx + o);
  };
  const int nbatch = (nwork + TC_NB - 1) / TC_NB;
  const int Cp = A.Cp;
  const uint32_t sbase = su32(sm);

  if (threadIdx.x == 0) {
    for (int k = 0; k < TC_NS; ++k) {
      bar_init(&S.coef_full[k], 1);
      bar_init(&S.stage_empty[k], 1 + 4);  // GEMM-1 commit + 4 scan warps
    }
    for (int k = 0; k < 2; ++k) {
      bar_init(&S.d1_full[k], 1);
      bar_init(&S.d1_empty[k], 4);
      bar_init(&S.w_full[k], 4);
      bar_init(&S.w_empty[k], 1);
      bar_init(&S.d2_full[k], 1);
      bar_init(&S.d2_empty[k], 4);
      bar_init(&S.red_full[k], 4);
      bar_init(&S.red_empty[k], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(&S.tmem)),
                 "r"(TC_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  // the pad block after U^T's last K block (rows 64..127 of GEMM 2's A there)
  for (int t = threadIdx.x; t < 2 * UT_KB / 16; t += blockDim.x) {
    const int plane = t / (UT_KB / 16), o = t % (UT_KB / 16);
    sts_v4(sbase + OFF_UT + plane * UT_PLANE + 4 * UT_KB + o * 16, make_float4(0.f, 0.f, 0.f, 0.f));
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = S.tmem;

  // per pixel state (scan warps)
  const int px = x0 + (lane & 15), py = y0 + 2 * warp + (lane >> 4);
  const bool inside = warp < 4 && px < A.w && py < A.h;
  float T = 1.f, suffix = 0.f;
  int lastp = 0;
  if (warp < 4) {
    // u = dL/dimg of this pixel over all Cp = B*C columns -> TMEM (A of
    // GEMM 1, lane = pixel) and U^T (A of GEMM 2, row = channel)
    float u[TC_KMAX];
    {
      // column c = b * C + ch of transmitter b: walk (b, ch) without divisions
      const float* src = A.dL + ((int64_t)py * A.w + px) * A.C;
      const int64_t tx_stride = (int64_t)A.h * A.w * A.C;
      int ch = 0;
#pragma unroll
      for (int c = 0; c < TC_KMAX; ++c) {
        u[c] = (inside && c < Cp) ? __ldg(src + ch) : 0.f;
        if (++ch == A.C) {
          ch = 0;
          src += tx_stride;
        }
      }
    }
    if (inside) {
      T = A.T_final[py * A.w + px];
      lastp = A.last[py * A.w + px];
    }
    const uint32_t trow = tmem + ((uint32_t)(32 * warp) << 16);
#pragma unroll
    for (int c0 = 0; c0 < TC_KMAX; c0 += 16) {
      uint32_t hi[16], lo[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const float x = u[c0 + k], xh = tf32_hi(x);
        hi[k] = __float_as_uint(xh);
        lo[k] = __float_as_uint(x - xh);
      }
      tmem_st16(trow + COL_UHI + c0, hi);
      tmem_st16(trow + COL_ULO + c0, lo);
    }
    // U^T: K block = warp (32 pixels), row = channel, k = lane
    const uint32_t uth = sbase + OFF_UT + warp * UT_KB, utl = uth + UT_PLANE;
#pragma unroll
    for (int c = 0; c < TC_KMAX; ++c) {
      const float x = u[c], xh = tf32_hi(x);
      const uint32_t o = sw128_off(c, lane);
      sts_f32(uth + o, xh);
      sts_f32(utl + o, x - xh);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  auto batch_range = [&](int b, int& b0, int& nb) {
    const int bend = nwork - TC_NB * b;
    b0 = bend > TC_NB ? bend - TC_NB : 0;
    nb = bend - b0;
  };

  if (warp == 6) {
    // ------------------------------------------------------------ loader
    for (int b = 0; b < nbatch; ++b) {
      const int s = b % TC_NS;
      int b0, nb;
      batch_range(b, b0, nb);
      bar_wait_sleep(&S.stage_empty[s], ((b / TC_NS) & 1) ^ 1);
      int idx = 0;
      bool dup = false;
      if (lane < nb) {
        int rel = b0 + lane;  // list position from the tile's start
        if (cmp) idx = centry(b0 + lane, rel);
        const int pos = start + rel;
        if (!cmp) idx = (int)(uint32_t)A.pairs[pos];
        dup = pos + 1 < tile_end && (int)(uint32_t)A.pairs[pos + 1] == idx;
        const float4 f0 = __ldg(A.rrec + 2 * (size_t)idx);
        const float4 f1 = __ldg(A.rrec + 2 * (size_t)idx + 1);
        S.fr[s][lane][0] = f0;
        // (xr, yr) are not used by the scan: z carries the list position
        S.fr[s][lane][1] = make_float4(f1.x, f1.y, __int_as_float(rel), f1.w);
        // conic recovered from the pre-scaled exponent coefficients (K2) and
        // sigma = 2^(log2 sigma), once per entry instead of once per pixel
        const float k2 = (float)(-2.0 / LOG2E), k1 = (float)(-1.0 / LOG2E);
        S.fr[s][lane][2] = make_float4(f0.z * k2, f0.w * k1, f1.x * k2, exp2f(f1.y));
      } else {
        // finite filler: the scan evaluates every slot branch-free
        S.fr[s][lane][0] = make_float4(0.f, 0.f, 0.f, 0.f);
        S.fr[s][lane][1] = make_float4(0.f, 0.f, -1.f, -1.f);
        S.fr[s][lane][2] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      S.idx[s][lane] = lane < nb ? (idx | (dup ? (int)0x80000000 : 0)) : -1;
      // coef rows: lane covers channels 2*lane, 2*lane+1 of every row
      float2 cv[TC_NB];
      const bool cin = 2 * lane < Cp;
#pragma unroll
      for (int r = 0; r < TC_NB; ++r) {
        const int ri = __shfl_sync(0xffffffffu, idx, r);
        cv[r] = (r < nb && cin) ? *(const float2*)(A.coef + (int64_t)ri * Cp + 2 * lane)
                                : make_float2(0.f, 0.f);
      }
      const uint32_t ch = sbase + OFF_COEF + s * COEF_STAGE;
      const int kb = lane >> 4, k = (2 * lane) & 31;
#pragma unroll
      for (int r = 0; r < TC_NB; ++r) {
        const uint32_t o = kb * 4096 + sw128_off(r, k);
        const float h0 = tf32_hi(cv[r].x), h1 = tf32_hi(cv[r].y);
        sts_v2(ch + o, h0, h1);
        sts_v2(ch + COEF_PLANE + o, cv[r].x - h0, cv[r].y - h1);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&S.coef_full[s]);
    }
  } else if (warp == 7) {
    // ------------------------------------------------------------ MMA issue
    if (lane == 0) {
      // D f32, A/B tf32, both K-major, N = 32, M = 128
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_NB >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      const int ksteps1 = A.Kp >> 3;
      // (the MMA thread waits without sleeping: try_wait suspends it in
      // hardware until the phase completes, and a late wake-up here delays
      // both GEMMs)
      auto gemm1 = [&](int b) {
        const int q = b % TC_NS, s = b & 1;
        bar_wait(&S.coef_full[q], (b / TC_NS) & 1);
        bar_wait(&S.d1_empty[s], ((b >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + COL_D1 + 32 * s;
        const uint32_t bhi = sbase + OFF_COEF + q * COEF_STAGE, blo = bhi + COEF_PLANE;
#pragma unroll 1
        for (int ks = 0; ks < ksteps1; ++ks) {
          const uint32_t ob = (ks >> 2) * 4096 + (ks & 3) * 32;
          mma_ts(d, tmem + COL_UHI + 8 * ks, desc_sw128(bhi + ob), idesc, ks > 0);
          mma_ts(d, tmem + COL_UHI + 8 * ks, desc_sw128(blo + ob), idesc, 1);
          mma_ts(d, tmem + COL_ULO + 8 * ks, desc_sw128(bhi + ob), idesc, 1);
        }
        tc_commit(&S.d1_full[s]);
        tc_commit(&S.stage_empty[q]);
      };
      auto gemm2 = [&](int b) {
        const int g = b & 1;
        bar_wait(&S.d2_empty[g], ((b >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + COL_D2 + 32 * g;
        const uint32_t ahi = sbase + OFF_UT, alo = ahi + UT_PLANE;
        const uint32_t bhi = sbase + OFF_W + g * W_STAGE, blo = bhi + W_PLANE;
#pragma unroll 1
        for (int ks = 0; ks < 16; ++ks) {
          const uint32_t oa = (ks >> 2) * UT_KB + (ks & 3) * 32;
          const uint32_t ob = (ks >> 2) * 4096 + (ks & 3) * 32;
          mma_ss(d, desc_sw128(ahi + oa), desc_sw128(bhi + ob), idesc, ks > 0);
          mma_ss(d, desc_sw128(ahi + oa), desc_sw128(blo + ob), idesc, 1);
          mma_ss(d, desc_sw128(alo + oa), desc_sw128(bhi + ob), idesc, 1);
        }
        tc_commit(&S.d2_full[g]);
        tc_commit(&S.w_empty[g]);
      };
      // GEMM 1 runs two batches ahead of the scan: when scan b ends, GEMM 1
      // of b + 2 (into the D1 buffer scan b just released) goes first, then
      // GEMM 2 of b
      gemm1(0);
      if (nbatch > 1) gemm1(1);
      for (int b = 0; b < nbatch; ++b) {
        bar_wait(&S.w_full[b & 1], (b >> 1) & 1);
        if (b + 2 < nbatch) gemm1(b + 2);
        gemm2(b);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ GEMM-2 epilogue
    // warps 4, 5, 8, 9: TMEM lane quadrant qe = warp % 4 (channels 32 qe ..),
    // entry half eh (entries 16 eh .. 16 eh + 15 of each batch)
    const int qe = warp & 3, eh = warp >= 8 ? 1 : 0, ew = 2 * eh + qe;
    const int c = 32 * qe + lane;  // channel = TMEM lane
    for (int b = 0; b < nbatch; ++b) {
      const int g = b & 1;
      int b0, nb;
      batch_range(b, b0, nb);
      // the batch's entries straight from the (L2-resident) list, loaded
      // before any wait
      int myidx = -1;
      if (lane < nb) {
        int rel = b0 + lane;
        if (cmp) centry(b0 + lane, rel);
        const int pos = start + rel;
        myidx = (int)(uint32_t)A.pairs[pos];
        if (pos + 1 < tile_end && (int)(uint32_t)A.pairs[pos + 1] == myidx)
          myidx |= (int)0x80000000;  // first copy of a seam duplicate
      }
      // (1) the geometric gradients: the four scan warps' partials summed in
      // warp order (fixed), off the scan warps' critical path
      bar_wait_sleep(&S.red_full[g], (b >> 1) & 1);
      {
        const float (*red)[4][6] = S.red[g];
        for (int e = 32 * ew + lane; e < TC_NB * 6; e += 128) {
          const int j = e / 6, f = e - j * 6;
          const int sj = __shfl_sync(0xffffffffu, myidx, j);
          if (j < nb) {
            const float x = ((red[j][0][f] + red[j][1][f]) + red[j][2][f]) + red[j][3][f];
            if (A.det) {
              const int64_t pos = start + b0 + j;
              A.dgg[(pos * 2 + half) * 6 + f] = sj < 0 ? 0.f : x;
            } else if (x != 0.f && sj >= 0) {
              atomicAdd(A.ggeo + (int64_t)sj * 8 + f, x);
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) bar_arrive(&S.red_empty[g]);
      // (2) dL/dcoef rows from GEMM 2
      bar_wait_sleep(&S.d2_full[g], (b >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(32 * qe) << 16) + COL_D2 + 32 * g + 16 * eh, v);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&S.d2_empty[g]);
      {
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int j = 16 * eh + jj;
          const int sj = __shfl_sync(0xffffffffu, myidx, j);
          if (j < nb && c < Cp) {
            const float x = sj < 0 ? 0.f : v[jj];
            if (A.det) {
              const int64_t pos = start + b0 + j;
              A.dgc[(pos * 2 + half) * Cp + c] = x;
            } else if (x != 0.f) {
              atomicAdd(A.gcoef + (int64_t)(sj & 0x7fffffff) * Cp + c, x);
            }
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ scan (warps 0-3)
    const float pcx = (float)px + 0.5f, pcy = (float)py + 0.5f;
    const float wR = (float)A.w, inv_w = 1.0f / wR;
    for (int b = 0; b < nbatch; ++b) {
      const int s = b & 1;
      int b0, nb;
      batch_range(b, b0, nb);
      bar_wait(&S.d1_full[s], (b >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d1row = tmem + ((uint32_t)(32 * warp) << 16) + COL_D1 + 32 * s;
      const int q = b % TC_NS;
      bar_wait(&S.coef_full[q], (b / TC_NS) & 1);   // records of this batch
      bar_wait(&S.w_empty[s], ((b >> 1) & 1) ^ 1);
      bar_wait(&S.red_empty[s], ((b >> 1) & 1) ^ 1);
      const uint32_t wh = sbase + OFF_W + s * W_STAGE, wl = wh + W_PLANE;
      const uint32_t wo = warp * 4096;  // K block of this warp's pixels
      float (*red)[4][6] = S.red[s];
#pragma unroll
      // groups of 8 entries, back to front, branch-free (invalid and
      // non-contributing entries select zeros): (1) the 8 alphas from the
      // records (independent; all shared loads of the group issue before any
      // shared store, so nothing serialises on possible aliasing), (2) the
      // serial T / suffix recurrence, (3) the gradients and 8 independent
      // warp reduce-scatters, (4) the W and partial-sum stores
      // (a rolled loop over the 4 groups: the unrolled batch is ~180 KB of
      // SASS and ran instruction-fetch bound)
#pragma unroll 1
      for (int g8 = TC_NB / 8 - 1; g8 >= 0; --g8) {
        // every step below runs across the group's 8 entries before the next
        // (the source order is the issue order ptxas keeps: 8 independent
        // chains in flight instead of one)
        float ucg[8];
        tmem_ld8(d1row + 8 * g8, ucg);
        float dx[8], dy[8], e1[8], e2[8];
        int rl[8];  // list positions (the loader's record z)
#pragma unroll
        for (int t = 7; t >= 0; --t) {
          const int j = 8 * g8 + t;
          const float4 f0 = S.fr[q][j][0], f1 = S.fr[q][j][1];
          const float dxr = pcx - f0.x;
          dx[t] = fmaf(-wR, rintf(dxr * inv_w), dxr);
          dy[t] = pcy - f0.y;
          const float tt = fmaf(f0.w, dy[t], f0.z * dx[t]);
          const float qcy = f1.x * dy[t];
          e1[t] = fmaf(dx[t], tt, fmaf(qcy, dy[t], f1.y));  // q' + log2 sigma
          e2[t] = fmaf(dx[t], tt, qcy * dy[t]);             // q'
          rl[t] = __float_as_int(f1.z);
        }
        float al[8], rom[8], ga[8];
        bool gon[8];
#pragma unroll
        for (int t = 7; t >= 0; --t) {
          const int j = 8 * g8 + t;
          const float raw = ex2_approx(e1[t]);
          ga[t] = ex2_approx(e2[t]);
          // fast_alpha_full's alpha: min(raw, 0.99), zero below 1/255
          const float a = fminf(raw, ALPHA_MAX_F);
          const bool on = (j < nb) & (rl[t] < lastp) & (a >= ALPHA_MIN_F);
          al[t] = on ? a : 0.f;
          gon[t] = on & (raw < ALPHA_MAX_F);
        }
#pragma unroll
        // 1 / (1 - alpha): MUFU rcp (<= 1 ulp, exact at 1) -- the IEEE __frcp_rn
        // adds a Newton step and a slow-path branch per entry
        for (int t = 7; t >= 0; --t) {
          float r;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.f - al[t]));
          rom[t] = r;
        }
        float wgt[8], dAg[8];
#pragma unroll
        for (int t = 7; t >= 0; --t) {
          const float Tb = T * rom[t];
          wgt[t] = Tb * al[t];
          const float dA = Tb * ucg[t] - suffix * rom[t];
          suffix = fmaf(wgt[t], ucg[t], suffix);
          T = Tb;
          dAg[t] = gon[t] ? dA * ga[t] : 0.f;
        }
        // gradients (cq = {ca, cb, cc, sigma} from the loader), then the 8
        // reduce-scatters level by level: lane 4f ends with field f
        float v[8][4];
#pragma unroll
        for (int t = 7; t >= 0; --t) {
          const int j = 8 * g8 + t;
          const float4 cq = S.fr[q][j][2];
          const float dq = -0.5f * dAg[t] * cq.w;
          float x[8];
          x[0] = dq * dx[t] * dx[t];
          x[1] = dq * dx[t] * dy[t];
          x[2] = dq * dy[t] * dy[t];
          x[3] = -(dq * 2.f * (cq.x * dx[t] + cq.y * dy[t]));
          x[4] = -(dq * 2.f * (cq.y * dx[t] + cq.z * dy[t]));
          x[5] = dAg[t];
          x[6] = 0.f;
          x[7] = 0.f;
          const bool hi = lane & 16;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float send = hi ? x[k] : x[k + 4];
            const float keep = hi ? x[k + 4] : x[k];
            v[t][k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
          }
        }
#pragma unroll
        for (int t = 7; t >= 0; --t) {
          const bool hi = lane & 8;
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const float send = hi ? v[t][k] : v[t][k + 2];
            const float keep = hi ? v[t][k + 2] : v[t][k];
            v[t][k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
          }
        }
#pragma unroll
        for (int t = 7; t >= 0; --t) {
          const bool hi = lane & 4;
          const float send = hi ? v[t][0] : v[t][1];
          const float keep = hi ? v[t][1] : v[t][0];
          v[t][0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
#pragma unroll
        for (int t = 7; t >= 0; --t) v[t][0] += __shfl_xor_sync(0xffffffffu, v[t][0], 2);
#pragma unroll
        for (int t = 7; t >= 0; --t) v[t][0] += __shfl_xor_sync(0xffffffffu, v[t][0], 1);
        const int fld = lane >> 2;
#pragma unroll
        for (int t = 7; t >= 0; --t) {
          const int j = 8 * g8 + t;
          // W[j][pixel] (B of GEMM 2: row = entry, k = pixel of this warp's block)
          const uint32_t o = wo + sw128_off(j, lane);
          const float hw = tf32_hi(wgt[t]);
          sts_f32(wh + o, hw);
          sts_f32(wl + o, wgt[t] - hw);
          if ((lane & 3) == 0 && fld < 6) red[j][warp][fld] = v[t][0];
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&S.w_full[s]);
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&S.d1_empty[s]);
      __syncwarp();
      if (lane == 0) {
        bar_arrive(&S.red_full[s]);
        bar_arrive(&S.stage_empty[q]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TC_TMEM_COLS));
  }
}

bool raster_bwd_tc_supported(const gsparc_frame_layout& L, int64_t Cp) {
  // the loader reads coef rows as float2 pairs: even row lengths only
  return L.dtype == GSPARC_F32 && Cp >= 16 && Cp <= TC_KMAX && (Cp & 1) == 0;
}

int launch_raster_bwd_tc(const gsparc_frame_layout& L, char* frame, int n_tx, int C,
                         const void* dL, bool det, cudaStream_t st) {
  BwdTcArgs A;
  A.pairs = (const uint64_t*)(frame + L.off_pairs);
  A.tile_start = (const int*)(frame + L.off_tile_start);
  A.wstop = (const int*)(frame + L.off_wstop);
  A.rrec = (const float4*)(frame + L.off_rrec);
  A.coef = (const float*)(frame + L.off_coef);
  A.dL = (const float*)dL;
  A.T_final = (const float*)(frame + L.off_T);
  A.last = (const int*)(frame + L.off_last);
  A.gcoef = (float*)(frame + L.off_gcoef);
  A.ggeo = (float*)(frame + L.off_ggeo);
  A.dgc = (float*)(frame + L.off_det_gcoef);
  A.dgg = (float*)(frame + L.off_det_ggeo);
  A.counters = (const int*)(frame + L.off_counters);
  A.Cp = n_tx * C;
  A.C = C;
  A.Kp = (A.Cp + 7) & ~7;
  A.w = L.width;
  A.h = L.height;
  A.ntx = L.ntx;
  static const int lpt =
      experiment_env("GSPARC_K5_LPT") ? atoi(experiment_env("GSPARC_K5_LPT")) : 1;
  A.lpt = lpt;
  A.det = det ? 1 : 0;
  A.ch_used = (const uint32_t*)(frame + L.off_ch_used);
  A.ch_idx = (const uint32_t*)(frame + L.off_ch_idx);
  A.ch_pos = (const int*)(frame + L.off_ch_pos);
  A.ch_n = (const int*)(frame + L.off_ch_n);
  static const int cmp_env =
      experiment_env("GSPARC_K5_COMPACT") ? atoi(experiment_env("GSPARC_K5_COMPACT")) : 1;
  A.compact = !det && cmp_env && L.off_ch_pos != 0;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_raster_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TC);
    attr_set = true;
  }
  k_raster_bwd_tc<<<2 * L.ntiles, 320, SMEM_TC, st>>>(A);
  return check_launch("k_raster_bwd_tc");
}

}  // namespace gs
