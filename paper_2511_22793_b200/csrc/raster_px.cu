// K4 (f32 frames): front-to-back compositing with one pixel per lane.
// Replaces do_tile / _tile_alphas (rasterizer.py:169-231).
//
// A CTA owns half a 16x16 tile (16 x 8 = 128 pixels, 4 warps of 16 x 2).
// The tile's depth-ordered list (K3) is consumed in chunks of 32 entries
// that survive a CTA-level cull: an entry whose alpha >= 1/255 ellipse
// (rrec.xr/yr, conservative) misses every pixel centre of the CTA has
// alpha = 0 for all of them, so it multiplies T by exactly 1 and is never
// included -- skipping it is exact.  Chunks are dense, so the 32 alphas of a
// chunk are evaluated branch-free with full ILP and a sequential
// T *= (1 - alpha) per lane (numpy's cumprod order, rasterizer.py:209-212).
//
// Pass A (k_pxa): a producer warp scans + culls the list into a shared ring
//   of chunks (mbarrier full/empty protocol); 4 consumer warps walk them
//   until every pixel has T < t_eps, writing T_final / count / last, the
//   per-warp visited prefix (wstop, for K5), the live-Gaussian list, and for
//   pass B: the chunk's source indices (ch_idx) and every pixel's T at the
//   start of every chunk (ch_T).  With SC in 1..4 the consumers also
//   accumulate the image on CUDA cores (fused small-channel path).
// Pass B (k_pxb): the T checkpoints make chunks independent, so two groups
//   of 4 weight warps take alternate chunks; each writes its 128 x 32 weight
//   tile straight into TMEM (tcgen05.st, lane = pixel), two stager warps
//   write coef^T for the chunk to shared memory (K-major SWIZZLE_128B), and
//   one thread issues
//       img[128 px, NP] += W[128, 32] . coef[32, NP]
//   as tcgen05.mma kind::tf32 with A from TMEM, 3xTF32 split
//   (Wh.ch + Wh.cl + Wl.ch) for fp32 accuracy, accumulator in TMEM.
#include <cuda.h>
#include <stdlib.h>

#include <type_traits>
#include <string.h>  // CUtensorMap (encoded through the runtime's driver entry point)

#include "common.cuh"
#include "kernels.cuh"

namespace gs {

constexpr int PX_K = 32;    // entries per chunk
constexpr int PX_RING = 4;  // pass-A ring depth (chunks)

struct PxArgs {
  const uint64_t* pairs;
  const int* tile_start;
  const float4* rrec;  // [n][2]
  const float* coef;   // [n][Cp]
  uint32_t* ch_used;   // [slots] CTA-level included-entry mask per chunk
  long long* dbg;      // optional per-CTA timing counters (experiments)
  uint32_t* ch_idx;    // [slots][32]
  float4* ch_rec;      // [slots][32][2]
  float* ch_T;         // [slots][128]
  int* ch_n;           // [2 * ntiles]
  int* wstop;          // [ntiles * 8]
  float* T_out;
  int* count_out;
  int* last_out;
  int* live;
  int* live_list;
  int* counters;
  float* img;
  float4* pxw;    // [2*ntiles][wmax][8][128] weights of the first wmax chunks
  uint32_t* ch_wm;  // [slots][4] per-warp included-entry mask
  const int* ready;  // pass A: K3's per-tile flags (null: the sort grid has completed)
  int pdl_b;         // pass B launched as a dependent (upstream reads after the wait)
  int mix_b;         // pass B: interleave top/bottom tiles in launch order
  int tile_major_b;  // pass B, several channel chunks: a half tile's chunk CTAs adjacent
  int wmax;
  int64_t Cp, n;
  int C, w, h, ntx, ntiles;
  float t_eps, wf, inv_w;
  int* ch_pos;  // [slots][32] list position of the entry (from the tile's start); null: not a backward frame
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// Same wait with a sleeping back-off: many warps polling mbarriers flood
// the shared-memory (MIO) pipe that the producers' copies also need.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(64);
  }
}

// First chunk slot of CTA (tile, half): see capi.cu gsparc_plan_frame.
__device__ __forceinline__ int64_t chunk_slot0(const int* tile_start, int tile, int half) {
  const int64_t s = tile_start[tile];
  const int64_t len = tile_start[tile + 1] - s;
  return 2 * ((s + 31 * (int64_t)tile) >> 5) + half * ((len + 31) >> 5);
}

// Pixel row (0..7) of a half tile held by lane group hi (lane >> 4) of the
// 32-pixel warp w: rows {w, 7 - w}, so every warp has one row of each end of
// the half tile (per-pixel list lengths change monotonically across a tile
// near the poles; rows {2w, 2w + 1} left one warp with both heavy rows).
// Pass A, pass B and pass B's epilogue share it (stored weights, T
// checkpoints and TMEM lanes are indexed by warp * 32 + lane).
__device__ __forceinline__ int half_row(int w, int hi) { return hi ? 7 - w : w; }

struct CtaGeom {
  int tile, half, x0, y0;
  float xc, xhalf, ylo, yhi;
  bool any;
};

__device__ __forceinline__ CtaGeom cta_geom(const PxArgs& A, int cta) {
  CtaGeom g;
  g.tile = cta >> 1;
  g.half = cta & 1;
  g.x0 = (g.tile % A.ntx) * TILE;
  g.y0 = (g.tile / A.ntx) * TILE + g.half * 8;
  const float xlo = g.x0 + 0.5f, xhi = (float)min(g.x0 + TILE, A.w) - 0.5f;
  g.ylo = g.y0 + 0.5f;
  g.yhi = (float)min(g.y0 + 8, A.h) - 0.5f;
  g.xc = 0.5f * (xlo + xhi);
  g.xhalf = 0.5f * (xhi - xlo);
  g.any = g.y0 < A.h;
  return g;
}

// Could the entry reach alpha >= 1/255 at any pixel centre of the CTA?
__device__ __forceinline__ bool cull_keep(float4 r0, float4 r1, const CtaGeom& g, float w,
                                          float inv_w) {
  float d = r0.x - g.xc;
  d = fmaf(-w, rintf(d * inv_w), d);
  const float dx = fabsf(d) - g.xhalf;
  const float dy = fmaxf(g.ylo - r0.y, r0.y - g.yhi);
  return r1.z >= 0.f && dx <= r1.z && dy <= r1.w;
}

// Tighter, still conservative cull: the largest exponent
//   q'(dx, dy) + log2(op),  q' = qa dx^2 + qb dx dy + qc dy^2  (concave)
// over the continuous rectangle spanned by the CTA's pixel centres is below
// log2(1/255) by a margin, so alpha < 1/255 at every pixel centre and the
// entry is never included (skipping it is exact, as for cull_keep).  The
// ellipse's bounding box (cull_keep) admits many such entries near the poles,
// where footprints are wide and sheared.  The maximum is 0 when the rectangle
// holds the centre, else on an edge (a 1-D concave quadratic, clamped).  The
// margin covers the f32 rounding of this and of the per-pixel evaluation;
// NaN, degenerate conics and azimuth wraps that differ across the CTA keep
// the entry.
__device__ __forceinline__ bool tight_keep(float4 r0, float4 r1, float xlo, float xhi, float ylo,
                                           float yhi, float w, float inv_w) {
  const float klo = rintf((xlo - r0.x) * inv_w), khi = rintf((xhi - r0.x) * inv_w);
  const float qa = r0.z, qb = r0.w, qc = r1.x;
  if (klo != khi || !(qa < 0.f && qc < 0.f)) return true;
  const float x0 = (xlo - r0.x) - w * klo, x1 = (xhi - r0.x) - w * klo;
  const float y0 = ylo - r0.y, y1 = yhi - r0.y;
  // The maximum lies on an edge facing the centre (its supporting line
  // separates the centre from the rectangle; a linear map preserves that),
  // so at most one x edge and one y edge are candidates.  The clamped
  // 1-D argmax uses fast reciprocals: a point near the argmax undershoots
  // the edge maximum only by |q| delta^2, far inside the margin.
  const bool ox = x0 > 0.f || x1 < 0.f, oy = y0 > 0.f || y1 < 0.f;
  float m = 0.f;
  if (ox || oy) {
    const float xe = x0 > 0.f ? x0 : x1, ye = y0 > 0.f ? y0 : y1;
    float rqa, rqc;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rqa) : "f"(qa));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rqc) : "f"(qc));
    const float ys = fminf(fmaxf(-0.5f * qb * xe * rqc, y0), y1);
    const float xs = fminf(fmaxf(-0.5f * qb * ye * rqa, x0), x1);
    const float fx = fmaf(xe, fmaf(qa, xe, qb * ys), qc * ys * ys);
    const float fy = fmaf(xs, fmaf(qa, xs, qb * ye), qc * ye * ye);
    m = fmaxf(ox ? fx : -INFINITY, oy ? fy : -INFINITY);
  }
  // margin: 0.05 plus 2e-5 of the largest term magnitude over the rectangle
  // (f32 rounding of the terms, and of dx: 1 ulp x |dq'/ddx| <= 2 |qa| X ulp)
  const float X = fmaxf(fabsf(x0), fabsf(x1)), Y = fmaxf(fabsf(y0), fabsf(y1));
  const float mag = fmaf(-qa * X, X, fmaf(fabsf(qb) * X, Y, -qc * Y * Y));
  const float v = m + r1.y;  // log2 of the largest raw alpha
  return !(v < -7.9943534f - fmaf(2e-5f, mag, 0.05f));
}

// ------------------------------------------------------------------ pass A
template <int SC>
__global__ void __launch_bounds__(160) k_pxa(PxArgs A) {
  constexpr int SCW = SC ? 4 : 1;
  __shared__ __align__(16) float4 s_ring[PX_RING][PX_K][2];
  __shared__ __align__(16) float s_cf[PX_RING][PX_K][SCW];
  __shared__ int s_hdr[PX_RING];
  __shared__ int s_wrap[PX_RING];  // chunk holds an entry whose wrap varies across the CTA
  __shared__ __align__(8) uint64_t s_full[PX_RING], s_empty[PX_RING];
  __shared__ int s_ndone, s_nch, s_stop[4];

  const long long t_startA = clock64();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int cta = blockIdx.x;  // (tile, half) = (cta >> 1, cta & 1)
  if (A.ready) {
    // launched while K3 runs: claim the next (tile, half) in the order the
    // sorts finished and wait until it is published.  K3 publishes every
    // tile, also on a pair-buffer overflow (then without a list), so the
    // overflow flag is read only after the acquire, which orders it after
    // K2's grid.  A wait that never ends (a frame whose sort did not run)
    // is bounded: the CTA flags an error and exits without touching the tile.
    __shared__ int s_cta;
    if (threadIdx.x == 0) {
      const int h = atomicAdd(A.counters + GSPARC_CNT_CLAIMED, 1) % (2 * A.ntiles);
      long long spins = 0;
      int v;
      while (!(v = flag_acquire(A.ready + (h >> 1)))) {
        __nanosleep(64);
        if (++spins > (1ll << 24)) break;
      }
      if (!v) {
        atomicExch(A.counters + GSPARC_CNT_OVERFLOW, 2);
        s_cta = -2;
      } else {
        s_cta = flag_acquire(A.counters + GSPARC_CNT_OVERFLOW) ? -1 : 2 * (v - 1) + (h & 1);
      }
    }
    __syncthreads();
    cta = s_cta;
    if (cta == -2) return;  // the sort grid never published: do not wait on it
    if (cta < 0) {
      pdl_wait();
      return;
    }
  } else if (A.counters[GSPARC_CNT_OVERFLOW]) {
    return;
  }
  if (A.dbg && threadIdx.x == 0) {
    A.dbg[cta * 16 + 13] = clock64() - t_startA;  // tile claimed
    A.dbg[cta * 16 + 14] = gtimer();
  }
  pdl_trigger();  // the lazy MLP (K1) may start and consume the live list as it grows
  const CtaGeom g = cta_geom(A, cta);
  // the tile's bounds and list were written by a grid that may still be
  // running: read them through L2
  const int start = __ldcg(A.tile_start + g.tile);
  const int len = __ldcg(A.tile_start + g.tile + 1) - start;
  const int64_t slot0 = 2 * ((start + 31 * (int64_t)g.tile) >> 5) + g.half * ((len + 31) >> 5);
  if (threadIdx.x == 0) {
    for (int s = 0; s < PX_RING; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_ndone = 0;
    s_nch = 0;
  }
  if (threadIdx.x < 4) s_stop[threadIdx.x] = 0;
  __syncthreads();

  if (warp == 4) {
    // ---------------- producer: scan, cull, compact into the ring
    const unsigned lt = (1u << lane) - 1u;
    int c = 0, fill = 0, acquired = 0;
    int wrap_c = 0, wrap_n = 0;  // wrap flags of chunks c and c + 1
    // first and last pixel-centre column of the CTA (pass A's pcx values)
    const float pxlo = g.x0 + 0.5f, pxhi = (float)min(g.x0 + TILE, A.w) - 0.5f;
    long long tpe = 0;
    auto acquire = [&](int k) {
      if (k > acquired) {
        const long long t0 = clock64();
        if (k >= PX_RING) mbar_wait(&s_empty[k % PX_RING], ((k / PX_RING) - 1) & 1);
        tpe += clock64() - t0;
        acquired = k;
      }
    };
    auto publish = [&](int k, int n) {
      __syncwarp();
      if (lane == 0) {
        if (n > 0) A.ch_used[slot0 + k] = 0u;  // consumers OR their masks in
        s_hdr[k % PX_RING] = n;
        s_wrap[k % PX_RING] = wrap_c;
        mbar_arrive(&s_full[k % PX_RING]);
      }
    };
    const int end = g.any ? len : 0;
    // software pipeline: list indices DI batches ahead, records DR batches
    // ahead (the record load depends on the index load)
    constexpr int DI = 10, DR = 6;
    auto ld_idx = [&](int p) -> uint32_t {
      return p + lane < end ? (uint32_t)__ldcg(A.pairs + start + p + lane) : 0xffffffffu;
    };
    auto ld_rec = [&](uint32_t i, float4& a, float4& b) {
      if (i != 0xffffffffu) {
        a = __ldg(A.rrec + 2 * (size_t)i);
        b = __ldg(A.rrec + 2 * (size_t)i + 1);
      } else {
        a = make_float4(0.f, 0.f, 0.f, 0.f);
        b = make_float4(0.f, -INFINITY, -1.f, -1.f);
      }
    };
    uint32_t qi[DI];
    float4 qa[DR], qb[DR];
#pragma unroll
    for (int j = 0; j < DI; ++j) qi[j] = ld_idx(32 * j);
#pragma unroll
    for (int j = 0; j < DR; ++j) ld_rec(qi[j], qa[j], qb[j]);
    // append one 32-entry batch (list positions p..p+31) to the ring
    auto append = [&](uint32_t idx, float4 r0, float4 r1, bool keep, int p) {
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      const int ns = __popc(m);
      // azimuth wrap of the entry over the CTA: rint((pcx - mx) / w) is
      // monotone in pcx, so equal values at the two end columns make it
      // uniform, and the consumers add the exact shift -w k instead
      // (fmaf(-w, k, dxr) == dxr + (-w k): the product is exact); a chunk
      // with a non-uniform entry takes the per-pixel wrap
      const float k_lo = rintf((pxlo - r0.x) * A.inv_w), k_hi = rintf((pxhi - r0.x) * A.inv_w);
      {
        const bool wr = keep && k_lo != k_hi;
        const bool second = fill + __popc(m & lt) >= PX_K;
        wrap_c |= __any_sync(0xffffffffu, wr && !second);
        wrap_n |= __any_sync(0xffffffffu, wr && second);
      }
      acquire(c);
      if (fill + ns > PX_K) acquire(c + 1);
      if (keep) {
        const int q = fill + __popc(m & lt);
        const int k = q < PX_K ? c : c + 1;
        const int e = q & (PX_K - 1);
        const float4 r1p =
            make_float4(r1.x, r1.y, __int_as_float(p + lane), __int_as_float((int)idx));
        s_ring[k % PX_RING][e][0] = r0;
        s_ring[k % PX_RING][e][1] = make_float4(r1.x, r1.y, r1p.z, -A.wf * k_lo);
        if (SC) {
#pragma unroll
          for (int ch = 0; ch < SCW; ++ch)
            s_cf[k % PX_RING][e][ch] = ch < SC ? __ldg(A.coef + (int64_t)idx * SC + ch) : 0.f;
        }
        const int64_t o = (slot0 + k) * PX_K + e;
        A.ch_idx[o] = idx;
        if (A.ch_pos) A.ch_pos[o] = p + lane;
        if (!SC && k >= A.wmax) {  // pass B recomputes these chunks' weights
          A.ch_rec[2 * o] = r0;
          A.ch_rec[2 * o + 1] = r1p;
        }
      }
      fill += ns;
      if (fill >= PX_K) {
        publish(c, PX_K);
        ++c;
        fill -= PX_K;
        wrap_c = wrap_n;
        wrap_n = 0;
      }
    };
    // two batches per step: their culls are independent chains, so the
    // producer warp -- alone on its scheduler and the limit of the CTAs
    // whose pixels walk the whole list -- runs them side by side
    for (int pos = 0; pos < end; pos += 64) {
      const uint32_t idxA = qi[0], idxB = qi[1];
      const float4 r0A = qa[0], r1A = qb[0], r0B = qa[1], r1B = qb[1];
#pragma unroll
      for (int j = 0; j + 2 < DR; ++j) {
        qa[j] = qa[j + 2];
        qb[j] = qb[j + 2];
      }
      ld_rec(qi[DR], qa[DR - 2], qb[DR - 2]);
      ld_rec(qi[DR + 1], qa[DR - 1], qb[DR - 1]);
#pragma unroll
      for (int j = 0; j + 2 < DI; ++j) qi[j] = qi[j + 2];
      qi[DI - 2] = ld_idx(pos + 32 * DI);
      qi[DI - 1] = ld_idx(pos + 32 * (DI + 1));
      if (*(volatile int*)&s_ndone == 4) break;  // every pixel finished
      // (non-short-circuit: both tests of both batches issue branch-free)
      const bool keepA = (idxA != 0xffffffffu) & cull_keep(r0A, r1A, g, A.wf, A.inv_w) &
                         tight_keep(r0A, r1A, pxlo, pxhi, g.ylo, g.yhi, A.wf, A.inv_w);
      const bool keepB = (idxB != 0xffffffffu) & cull_keep(r0B, r1B, g, A.wf, A.inv_w) &
                         tight_keep(r0B, r1B, pxlo, pxhi, g.ylo, g.yhi, A.wf, A.inv_w);
      append(idxA, r0A, r1A, keepA, pos);
      if (pos + 32 < end) append(idxB, r0B, r1B, keepB, pos + 32);
    }
    if (fill > 0) {  // zero-opacity padding: alpha = 0, never included
      if (lane >= fill) {
        s_ring[c % PX_RING][lane][0] = make_float4(0.f, 0.f, 0.f, 0.f);
        s_ring[c % PX_RING][lane][1] = make_float4(0.f, -INFINITY, __int_as_float(-1), 0.f);
        if (SC) {
#pragma unroll
          for (int ch = 0; ch < SCW; ++ch) s_cf[c % PX_RING][lane][ch] = 0.f;
        }
        const int64_t o = (slot0 + c) * PX_K + lane;
        A.ch_idx[o] = 0xffffffffu;
        if (!SC && c >= A.wmax) {
          A.ch_rec[2 * o] = make_float4(0.f, 0.f, 0.f, 0.f);
          A.ch_rec[2 * o + 1] = make_float4(0.f, -INFINITY, __int_as_float(-1), __int_as_float(-1));
        }
      }
      publish(c, fill);
      ++c;
    }
    acquire(c);
    publish(c, -1);  // end of list
    if (A.dbg && lane == 0) {
      A.dbg[cta * 16 + 0] = tpe;
      A.dbg[cta * 16 + 1] = clock64() - t_startA;
      A.dbg[cta * 16 + 2] = c;
    }
  } else {
    // ---------------- consumers: one pixel per lane
    const int px = g.x0 + (lane & 15), py = g.y0 + half_row(warp, lane >> 4);
    const bool inside = px < A.w && py < A.h;
    const float pcx = (float)px + 0.5f, pcy = (float)py + 0.5f;
    const float teps = A.t_eps, wf = A.wf, inv_w = A.inv_w;
    float T = inside ? 1.f : 0.f;  // outside pixels are never live
    int cnt = 0, last = 0, lastch = 0;
    float acc[SCW];
#pragma unroll
    for (int ch = 0; ch < SCW; ++ch) acc[ch] = 0.f;
    bool wdone = !__any_sync(0xffffffffu, T >= teps);
    if (wdone && lane == 0) atomicAdd(&s_ndone, 1);
    long long twf = 0, tcc = 0;
    for (int c = 0;; ++c) {
      const int s = c % PX_RING;
      const long long tf0 = clock64();
      mbar_wait(&s_full[s], (c / PX_RING) & 1);
      twf += clock64() - tf0;
      const int n = *(volatile int*)&s_hdr[s];
      if (n < 0) break;
      const long long tc0 = clock64();
      if (!SC && c >= A.wmax) A.ch_T[(slot0 + c) * 128 + warp * 32 + lane] = T;  // pass B restart
      // the pixel's 32 blending weights of this chunk, stored for pass B
      // (coalesced: entry quad j of the CTA's 128 pixels is one 2 KB row)
      const bool wst = !SC && c < A.wmax;
      float4* wrow = A.pxw + ((int64_t)cta * A.wmax + c) * 8 * 128 + warp * 32 + lane;
      unsigned um = 0;
      if (!wdone) {
        unsigned actm = 0;
        float Tl = T;
        float wq[PX_K];
        // the ring's r1.w holds the entry's azimuth shift -w k when the
        // chunk's wraps are uniform over the CTA (s_wrap == 0): same bits as
        // the per-pixel wrap, three instructions fewer per entry
        auto walk = [&](auto uniform_tag) {
          constexpr bool UNI = decltype(uniform_tag)::value;
#pragma unroll
          for (int k = 0; k < PX_K; ++k) {
            const float4 r0 = s_ring[s][k][0], r1 = s_ring[s][k][1];
            const float a = UNI ? fast_alpha_shift(pcx, pcy, r0, r1)
                                : fast_alpha_uncut(pcx, pcy, r0, r1, wf, inv_w);
            const bool act = Tl >= teps && a >= ALPHA_MIN_F;  // = fast_alpha(..) > 0
            const float wgt = act ? Tl * a : 0.f;
            if (SC) {
              const float4 cf = *(const float4*)&s_cf[s][k][0];
              acc[0] = fmaf(wgt, cf.x, acc[0]);
              if (SC > 1) acc[1] = fmaf(wgt, cf.y, acc[1]);
              if (SC > 2) acc[2] = fmaf(wgt, cf.z, acc[2]);
              if (SC > 3) acc[3] = fmaf(wgt, cf.w, acc[3]);
            } else {
              wq[k] = wgt;
            }
            Tl = act ? fmaf(-Tl, a, Tl) : Tl;  // T (1 - alpha), one rounding
            actm |= act ? (1u << k) : 0u;
          }
        };
        if (s_wrap[s])
          walk(std::integral_constant<bool, false>());
        else
          walk(std::integral_constant<bool, true>());
        T = Tl;
        if (actm) {
          cnt += __popc(actm);
          last = __float_as_int(s_ring[s][31 - __clz(actm)][1].z) + 1;
        }
        um = __reduce_or_sync(0xffffffffu, actm);
        if (!SC && wst && um) {
#pragma unroll
          for (int j = 0; j < PX_K / 4; ++j)
            wrow[j * 128] = make_float4(wq[4 * j], wq[4 * j + 1], wq[4 * j + 2], wq[4 * j + 3]);
        }
        if (um) {
          lastch = c + 1;
          if (lane == 0) atomicOr(A.ch_used + slot0 + c, um);
        }
        wdone = !__any_sync(0xffffffffu, T >= teps);
        if (wdone && lane == 0) atomicAdd(&s_ndone, 1);
      }
      if (wst && lane == 0) A.ch_wm[(slot0 + c) * 4 + warp] = um;  // 0: no weights stored
      tcc += clock64() - tc0;
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[s]);
    }
    if (A.dbg && lane == 0) {
      A.dbg[cta * 16 + 3 + warp] = twf;
      A.dbg[cta * 16 + 7 + warp] = tcc;
    }
    if (inside) {
      const int q = py * A.w + px;
      A.T_out[q] = inside ? T : 1.f;
      A.count_out[q] = cnt;
      A.last_out[q] = last;
      if (SC) {
#pragma unroll
        for (int ch = 0; ch < SC; ++ch) {
          const int b = ch / A.C, cc = ch - b * A.C;
          A.img[(((int64_t)b * A.h + py) * A.w + px) * A.C + cc] = acc[ch];
        }
      }
    }
    const int wmax = __reduce_max_sync(0xffffffffu, last);
    if (lane == 0) {
      A.wstop[g.tile * 8 + g.half * 4 + warp] = wmax;
      atomicMax(&s_nch, lastch);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) A.ch_n[cta] = s_nch;
  if (A.dbg && threadIdx.x == 0) {
    A.dbg[cta * 16 + 11] = clock64() - t_startA;
    A.dbg[cta * 16 + 12] = s_nch;
  }
  // live list (for the lazy MLP): entries of this CTA's chunks with an
  // included contribution; the first CTA to flag a Gaussian appends it.
  // Done once per CTA, off the per-chunk critical path.
  // Loads, flag exchanges and list appends of up to LE entries per thread in
  // flight together; one list reservation per warp and round.
  const int nused = s_nch * PX_K;
  constexpr int LE = 4;
  for (int t0 = threadIdx.x; t0 - (int)threadIdx.x < nused; t0 += LE * (int)blockDim.x) {
    uint32_t used[LE];
    int idx[LE];
#pragma unroll
    for (int k = 0; k < LE; ++k) {
      const int t = t0 + k * blockDim.x, c = t >> 5;
      used[k] = t < nused ? __ldcg(A.ch_used + slot0 + c) : 0u;
      idx[k] = t < nused ? (int)__ldcg(A.ch_idx + (slot0 + c) * PX_K + (t & 31)) : -1;
    }
    bool fresh[LE];
#pragma unroll
    for (int k = 0; k < LE; ++k) {
      const int t = t0 + k * blockDim.x;
      fresh[k] = ((used[k] >> (t & 31)) & 1u) && atomicExch(A.live + idx[k], 1) == 0;
    }
    int nf = 0;
#pragma unroll
    for (int k = 0; k < LE; ++k) nf += fresh[k];
    int incl = nf;  // warp inclusive scan of the fresh counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if ((threadIdx.x & 31) >= o) incl += u;
    }
    const int wtot = __shfl_sync(0xffffffffu, incl, 31);
    int base = 0;
    if ((threadIdx.x & 31) == 31 && wtot) base = atomicAdd(A.counters + GSPARC_CNT_LIVE, wtot);
    base = __shfl_sync(0xffffffffu, base, 31) + incl - nf;
#pragma unroll
    for (int k = 0; k < LE; ++k)
      if (fresh[k]) A.live_list[base++] = idx[k];
  }
  // this CTA's live-list entries are written: count it finished (K1 stops
  // waiting for entries once every pass-A CTA has)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(A.counters + GSPARC_CNT_PXA_DONE, 1);
  }
  if (A.dbg && threadIdx.x == 0) A.dbg[cta * 16 + 15] = gtimer();
  // this grid completes only after K3 has (its writes are then visible to
  // every later kernel in the stream)
  if (A.ready) pdl_wait();
}

// ------------------------------------------------------------------ pass B
// K-major SWIZZLE_128B UMMA descriptor: rows of 128 B, 8-row atoms 1024 B
// apart (SBO), LBO unused, version 1, layout type 2.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db,
                                            uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]));
}

// Pass B:  img[128 px, NP] += W[128 px, 32] . coef[32, NP] per chunk.
//   A = W (tf32 hi/lo) in TMEM, lane = pixel, written with tcgen05.st;
//   B = coef (hi = the f32 row, lo = x - tf32(x)) in shared memory, MN-major
//       SWIZZLE_128B_BASE32B (atoms of 4 entries x 32 channels);
//   D = img in TMEM (lane = pixel, column = channel).
// Two groups of 4 weight warps take alternate chunks; a group owns its A and
// B stage, stages both operands of its chunk (the coef rows of the entries
// the pass-A used mask marks -- rows of other entries keep stale finite data
// and meet zero weights), and signals one barrier.  The coef loads are
// issued before the alpha math so their latency hides under it.  One thread
// issues 4 K-steps x 3 (Wh.ch + Wh.cl + Wl.ch) MMAs per chunk.
// (A dedicated producer warp, cp.async or TMA tile::gather4, was measured
// slower: its serial issue time per chunk set the critical path.)
template <int NP>
struct PxbCfg {
  static constexpr int NA = (NP + 31) / 32;            // 32-channel atoms
  static constexpr int PLANE = NA * 4 * 1024;          // 32 entries x NA atoms
  static constexpr int STAGE = 2 * PLANE;              // hi | lo
  static constexpr uint32_t D_COLS = NP <= 32 ? 32 : NP <= 64 ? 64 : NP <= 128 ? 128 : 256;
  static constexpr uint32_t A_COL0 = D_COLS;
  static constexpr uint32_t TMEM_COLS = D_COLS + 128 <= 256 ? 256 : 512;
  static constexpr int THREADS = 256;                  // 2 groups x 4 weight warps
  static constexpr int MIN_CTAS = TMEM_COLS == 256 ? 2 : 1;
  // 16K registers per SM sub-partition: 2 CTAs x 8 warps = 4 warps each
  static constexpr int MAXREG = MIN_CTAS == 2 ? 128 : 224;
  static constexpr int PPR = NA * 8;                   // 16 B pieces per coef row
  static constexpr int NPF = (PX_K * PPR + 127) / 128; // pieces per group thread
  static constexpr int EP_ROW = NP * 4 + 16;           // epilogue staging row (padded)
  static constexpr int SMEM = (2 * STAGE > 128 * EP_ROW ? 2 * STAGE : 128 * EP_ROW) + 1024;
};

__device__ __forceinline__ uint32_t base32b_off(int k, int j, int na) {
  // byte offset of 16 B piece j (channels 4j..4j+3) of entry k
  return (uint32_t)((k >> 2) * (na * 512) + (j >> 3) * 512 + (k & 3) * 128 +
                    ((((j & 7) >> 1) ^ (k & 3)) << 5) + ((j & 1) << 4));
}

// MN-major descriptor for 32-bit data: layout SWIZZLE_128B_BASE32B (type 1,
// the only MN-major swizzle tf32 accepts -- plain SWIZZLE_128B reads zeros,
// see scripts/umma_probe.cu).  LBO = atom stride along N (512 B), SBO =
// stride between 4-entry groups along K (NA * 512 B).
__device__ __forceinline__ uint64_t umma_desc_mn_b32(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(512 >> 4) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)1 << 61;
  return d;
}

template <int NP>
__global__ void __launch_bounds__(PxbCfg<NP>::THREADS) __maxnreg__(PxbCfg<NP>::MAXREG)
    k_pxb(PxArgs A) {
  using CF = PxbCfg<NP>;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  unsigned char* sB = sm;  // [2 stages][hi|lo][8 entry groups][NA atoms][4 rows][128 B]
  __shared__ __align__(16) float4 s_rec[8][2 * PX_K];  // per weight warp
  __shared__ int s_cidx[8][PX_K];                       // source index of K column
  __shared__ __align__(8) uint64_t s_full[2], s_empty[2], s_done;
  __shared__ uint32_t s_tmem;
  __shared__ int s_next;  // next chunk whose MMAs may be issued (order token)
  __shared__ int s_acc;   // accumulator initialised (an MMA was issued)

  const long long t_start = clock64();
  // (tile, half) of this CTA: with mix_b, consecutive CTAs alternate between
  // a tile of the top half of the image and one of the bottom half, so the
  // two CTAs an SM receives together rarely are both of a heavy tile row
  int cta = blockIdx.x, ychunk = blockIdx.y;
  if (A.mix_b) {
    const int k = blockIdx.x >> 1, nt = A.ntiles;
    const int tile = (k & 1) ? nt - 1 - (k >> 1) : (k >> 1);
    cta = 2 * tile + (blockIdx.x & 1);
  }
  if (A.tile_major_b) {
    // the channel-chunk CTAs of one half tile are consecutive in launch
    // order, so they run together: its stored weights come from DRAM once
    // (then L2) and its pixels' image rows are completed while in L2
    const int lin = blockIdx.x + blockIdx.y * gridDim.x;
    cta = lin / gridDim.y;
    ychunk = lin - cta * gridDim.y;
  }
  if (A.dbg && threadIdx.x == 0) A.dbg[cta * 16 + 12] = gtimer();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const CtaGeom g = cta_geom(A, cta);
  const int col0 = ychunk * NP;
  // ordinary launch: the chunk count and list bounds are read first so their
  // latency overlaps the prologue; a dependent launch reads them after its
  // grid-dependency wait
  int64_t slot0 = 0;
  int nch = 0;
  if (!A.pdl_b) {
    slot0 = chunk_slot0(A.tile_start, g.tile, g.half);
    nch = g.any && !A.counters[GSPARC_CNT_OVERFLOW] ? A.ch_n[cta] : 0;
  }

  if (threadIdx.x == 0) {
    for (int k = 0; k < 2; ++k) {
      mbar_init(&s_full[k], 4);
      mbar_init(&s_empty[k], 1);
    }
    mbar_init(&s_done, 1);
    s_next = 0;
    s_acc = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(CF::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  // launched as a dependent of the previous kernel (the lazy MLP or pass A):
  // the prologue above overlaps its tail; nothing upstream is read before
  // this wait
  if (A.pdl_b) {
    pdl_wait();
    slot0 = chunk_slot0(A.tile_start, g.tile, g.half);
    nch = g.any && !A.counters[GSPARC_CNT_OVERFLOW] ? A.ch_n[cta] : 0;
  }
  if (A.dbg && threadIdx.x == 0) {
    A.dbg[cta * 16 + 13] = clock64() - t_start;
    A.dbg[cta * 16 + 5] = gtimer();  // upstream grid complete
  }

  if (warp < 8) {
    // ---------------- weight groups: group gq takes chunks c = gq (mod 2)
    const int gq = warp >> 2, q = warp & 3, gt = q * 32 + lane;  // thread in group
    const int px = g.x0 + (lane & 15), py = g.y0 + half_row(q, lane >> 4);
    const float pcx = (float)px + 0.5f, pcy = (float)py + 0.5f;
    const float teps = A.t_eps, wf = A.wf, inv_w = A.inv_w;
    float4* rs = s_rec[warp];
    const uint32_t a_hi = tmem + ((uint32_t)(32 * q) << 16) + CF::A_COL0 + 64 * gq;
    const uint32_t a_lo = a_hi + 32;
    unsigned char* bhi = sB + gq * CF::STAGE;
    unsigned char* blo = bhi + CF::PLANE;
    // instruction descriptor: D f32, A/B tf32, A K-major, B MN-major,
    // N = NP, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) |
                           ((uint32_t)(NP >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const bool vec = (A.Cp & 3) == 0;
    const int ncol = (int)min((int64_t)NP, A.Cp - col0);   // channels of this CTA
    const int ppr = (ncol + 3) >> 2;                        // pieces with channels
    float4 n0 = make_float4(0.f, 0.f, 0.f, 0.f), n1 = n0;
    float nT = 0.f;
    uint32_t nused = 0;
    int nidx = -1;
    uint32_t nwm = 0;
    int* cidx = s_cidx[warp];
    // chunks c < wmax: pass A stored the pixels' weights (pxw); later chunks
    // recompute them from the T checkpoint and the entry records
    auto prefetch = [&](int c, bool wp) {
      if (c < nch) {
        const int64_t slot = slot0 + c;
        nused = A.ch_used[slot];
        if (wp) {
          nidx = (int)A.ch_idx[slot * PX_K + lane];
          nwm = A.ch_wm[slot * 4 + q];
        } else {
          n0 = A.ch_rec[2 * (slot * PX_K + lane)];
          n1 = A.ch_rec[2 * (slot * PX_K + lane) + 1];
          nT = A.ch_T[slot * 128 + q * 32 + lane];
        }
      }
    };
    long long tw = 0, tc = 0;
    auto chunk = [&](auto wp_tag, int c) {
      constexpr bool wp = decltype(wp_tag)::value;
      const int k = c >> 1;
      float T = nT;
      const uint32_t used = nused;
      __syncwarp();  // previous chunk's readers are done with rs / cidx
      // K column j of the chunk's MMA and the coef rows to load (mask lm):
      //   stored weights: column j = entry j (list order); entries no pixel
      //     of the CTA includes have zero weight everywhere, their B rows keep
      //     stale finite data and are not loaded;
      //   recomputed: the used entries compacted to the front (skipping an
      //     unused entry is exact: every live pixel sees alpha = 0 there),
      //     padding slots get zero records.
      int nu;
      uint32_t lm;
      if (wp) {
        cidx[lane] = nidx;
        nu = PX_K;
        lm = used;
      } else {
        nu = __popc(used);
        lm = nu >= 32 ? 0xffffffffu : (1u << nu) - 1u;
        if (lane >= nu) {  // padding slots: zero opacity (log2 = -inf), alpha = 0
          rs[2 * lane] = make_float4(0.f, 0.f, 0.f, 0.f);
          rs[2 * lane + 1] = make_float4(0.f, -INFINITY, __int_as_float(-1), __int_as_float(-1));
          cidx[lane] = -1;
        }
        if ((used >> lane) & 1u) {  // used entries, in list order
          const int slot = __popc(used & ((1u << lane) - 1u));
          rs[2 * slot] = n0;
          rs[2 * slot + 1] = n1;
          cidx[slot] = __float_as_int(n1.w);
        }
      }
      float4 wr[PX_K / 4];
      if (wp) {  // this pixel's stored weights (none stored: all zero)
        const uint32_t wm = nwm;
        const float4* src = A.pxw + ((int64_t)cta * A.wmax + c) * 8 * 128 + q * 32 + lane;
#pragma unroll
        for (int j = 0; j < PX_K / 4; ++j)
          wr[j] = wm ? __ldcg(src + j * 128) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if (!wp || c + 2 < A.wmax) prefetch(c + 2, wp);
      __syncwarp();
      // coef rows of the loaded columns, issued now and consumed after the
      // weights: piece p = gt + 128 u of the 32 x PPR (column, 16 B piece)
      // grid; the column is uniform per warp for PPR >= 32
      float4 cv[CF::NPF];
#pragma unroll
      for (int u = 0; u < CF::NPF; ++u) {
        const int p = gt + 128 * u;
        const int e = p / CF::PPR, jj = p - e * CF::PPR;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e < PX_K && ((lm >> e) & 1u) && jj < ppr) {
          const int idx = cidx[e];
          if (idx >= 0) {
            const float* row = A.coef + (int64_t)idx * A.Cp + col0 + 4 * jj;
            if (vec) {
              v = __ldg((const float4*)row);
            } else {
              const int nv = ncol - 4 * jj;
              v.x = __ldg(row);
              if (nv > 1) v.y = __ldg(row + 1);
              if (nv > 2) v.z = __ldg(row + 2);
              if (nv > 3) v.w = __ldg(row + 3);
            }
          }
        }
        cv[u] = v;
      }
      const long long t0 = clock64();
      float wv[PX_K];
      if (wp) {
#pragma unroll
        for (int j = 0; j < PX_K / 4; ++j) {
          wv[4 * j] = wr[j].x;
          wv[4 * j + 1] = wr[j].y;
          wv[4 * j + 2] = wr[j].z;
          wv[4 * j + 3] = wr[j].w;
        }
      } else {
#pragma unroll
        for (int e = 0; e < PX_K; ++e) wv[e] = 0.f;
        if (__any_sync(0xffffffffu, T >= teps)) {
#pragma unroll
          for (int e0 = 0; e0 < PX_K; e0 += 8) {
            if (e0 >= nu) break;  // uniform: groups of 8 keep the ILP
#pragma unroll
            for (int e = e0; e < e0 + 8; ++e) {
              const float a = fast_alpha(pcx, pcy, rs[2 * e], rs[2 * e + 1], wf, inv_w);
              const bool act = T >= teps && a > 0.f;
              wv[e] = act ? T * a : 0.f;
              T = act ? fmaf(-T, a, T) : T;
            }
          }
        }
      }
      const long long t1 = clock64();
      if (k >= 1) mbar_wait_sleep(&s_empty[gq], (k - 1) & 1);
      const long long t2 = clock64();
      tc += t1 - t0;
      tw += t2 - t1;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t hi[16], lo[16];
#pragma unroll
        for (int jx = 0; jx < 16; ++jx) {
          const float v = wv[16 * hh + jx];
          hi[jx] = __float_as_uint(v) & 0xFFFFE000u;
          lo[jx] = __float_as_uint(v - __uint_as_float(hi[jx]));
        }
        tmem_st16(a_hi + 16 * hh, hi);
        tmem_st16(a_lo + 16 * hh, lo);
      }
      // coef hi/lo planes: every row of a K-step the MMAs read (8 entries
      // with at least one loaded row), unloaded rows as zeros (cv = 0), so
      // the stage never feeds stale or uninitialised data to a used K-step
#pragma unroll
      for (int u = 0; u < CF::NPF; ++u) {
        const int p = gt + 128 * u;
        const int e = p / CF::PPR, jj = p - e * CF::PPR;
        if (e < PX_K && ((lm >> (e & ~7)) & 0xFFu) && jj < ppr) {
          const float4 x = cv[u];
          float4 h;
          h.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
          h.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
          h.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
          h.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
          const uint32_t off = base32b_off(e, jj, CF::NA);
          *(float4*)(bhi + off) = h;
          *(float4*)(blo + off) = make_float4(x.x - h.x, x.y - h.y, x.z - h.z, x.w - h.w);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_full[gq]);
      if (q == 0 && lane == 0) {
        // this group's leader issues the chunk's MMAs once all 4 warps have
        // staged it, in chunk order (token), so the accumulation order --
        // and the image -- is the same on every run
        mbar_wait(&s_full[gq], k & 1);
        while (*(volatile int*)&s_next != c) {
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t ma_hi = tmem + CF::A_COL0 + 64 * gq, ma_lo = ma_hi + 32;
        const uint32_t mb_hi = smem_u32(bhi), mb_lo = mb_hi + CF::PLANE;
        // K-steps whose 8 columns carry no coef row are all-zero in A: skip
        // them (the first MMA issued initialises the accumulator)
#pragma unroll
        for (int ks = 0; ks < PX_K / 8; ++ks) {
          if (((lm >> (8 * ks)) & 0xFFu) == 0u) continue;
          const uint32_t acc0 = s_acc ? 1u : 0u;
          s_acc = 1;
          const uint32_t ko = ks * CF::NA * 1024;  // 8 entries = 2 atom rows of K
          mma_tf32_ts(tmem, ma_hi + 8 * ks, umma_desc_mn_b32(mb_hi + ko, CF::NA * 512), idesc,
                      acc0);
          mma_tf32_ts(tmem, ma_hi + 8 * ks, umma_desc_mn_b32(mb_lo + ko, CF::NA * 512), idesc,
                      1u);
          mma_tf32_ts(tmem, ma_lo + 8 * ks, umma_desc_mn_b32(mb_hi + ko, CF::NA * 512), idesc,
                      1u);
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                smem_u32(&s_empty[gq]))
            : "memory");
        if (c == nch - 1)
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                  smem_u32(&s_done))
              : "memory");
        __threadfence_block();
        *(volatile int*)&s_next = c + 1;
      }
      __syncwarp();
    };
    // stored-weight chunks, then (beyond wmax) recomputed ones
    const int nw = min(nch, A.wmax);
    int c = gq;
    if (c < nw) prefetch(c, true);
    for (; c < nw; c += 2) chunk(std::integral_constant<bool, true>(), c);
    if (c < nch) prefetch(c, false);
    for (; c < nch; c += 2) chunk(std::integral_constant<bool, false>(), c);
    if (A.dbg && lane == 0 && q == 0) {
      A.dbg[cta * 16 + 6 + gq] = tw;
      A.dbg[cta * 16 + 8 + gq] = tc;
    }
  }

  // ---------------- epilogue: warp w reads TMEM lanes 32 (w % 4).. (= pixels),
  // columns [0, NPH) for w < 4 and [NPH, NP) for the second group
  if (warp < 8) {
    constexpr int NPH = ((NP / 2 + 7) / 8) * 8;
    const int q = warp & 3;
    const int cbeg = warp < 4 ? 0 : NPH, cend = warp < 4 ? NPH : NP;
    const int px = g.x0 + (lane & 15), py = g.y0 + half_row(q, lane >> 4);
    const bool inside = px < A.w && py < A.h;
    if (nch > 0) {
      mbar_wait_sleep(&s_done, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    const long long te0 = clock64();
    if (A.dbg && threadIdx.x == 0) A.dbg[cta * 16 + 14] = te0 - t_start;
    const bool fast = (A.C % 8) == 0 && (A.Cp % 8) == 0;
    const int ncol_cta = (int)min((int64_t)NP, A.Cp - col0);
    // image rows through shared memory: when the CTA's columns are one
    // contiguous run of every pixel's row (one TX, 16 B multiples), the
    // accumulator goes TMEM -> shared memory (row per pixel, padded) and
    // each pixel's run is written by one bulk copy -- full-line writes
    // instead of 32 B pieces 4 C bytes apart
    const bool bulk = nch > 0 && (A.C % 4) == 0 && (col0 % 4) == 0 && (ncol_cta % 4) == 0 &&
                      col0 / A.C == (col0 + ncol_cta - 1) / A.C;
    if (bulk) {
      constexpr int RSB = CF::EP_ROW;  // row stride (bytes)
      const int row = q * 32 + lane;
      unsigned char* ep = sB + row * RSB;
#pragma unroll 1
      for (int c0 = cbeg; c0 < cend; c0 += 8) {
        uint32_t v[8];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c0 < ncol_cta) {
          uint4* d4 = (uint4*)(ep + 4 * c0);
          d4[0] = make_uint4(v[0], v[1], v[2], v[3]);
          if (c0 + 4 < ncol_cta) d4[1] = make_uint4(v[4], v[5], v[6], v[7]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync 1, 256;" ::: "memory");  // the 8 epilogue warps
      // warp w copies pixels 16 w .. 16 w + 15 (TMEM lane = pixel)
      if (lane < 16) {
        const int r = 16 * warp + lane, rq = r >> 5, rl = r & 31;
        const int bx = g.x0 + (rl & 15), by = g.y0 + half_row(rq, rl >> 4);
        if (bx < A.w && by < A.h) {
          const int64_t b = col0 / A.C, ch = col0 - b * A.C;
          float* dst = A.img + ((b * A.h + by) * (int64_t)A.w + bx) * A.C + ch;
          asm volatile(
              "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
              "r"(smem_u32(sB + r * RSB)), "r"(ncol_cta * 4)
              : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem read out
      }
    } else {
#pragma unroll 1
    for (int c0 = cbeg; c0 < cend; c0 += 8) {
      uint32_t v[8];
      if (nch > 0) {
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      } else {
#pragma unroll
        for (int jx = 0; jx < 8; ++jx) v[jx] = 0u;
      }
      const int64_t cc0 = col0 + c0;
      if (!inside || cc0 >= A.Cp) continue;
      if (fast) {
        const int64_t b = cc0 / A.C, ch = cc0 - b * A.C;
        float4* dst = (float4*)(A.img + ((b * A.h + py) * (int64_t)A.w + px) * A.C + ch);
        dst[0] = make_float4(__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]),
                             __uint_as_float(v[3]));
        dst[1] = make_float4(__uint_as_float(v[4]), __uint_as_float(v[5]), __uint_as_float(v[6]),
                             __uint_as_float(v[7]));
      } else if ((A.C & 1) == 0 && (A.Cp & 1) == 0) {
        // even channel counts (config 1: 64 TX x 2): channel pairs as 8 B
        // stores -- a warp's 16 pixels of a row write 16 C contiguous bytes
#pragma unroll
        for (int jx = 0; jx < 8; jx += 2) {
          const int64_t cc = cc0 + jx;
          if (cc < A.Cp) {
            const int64_t b = cc / A.C, ch = cc - b * A.C;
            *(float2*)(A.img + ((b * A.h + py) * (int64_t)A.w + px) * A.C + ch) =
                make_float2(__uint_as_float(v[jx]), __uint_as_float(v[jx + 1]));
          }
        }
      } else {
#pragma unroll
        for (int jx = 0; jx < 8; ++jx) {
          const int64_t cc = cc0 + jx;
          if (cc < A.Cp) {
            const int64_t b = cc / A.C, ch = cc - b * A.C;
            A.img[((b * A.h + py) * (int64_t)A.w + px) * A.C + ch] = __uint_as_float(v[jx]);
          }
        }
      }
    }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(CF::TMEM_COLS));
  }
  if (A.dbg && threadIdx.x == 0) {
    A.dbg[cta * 16 + 10] = clock64() - t_start;
    A.dbg[cta * 16 + 11] = nch;
    A.dbg[cta * 16 + 15] = gtimer();
  }
}

long long* gsparc_dbg_ptr = nullptr;  // experiments: timing rows (K3 | K4a | K4b)

// experiments: one buffer of 16-slot rows: K3 rows [0, 4096), K4a rows
// [4096, 8192), K4b rows [8192, 12288), K2 rows [12288, 16384); cleared once (a per-launch memset
// would split the K3 -> K4a programmatic launch)
long long* dbg_rows(int which) {
  if (!gsparc_dbg_ptr) {
    cudaMalloc(&gsparc_dbg_ptr, sizeof(long long) * 16 * 16384);
    cudaMemset(gsparc_dbg_ptr, 0, sizeof(long long) * 16 * 16384);
  }
  return gsparc_dbg_ptr + (int64_t)which * 16 * 4096;
}

template <int NP>
static void launch_pxb(const PxArgs& A, int chunks_y, bool after_mlp, cudaStream_t st) {
  using CF = PxbCfg<NP>;
  size_t smem = CF::SMEM;
  // two CTAs per SM at most (TMEM); keep a third from being scheduled
  if (CF::MIN_CTAS == 2 && smem < 78 * 1024) smem = 78 * 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_pxb<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // without this the driver picks a ~100 KB carveout: one CTA per SM
    cudaFuncSetAttribute(k_pxb<NP>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         cudaSharedmemCarveoutMaxShared);
    attr = true;
  }
  PxArgs B = A;
  B.dbg = nullptr;
  B.pdl_b = 0;
  // top/bottom interleave: measured on the render path with one channel
  // chunk (config 3: 105.8 -> 104.7 us); with a dependent launch (config 5)
  // or behind pass A (config 1) it was 1-2% slower, so it is off there
  static const int mix = experiment_env("GSPARC_PXB_MIX") ? atoi(experiment_env("GSPARC_PXB_MIX")) : -1;
  B.mix_b = mix >= 0 ? mix : (after_mlp && chunks_y == 1);
  static const int tmaj = experiment_env("GSPARC_PXB_TMAJ") ? atoi(experiment_env("GSPARC_PXB_TMAJ")) : 1;
  B.tile_major_b = chunks_y > 1 && tmaj && !B.mix_b;
  if (experiment_env("GSPARC_PXB_DBG")) B.dbg = dbg_rows(2);  // experiments only
  // dependent launch behind the streaming MLP (render path, pass 2): the
  // MLP triggers once pass A has finished, so the prologue (TMEM allocation,
  // barriers, stage clearing) overlaps the MLP's last Gaussians.  Directly
  // behind pass A (pass 0) the early CTAs only park on the SMs (config 1
  // -2.5%).
  static const bool pdl_env = !getenv("GSPARC_NO_PDL") && !experiment_env("GSPARC_NO_PDL_B");
  const bool pdl = pdl_env && after_mlp;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(A.ntiles * 2, chunks_y);
  cfg.blockDim = dim3(CF::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  if (pdl) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    B.pdl_b = 1;
  }
  cudaLaunchKernelEx(&cfg, k_pxb<NP>, B);
}

static PxArgs make_px_args(const gsparc_frame_layout& L, char* frame, int n_tx, int C,
                           double t_eps, void* img) {
  PxArgs A;
  A.pairs = (const uint64_t*)(frame + L.off_pairs);
  A.tile_start = (const int*)(frame + L.off_tile_start);
  A.rrec = (const float4*)(frame + L.off_rrec);
  A.coef = (const float*)(frame + L.off_coef);
  A.ch_used = (uint32_t*)(frame + L.off_ch_used);
  A.dbg = nullptr;
  A.ch_idx = (uint32_t*)(frame + L.off_ch_idx);
  A.ch_pos = L.off_ch_pos ? (int*)(frame + L.off_ch_pos) : nullptr;  // backward frames
  A.ch_rec = (float4*)(frame + L.off_ch_rec);
  A.ch_T = (float*)(frame + L.off_ch_T);
  A.ch_n = (int*)(frame + L.off_ch_n);
  A.wstop = (int*)(frame + L.off_wstop);
  A.T_out = (float*)(frame + L.off_T);
  A.count_out = (int*)(frame + L.off_count);
  A.last_out = (int*)(frame + L.off_last);
  A.live = (int*)(frame + L.off_live);
  A.live_list = (int*)(frame + L.off_live_list);
  A.counters = (int*)(frame + L.off_counters);
  A.img = (float*)img;
  A.pxw = (float4*)(frame + L.off_pxw);
  A.ch_wm = (uint32_t*)(frame + L.off_ch_wm);
  A.wmax = (int)L.pxw_chunks;
  A.ready = nullptr;
  A.pdl_b = 0;
  A.mix_b = 0;
  A.tile_major_b = 0;
  A.Cp = (int64_t)n_tx * C;
  A.n = L.n;
  A.C = C;
  A.w = L.width;
  A.h = L.height;
  A.ntx = L.ntx;
  A.ntiles = L.ntiles;
  A.t_eps = (float)t_eps;
  A.wf = (float)L.width;
  A.inv_w = 1.0f / (float)L.width;
  return A;
}

// pass 1: weights only (aux, live list, chunk lists), any Cp
// pass 0: fused; Cp <= 4 accumulates in pass A, wider runs A then B
// pass 2: accumulation only (after pass 1 and the MLP)
int launch_raster_px(const gsparc_frame_layout& L, char* frame, int n_tx, int C, double t_eps,
                     int pass, void* img, cudaStream_t st) {
  PxArgs A = make_px_args(L, frame, n_tx, C, t_eps, img);
  const int64_t Cp = A.Cp;
  if (pass != 2 && experiment_env("GSPARC_PXA_DBG")) {  // experiments only: pass-A timing
    A.dbg = dbg_rows(1);
  }
  if (pass != 2) {
    const int grid = L.ntiles * 2;
    // programmatic dependent launch: pass A's CTAs start while K3 (the
    // stream's previous kernel, which triggers at its start) still sorts
    // other tiles; each waits for its own tile's flag.  If the previous
    // kernel is not K3 the launch degrades to ordinary stream order and the
    // flags (set by the frame's K3) are already up.
    static const bool pdl = !getenv("GSPARC_NO_PDL");
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(160);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    // two pass-A CTAs per SM at most (a shared-memory reservation): CTAs
    // that start while K3 still runs would otherwise pile up four to an SM
    // on the first free SMs and run the heaviest tiles at half speed
    static const int pad_kb = experiment_env("GSPARC_PXA_SMEM") ? atoi(experiment_env("GSPARC_PXA_SMEM")) : 90;
    if (pdl && pad_kb > 0) {
      static bool attr = false;
      if (!attr) {
        const void* ks[5] = {(const void*)k_pxa<0>, (const void*)k_pxa<1>, (const void*)k_pxa<2>,
                             (const void*)k_pxa<3>, (const void*)k_pxa<4>};
        static const int carve =
            experiment_env("GSPARC_PXA_CARVE") ? atoi(experiment_env("GSPARC_PXA_CARVE")) : 100;
        for (const void* k : ks) {
          cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, pad_kb * 1024);
          cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
        }
        attr = true;
      }
      cfg.dynamicSmemBytes = pad_kb * 1024;
    }
    if (pdl) {
      A.ready = (const int*)(frame + L.off_tile_cursor);
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
    }
    if (pass == 0 && Cp <= 4) {
      switch (Cp) {
        case 1: cudaLaunchKernelEx(&cfg, k_pxa<1>, A); break;
        case 2: cudaLaunchKernelEx(&cfg, k_pxa<2>, A); break;
        case 3: cudaLaunchKernelEx(&cfg, k_pxa<3>, A); break;
        default: cudaLaunchKernelEx(&cfg, k_pxa<4>, A); break;
      }
      return check_launch("k_pxa");
    }
    cudaLaunchKernelEx(&cfg, k_pxa<0>, A);
    GS_TRY(check_launch("k_pxa"));
    A.ready = nullptr;
    if (pass == 1) return GSPARC_OK;
  }
  // wide batches (> 256 columns, e.g. config 5's 2048) in 128-column chunks:
  // two CTAs per SM (256 TMEM columns each) hide the coef-row load latency
  // that a 256-column CTA alone on its SM waits on
  const int np_max = Cp > 256 ? 128 : 256;
  const int chunks = (int)((Cp + np_max - 1) / np_max);
  const int64_t per = (Cp + chunks - 1) / chunks;
  const bool after_mlp = pass == 2;
  if (per <= 32) launch_pxb<32>(A, chunks, after_mlp, st);
  else if (per <= 64) launch_pxb<64>(A, chunks, after_mlp, st);
  else if (per <= 104) launch_pxb<104>(A, chunks, after_mlp, st);
  else if (per <= 128) launch_pxb<128>(A, chunks, after_mlp, st);
  else launch_pxb<256>(A, chunks, after_mlp, st);
  return check_launch("k_pxb");
}

}  // namespace gs
