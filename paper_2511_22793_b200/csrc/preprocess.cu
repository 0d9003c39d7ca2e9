// K2: per-Gaussian preprocessing in f64 (one thread per Gaussian, source
// order).  Replaces geometry.cull (geometry.py:198-224) and the geometry of
// rasterizer._Prepared (rasterizer.py:75-102); the tile rectangle follows
// rasterizer._tile_lists (rasterizer.py:117-141).  Arithmetic uses
// round-to-nearest intrinsics in numpy's evaluation order so the depth key
// (and therefore the sort order) is bit-identical to numpy's.
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"

namespace gs {

long long* dbg_rows(int which);

struct PrepArgs {
  gsparc_cloud cloud;
  Pose pose;
  GeoConst gc;
  uint64_t* key;
  float4* rec32;
  double* rec64;
  float4* rrec;
  int4* rect;
  int* live;
  int* live_list;
  int* counters;
  int* tile_count;
  int* tile_cursor;
  uint64_t* stage;
  int2* seg;
  int64_t capacity;
  int seg_stride;
  long long* dbg;  // experiments: per-CTA phase clocks (GSPARC_PREP_DBG)
  int bin_small;   // rectangles up to this many tiles are binned by one thread
                   // (40: K2 24.5 -> 22.6 us on config 3; 8 was slower than
                   // none -- the average rectangle has ~10 tiles)
};

__device__ __forceinline__ double dot3_seq(double a0, double a1, double a2, double b0, double b1,
                                           double b2) {
  return add(add(mul(a0, b0), mul(a1, b1)), mul(a2, b2));
}

__device__ __forceinline__ double np_floor_div16(double v) { return floor(v / 16.0); }


// Visits every (tile, Gaussian) pair of the warp's Gaussians flagged in bigm,
// one Gaussian at a time, consecutive tiles of its rectangle (row-major, the
// seam-wrapped range after the main one) on consecutive lanes.  Warp-uniform.
template <typename F>
__device__ __forceinline__ void for_big_tiles(unsigned bigm, int ry0, int ry1, int ra0, int ra1,
                                              int rb0, int rb1, uint64_t payload, int lane,
                                              int ntx, F f) {
  while (bigm) {
    const int src = __ffs(bigm) - 1;
    bigm &= bigm - 1;
    const int y0 = __shfl_sync(0xffffffffu, ry0, src), y1 = __shfl_sync(0xffffffffu, ry1, src);
    const int a0 = __shfl_sync(0xffffffffu, ra0, src), a1 = __shfl_sync(0xffffffffu, ra1, src);
    const int b0 = __shfl_sync(0xffffffffu, rb0, src), b1 = __shfl_sync(0xffffffffu, rb1, src);
    const uint64_t v =
        ((uint64_t)__shfl_sync(0xffffffffu, (uint32_t)(payload >> 32), src) << 32) |
        __shfl_sync(0xffffffffu, (uint32_t)payload, src);
    const int na = a1 - a0 + 1, nb = b1 >= b0 ? b1 - b0 + 1 : 0, nrow = na + nb;
    const int total = (y1 - y0 + 1) * nrow;
    for (int j = lane; j < total; j += 32) {
      const int r = j / nrow, cc = j - r * nrow;
      const int tx = cc < na ? a0 + cc : b0 + (cc - na);
      f((y0 + r) * ntx + tx, v);
    }
  }
}

// Tile binning is fused in (the counting-sort digit of rasterizer.py:115-145's
// per-tile lists): every CTA histograms its Gaussians' tile rectangles,
// reserves one contiguous stage range for all of them, writes one segment
// {offset, length} per tile into its own slot and scatters its packed pairs
// (coarse depth << 32 | index).  Order inside a tile is irrelevant: K3 sorts
// each tile's gathered segments by the full key.
__global__ void __launch_bounds__(PREP_T, 4) k_preprocess(PrepArgs A) {
  extern __shared__ int s_tiles[];  // per-CTA tile histogram [ntiles], offsets [ntiles+1], tmp
  const int ntiles = A.gc.ntx * A.gc.nty;
  int* s_off = s_tiles + ntiles;
  int* s_tmp = s_off + ntiles + 1;
  __shared__ int s_base;
  const long long t_d0 = clock64();
  if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 14] = gtimer();
  pdl_trigger();  // K3 may be scheduled as SMs free up (it waits for this grid)
  for (int t = threadIdx.x; t < ntiles; t += blockDim.x) s_tiles[t] = 0;
  __syncthreads();

  // Two warps per 32 Gaussians: the even warp runs the view-dependent
  // chain (projection, pole clamp, J) and the opacity with the raster
  // record's logs, the odd warp the covariance chain (quaternion, scales,
  // V = W Sigma W^T) and the MLP's elevation input, concurrently (the two
  // chains measured 7.2k / 6.8k cycles); the odd warp's results reach the
  // even warp through shared memory (exact), which finishes cov2d, the tile
  // rectangle and the records.  Twice the
  // warps and half the dependent f64 chain per thread of a
  // one-thread-per-Gaussian mapping, with no divergence inside a warp.
  __shared__ double s_cov[PREP_T / 64][10][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const bool cov_lane = (wid & 1) != 0;
  const int64_t i = (int64_t)blockIdx.x * PREP_G + (wid >> 1) * 32 + lane;
  const bool valid = i < A.cloud.n;
  const double* W = A.pose.W;
  bool kept_out = false;
  int np_out = 0;
  uint64_t packed = 0;
  int ry0 = 0, ry1 = -1, ra0 = 0, ra1 = -1, rb0 = 0, rb1 = -1;
  double x = 0, y = 0, z = 0, depth = 0, theta = 0, mx = 0, my = 0, rho2_u = 0;
  double J00 = 0, J02 = 0, J10 = 0, J11 = 0, J12 = 0;
  bool keep = false;
  double V[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
  double opac = 0, phi = 0, Q = -1.0;
  float log2op = 0.f;
  if (valid && !cov_lane) {
    const double* P = A.cloud.positions + 3 * i;
    // every input load first: a load behind the f64 chain would be a second
    // DRAM round trip on a cold cache
    const double logit = __ldg(A.cloud.raw_opacities + i);
    double p0 = sub(__ldg(P), A.pose.rx[0]), p1 = sub(__ldg(P + 1), A.pose.rx[1]),
           p2 = sub(__ldg(P + 2), A.pose.rx[2]);
    // (p - rx) @ W.T  (geometry.py:61-64)
    x = dot3_seq(p0, p1, p2, W[0], W[1], W[2]);
    y = dot3_seq(p0, p1, p2, W[3], W[4], W[5]);
    z = dot3_seq(p0, p1, p2, W[6], W[7], W[8]);
    double xx = mul(x, x), yy = mul(y, y), zz = mul(z, z);
    double r2 = add(add(xx, yy), zz);
    depth = __dsqrt_rn(r2);  // np.linalg.norm(axis=1)
    keep = (depth >= NEAR_PLANE) && (depth <= FAR_PLANE);
    // elevation >= -90 deg is a no-op except for NaN (geometry.py:210-212)
    double sn = y / fmax(depth, 1e-30);
    keep = keep && (sn == sn);

    // projection (geometry.py:67-80), r == depth
    theta = atan2(x, z);
    mx = mul(add(theta / A.gc.pi, 1.0), A.gc.w * 0.5);
    double c_sn = fmin(fmax(y / depth, -1.0), 1.0);
    double el = asin(c_sn);
    my = mul(mul(2.0, el), A.gc.h / A.gc.pi);

    // pole clamp (geometry.py:98-113, 131-138): points above 89 deg are
    // evaluated at 89 deg with the same azimuth and radius
    double jx = x, jy = y, jz = z;
    rho2_u = add(xx, zz);
    double jr2 = r2, rho2 = rho2_u;
    if (el > A.gc.pole_lim) {
      double tgt_rho = mul(depth, A.gc.cos_lim);
      jx = mul(tgt_rho, sin(theta));
      jy = mul(depth, A.gc.sin_lim);
      jz = mul(tgt_rho, cos(theta));
      double a = mul(jx, jx), b = mul(jy, jy), c = mul(jz, jz);
      jr2 = add(add(a, b), c);
      rho2 = add(a, c);
    }
    double rho = __dsqrt_rn(rho2);
    const double ca = A.gc.ca, ce = A.gc.ce;
    // J (geometry.py:143-148)
    J00 = mul(ca, jz) / rho2;
    J02 = mul(-ca, jx) / rho2;
    double r2rho = mul(jr2, rho);
    J10 = mul(mul(-ce, jx), jy) / r2rho;
    J11 = mul(ce, rho) / jr2;
    J12 = mul(mul(-ce, jy), jz) / r2rho;

    // opacity and the raster record's logs: the view chain is the shorter
    // of the two, so these run here, ahead of the exchange
    if (logit >= 0.0) {
      opac = 1.0 / (1.0 + exp(-logit));
    } else {
      double e = exp(logit);
      opac = e / (1.0 + e);
    }
    if (A.rrec) {
      log2op = (float)log2(opac);
      const double o255 = 255.0 * opac;
      Q = o255 > 1.0 ? 2.0 * log(o255) : -1.0;
    }
  }
  if (valid && cov_lane) {
    // Sigma = (R diag s)(R diag s)^T (scene.py:84-88, 117-139)
    const double* P = A.cloud.positions + 3 * i;
    const double P0 = __ldg(P), P1 = __ldg(P + 1), P2 = __ldg(P + 2);  // loads first
    const double* qp = A.cloud.rotations + 4 * i;
    const double* lsp = A.cloud.log_scales + 3 * i;
    const double q[4] = {__ldg(qp), __ldg(qp + 1), __ldg(qp + 2), __ldg(qp + 3)};
    const double ls[3] = {__ldg(lsp), __ldg(lsp + 1), __ldg(lsp + 2)};
    double qn = __dsqrt_rn(add(add(add(mul(q[0], q[0]), mul(q[1], q[1])), mul(q[2], q[2])),
                               mul(q[3], q[3])));
    double qw = q[0] / qn, qx = q[1] / qn, qy = q[2] / qn, qz = q[3] / qn;
    double R[3][3];
    R[0][0] = 1.0 - 2.0 * add(mul(qy, qy), mul(qz, qz));
    R[0][1] = 2.0 * sub(mul(qx, qy), mul(qw, qz));
    R[0][2] = 2.0 * add(mul(qx, qz), mul(qw, qy));
    R[1][0] = 2.0 * add(mul(qx, qy), mul(qw, qz));
    R[1][1] = 1.0 - 2.0 * add(mul(qx, qx), mul(qz, qz));
    R[1][2] = 2.0 * sub(mul(qy, qz), mul(qw, qx));
    R[2][0] = 2.0 * sub(mul(qx, qz), mul(qw, qy));
    R[2][1] = 2.0 * add(mul(qy, qz), mul(qw, qx));
    R[2][2] = 1.0 - 2.0 * add(mul(qx, qx), mul(qy, qy));
    double s0 = exp(ls[0]), s1 = exp(ls[1]), s2 = exp(ls[2]);
    double M[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      M[r][0] = mul(R[r][0], s0);
      M[r][1] = mul(R[r][1], s1);
      M[r][2] = mul(R[r][2], s2);
    }
    double S[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        S[r][c] = add(add(mul(M[r][0], M[c][0]), mul(M[r][1], M[c][1])), mul(M[r][2], M[c][2]));
    // V = W S W^T
    double WS[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        WS[r][c] = add(add(mul(W[3 * r + 0], S[0][c]), mul(W[3 * r + 1], S[1][c])),
                       mul(W[3 * r + 2], S[2][c]));
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c)
        V[r][c] = add(add(mul(WS[r][0], W[3 * c + 0]), mul(WS[r][1], W[3 * c + 1])),
                      mul(WS[r][2], W[3 * c + 2]));
    // the MLP's elevation input (mlp.py:88, unclamped) from the view-space
    // position, recomputed here with the view chain's operations
    const double p0 = sub(P0, A.pose.rx[0]), p1 = sub(P1, A.pose.rx[1]),
                 p2 = sub(P2, A.pose.rx[2]);
    const double vx = dot3_seq(p0, p1, p2, W[0], W[1], W[2]);
    const double vy = dot3_seq(p0, p1, p2, W[3], W[4], W[5]);
    const double vz = dot3_seq(p0, p1, p2, W[6], W[7], W[8]);
    phi = atan2(vy, __dsqrt_rn(add(mul(vx, vx), mul(vz, vz))));
  }
  if (A.dbg && lane == 0) A.dbg[blockIdx.x * 16 + wid] = clock64() - t_d0;  // chains done
  if (cov_lane) {
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) s_cov[wid >> 1][3 * r + c][lane] = V[r][c];
    s_cov[wid >> 1][9][lane] = phi;
  }
  __syncthreads();
  if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 8] = clock64() - t_d0;
  if (!cov_lane) {
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) V[r][c] = s_cov[wid >> 1][3 * r + c][lane];
    phi = s_cov[wid >> 1][9][lane];
  }
  if (valid && !cov_lane) {
    // cov2d = J V J^T (rasterizer.py:92-95), J row 0 has J01 = 0
    double JV0[3], JV1[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      JV0[c] = add(mul(J00, V[0][c]), mul(J02, V[2][c]));
      JV1[c] = add(add(mul(J10, V[0][c]), mul(J11, V[1][c])), mul(J12, V[2][c]));
    }
    double c00 = add(mul(JV0[0], J00), mul(JV0[2], J02));
    double c01 = add(add(mul(JV0[0], J10), mul(JV0[1], J11)), mul(JV0[2], J12));
    double c10 = add(mul(JV1[0], J00), mul(JV1[2], J02));
    double c11 = add(add(mul(JV1[0], J10), mul(JV1[1], J11)), mul(JV1[2], J12));
    double a = add(c00, COV2D_REG);
    double b = mul(0.5, add(c01, c10));
    double c = add(c11, COV2D_REG);
    double det = sub(mul(a, c), mul(b, b));
    double ry = mul(FOOTPRINT_SIGMA, __dsqrt_rn(fmax(c, 0.0)));
    double rxr = mul(FOOTPRINT_SIGMA, __dsqrt_rn(a));
    keep = keep && (add(my, ry) >= 0.0) && (sub(my, ry) <= (double)A.gc.h);


    // tile rectangle (rasterizer.py:117-141)
    const int ntx = A.gc.ntx, nty = A.gc.nty;
    const double wd = (double)A.gc.w;
    int y0 = 0, y1 = -1, a0 = 0, a1 = -1, b0 = 0, b1 = -1, npairs = 0;
    if (keep) {
      double fy0 = floor(sub(sub(my, ry), 0.5) / 16.0);
      double fy1 = floor(add(add(my, ry), 0.5) / 16.0);
      y0 = (int)fmin(fmax(fy0, 0.0), (double)(nty - 1));
      y1 = (int)fmin(fmax(fy1, 0.0), (double)(nty - 1));
      double lo = sub(sub(mx, rxr), 0.5);
      {  // np.mod
        double m = fmod(lo, wd);
        if (m != 0.0) {
          if ((wd < 0.0) != (m < 0.0)) m = add(m, wd);
        } else {
          m = 0.0;
        }
        lo = m;
      }
      double span = add(mul(2.0, rxr), 1.0);
      if (span >= wd) {
        a0 = 0;
        a1 = ntx - 1;
      } else {
        double hi = add(lo, span);
        a0 = (int)np_floor_div16(lo);
        if (hi < wd) {
          a1 = (int)np_floor_div16(hi);
        } else {
          a1 = ntx - 1;
          b0 = 0;
          b1 = (int)np_floor_div16(sub(hi, wd));
        }
      }
      npairs = (y1 - y0 + 1) * ((a1 - a0 + 1) + (b1 - b0 + 1));
    }

    uint64_t k = keep ? (uint64_t)__double_as_longlong(depth) : ~0ULL;
    A.key[i] = k;
    A.rec32[2 * i] = make_float4((float)mx, (float)my, (float)(c / det), (float)(-b / det));
    A.rec32[2 * i + 1] = make_float4((float)(a / det), (float)opac, (float)theta, (float)phi);
    if (A.rrec) {  // f32 raster record (common.cuh "f32 raster alpha")
      const double ca_ = c / det, cb_ = -b / det, cc_ = a / det;
      float xr = -1.f, yr = -1.f;
      if (Q > 0.0) {  // 255 opacity > 1
        xr = (float)(sqrt(Q * a) * (1.0 + 1e-4) + 0.01);
        yr = (float)(sqrt(Q * fmax(c, 0.0)) * (1.0 + 1e-4) + 0.01);
      }
      A.rrec[2 * i] = make_float4((float)mx, (float)my, (float)(-0.5 * LOG2E * ca_),
                                  (float)(-LOG2E * cb_));
      // opacity enters the f32 raster as log2(opacity), folded into the
      // exponent: alpha_raw = 2^(q' + log2 opacity)
      A.rrec[2 * i + 1] = make_float4((float)(-0.5 * LOG2E * cc_), log2op, xr, yr);
    }
    if (A.rec64) {
      double* r = A.rec64 + 8 * i;
      r[0] = mx;
      r[1] = my;
      r[2] = c / det;
      r[3] = -b / det;
      r[4] = a / det;
      r[5] = opac;
      r[6] = theta;
      r[7] = phi;
    }
    A.live[i] = 0;  // K4 pass A flags the Gaussians with a contribution
    A.live_list[i] = -1;  // entries appear as pass A appends them (streaming K1)
    A.rect[i] = make_int4(y0 | (y1 << 16), (a0 & 0xffff) | (a1 << 16), (b0 & 0xffff) | (b1 << 16),
                          npairs);
    if (keep && npairs <= A.bin_small) {  // larger rectangles: whole warp, below
      for (int ty = y0; ty <= y1; ++ty) {
        for (int tx = a0; tx <= a1; ++tx) atomicAdd(s_tiles + ty * ntx + tx, 1);
        for (int tx = b0; tx <= b1; ++tx) atomicAdd(s_tiles + ty * ntx + tx, 1);
      }
    }
    kept_out = keep;
    np_out = npairs;
    packed = ((uint64_t)(uint32_t)((k - DEPTH_KEY_BASE) >> COARSE_SHIFT) << 32) | (uint32_t)i;
    ry0 = y0;
    ry1 = y1;
    ra0 = a0;
    ra1 = a1;
    rb0 = b0;
    rb1 = b1;
  }
  // launched as a dependent of the frame-clearing kernel: the f64 chains
  // above overlap it; the first global counter update comes after this
  pdl_wait();
  {
    unsigned kept_warp = __reduce_add_sync(0xffffffffu, kept_out ? 1u : 0u);
    if ((threadIdx.x & 31) == 0 && kept_warp) atomicAdd(A.counters + GSPARC_CNT_KEPT, (int)kept_warp);
  }
  // rectangles of more than bin_small tiles are expanded by the whole warp,
  // one Gaussian at a time, a tile per lane (a per-thread loop would hold
  // the warp for the largest rectangle's count of dependent atomics)
  const unsigned bigm = __ballot_sync(0xffffffffu, kept_out && np_out > A.bin_small);
  for_big_tiles(bigm, ry0, ry1, ra0, ra1, rb0, rb1, packed, lane, A.gc.ntx,
                [&](int t, uint64_t) { atomicAdd(s_tiles + t, 1); });
  // this CTA's pair count: per-warp sums now, reserved in the global pair
  // buffer (one returning atomic) while the tile scan runs
  __shared__ int s_wnp[PREP_T / 32], s_wt[PREP_T / 32], s_total;
  {
    const int wnp = __reduce_add_sync(0xffffffffu, kept_out ? np_out : 0);
    if (lane == 0) s_wnp[threadIdx.x >> 5] = wnp;
  }
  __syncthreads();
  if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 9] = clock64() - t_d0;  // rect+hist
  bool fits;
  if (ntiles <= PREP_T) {
    // one tile per thread: warp scan of the histogram, warp totals in shared
    // memory, one barrier (shared with the reservation's broadcast)
    const int w = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
      int total = 0;
#pragma unroll
      for (int k = 0; k < PREP_T / 32; ++k) total += s_wnp[k];
      const int base = total ? atomicAdd(A.counters + GSPARC_CNT_PAIRS, total) : 0;
      s_base = base;
      s_total = total;
      if ((int64_t)base + total > A.capacity) A.counters[GSPARC_CNT_OVERFLOW] = 1;
    }
    const int t = threadIdx.x;
    const int v = t < ntiles ? s_tiles[t] : 0;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane == 31) s_wt[w] = inc;
    __syncthreads();
    int pre = 0;
#pragma unroll
    for (int k = 0; k < PREP_T / 32; ++k) pre += k < w ? s_wt[k] : 0;
    if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 10] = clock64() - t_d0;
    const int base = s_base;
    fits = (int64_t)base + s_total <= A.capacity;
    // segment slot = this CTA's index (no returning atomics); empty
    // segments have length 0
    if (t < ntiles) {
      const int off = base + pre + inc - v;
      if (v) atomicAdd(A.tile_count + t, v);
      if (fits) A.seg[(int64_t)t * A.seg_stride + blockIdx.x] = make_int2(off, v);
      s_off[t] = off;
    }
    __syncthreads();
  } else {
    block_exclusive_scan(s_tiles, s_off, ntiles, s_tmp);  // ends with a barrier
    if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 10] = clock64() - t_d0;
    const int total = s_off[ntiles];
    if (threadIdx.x == 0) {
      const int base = total ? atomicAdd(A.counters + GSPARC_CNT_PAIRS, total) : 0;
      s_base = base;
      if ((int64_t)base + total > A.capacity) A.counters[GSPARC_CNT_OVERFLOW] = 1;
    }
    __syncthreads();
    const int base = s_base;
    fits = (int64_t)base + total <= A.capacity;
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) {
      const int v = s_tiles[t];
      if (v) atomicAdd(A.tile_count + t, v);
      if (fits) A.seg[(int64_t)t * A.seg_stride + blockIdx.x] = make_int2(base + s_off[t], v);
      s_off[t] += base;
    }
    __syncthreads();
  }
  if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 11] = clock64() - t_d0;
  if (fits)
    for_big_tiles(bigm, ry0, ry1, ra0, ra1, rb0, rb1, packed, lane, A.gc.ntx,
                  [&](int t, uint64_t v) { A.stage[atomicAdd(s_off + t, 1)] = v; });
  if (kept_out && fits && np_out <= A.bin_small) {
    const int ntx = A.gc.ntx;
    for (int ty = ry0; ty <= ry1; ++ty) {
      for (int tx = ra0; tx <= ra1; ++tx) {
        const int t = ty * ntx + tx;
        A.stage[atomicAdd(s_off + t, 1)] = packed;
      }
      for (int tx = rb0; tx <= rb1; ++tx) {
        const int t = ty * ntx + tx;
        A.stage[atomicAdd(s_off + t, 1)] = packed;
      }
    }
  }
  if (A.dbg) {
    __syncthreads();
    if (threadIdx.x == 0) {
      A.dbg[blockIdx.x * 16 + 12] = clock64() - t_d0;
      A.dbg[blockIdx.x * 16 + 15] = gtimer();
    }
  }
}

// Clears the frame's counters | tile_count | tile_cursor (back to back) and
// lets K2 start at once (K2 waits for it before its first counter update).
__global__ void __launch_bounds__(256) k_clear_frame(int* p, int n) {
  pdl_trigger();
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0;
}

int launch_preprocess(const gsparc_cloud& cloud, const gsparc_view& view,
                      const gsparc_frame_layout& L, char* frame, cudaStream_t st) {
  PrepArgs A;
  A.cloud = cloud;
  for (int k = 0; k < 3; ++k) A.pose.rx[k] = view.rx[k];
  for (int k = 0; k < 9; ++k) A.pose.W[k] = view.rotation[k];
  A.gc = make_geo_const(L.width, L.height);
  A.key = (uint64_t*)(frame + L.off_key);
  A.rec32 = (float4*)(frame + L.off_rec32);
  A.rec64 = L.dtype == GSPARC_F64 ? (double*)(frame + L.off_rec64) : nullptr;
  A.rrec = L.dtype == GSPARC_F32 ? (float4*)(frame + L.off_rrec) : nullptr;
  A.rect = (int4*)(frame + L.off_rect);
  A.counters = (int*)(frame + L.off_counters);
  A.tile_count = (int*)(frame + L.off_tile_count);
  A.tile_cursor = (int*)(frame + L.off_tile_cursor);
  A.live = (int*)(frame + L.off_live);
  A.live_list = (int*)(frame + L.off_live_list);
  A.stage = (uint64_t*)(frame + L.off_stage);
  A.seg = (int2*)(frame + L.off_seg);
  A.capacity = L.pair_capacity;
  A.seg_stride = (int)L.seg_stride;
  A.dbg = experiment_env("GSPARC_PREP_DBG") ? dbg_rows(3) : nullptr;  // experiments only
  A.bin_small = experiment_env("GSPARC_BIN_SMALL") ? atoi(experiment_env("GSPARC_BIN_SMALL")) : 40;
  // counters | tile_count | tile_cursor are laid out back to back
  const int64_t zero_end = L.off_tile_cursor + (int64_t)sizeof(int) * L.ntiles;
  if (L.off_tile_count < L.off_counters || L.off_tile_cursor < L.off_tile_count) {
    set_error("preprocess: unexpected frame layout");
    return GSPARC_ERR_ARG;
  }
  static const bool pdl = !getenv("GSPARC_NO_PDL") && !experiment_env("GSPARC_NO_PDL_K2");
  if (pdl) {
    const int nz = (int)((zero_end - L.off_counters) / (int64_t)sizeof(int));
    k_clear_frame<<<1, 256, 0, st>>>((int*)(frame + L.off_counters), nz);
    GS_TRY(check_launch("k_clear_frame"));
  } else if (cudaMemsetAsync(frame + L.off_counters, 0, zero_end - L.off_counters, st) !=
             cudaSuccess) {
    return check_launch("preprocess memset");
  }
  if (cloud.n > 0) {
    const int blocks = (int)((cloud.n + PREP_G - 1) / PREP_G);
    if (blocks > L.seg_stride) {
      set_error("preprocess: frame planned for fewer Gaussians");
      return GSPARC_ERR_ARG;
    }
    const size_t smem = sizeof(int) * (2 * (size_t)L.ntiles + 1 + PREP_T / 32 + 1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(PREP_T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    if (pdl) {
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
    }
    cudaLaunchKernelEx(&cfg, k_preprocess, A);
  }
  return check_launch("k_preprocess");
}

}  // namespace gs
