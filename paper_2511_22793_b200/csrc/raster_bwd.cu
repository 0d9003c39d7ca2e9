// K5: per-tile backward of the compositing, back to front.
// Replaces the per-tile loop of rasterizer.rasterize_backward
// (rasterizer.py:286-326).  Instead of the reference's f64 front-to-back
// cumprod + reverse cumsum, each pixel walks its included range backwards
// from the stored final transmittance (T_before = T_after / (1 - alpha),
// SPEC.md rasterize_backward "re-deriving each T_i from stored final
// transmittance"), keeping the suffix sum  S_k = sum_{j>k} wgt_j (u . c_j)
// exactly as accumulated, which avoids the cancellation of total - prefix.
//
// Gradients are linear in dL, so channels are split into chunks of CB
// (grid.y); every chunk contributes its share of dL/dalpha to the geometric
// accumulators.  Per batch:
//   * scan: per pixel, d alpha, d(sigma g), d conic, d mean2d (reduced over
//     the warp by shuffles, over the CTA in shared memory);
//   * dL/dcoef[k, c] = sum_p wgt[k,p] u[p,c] as a shared-memory GEMM over the
//     tile's 256 pixels;
//   * one global atomicAdd per (Gaussian, tile, value).
#include "common.cuh"
#include "kernels.cuh"

namespace gs {

struct BwdArgs {
  const uint64_t* pairs;
  const int* tile_start;
  const int* wstop;  // visited prefix per 32-pixel warp (forward AUX pass)
  const float4* rec32;
  const float4* rrec;  // f32 raster record (f32 frames: same alpha as K4)
  const double* rec64;
  const void* coef;
  const void* dL;  // [B,h,w,C]
  const void* T_final;
  const int* last;
  void* gcoef;  // [n, Cp]
  void* ggeo;   // [n, 8]
  void* dgc;    // deterministic: [pairs, nsub, Cp] partials
  void* dgg;    // deterministic: [pairs, nsub, nchunks, 6] partials
  const int* counters;
  int64_t Cp;
  int C, nchunks;
  int w, h, ntx, sr, nsub;
};

template <typename R, int CB, int NB, bool DET>
__global__ void __launch_bounds__(256) k_raster_bwd(BwdArgs A) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int P = blockDim.x;              // pixels of this sub-tile
  const int UP = P + 1;                  // s_u pitch: the GEMM's lanes read
                                         // different channels, same pixel
  const int WP = P + 1;                  // s_wgt pitch (GEMM rows of 4 entries)
  R* s_u = (R*)smraw;                    // [CB][P + 1]
  R* s_wgt = s_u + CB * UP;              // [NB][P + 1]
  R* s_coef = s_wgt + NB * WP;           // [NB][CB]
  R* s_red = s_coef + NB * CB;           // [NB][6] (DET: [NB][8 warps][6])
  Rec<R>* s_rec = (Rec<R>*)(s_red + NB * 6 * (DET ? 8 : 1));  // [NB]
  int* s_idx = (int*)(s_rec + NB);       // [NB]; bit 31: first copy of a seam duplicate
  float4* s_fr = (float4*)(((uintptr_t)(s_idx + NB) + 15) & ~(uintptr_t)15);  // [NB][2] (f32)

  if (A.counters[GSPARC_CNT_OVERFLOW]) return;
  const int sidx = blockIdx.x, chunk = blockIdx.y;
  const int tile = sidx / A.nsub, part = sidx - tile * A.nsub;
  const int tid = threadIdx.x, pix = tid;
  const int lane = tid & 31;
  const int tx_ = tile % A.ntx, ty = tile / A.ntx;
  const int px = tx_ * TILE + (pix & (TILE - 1));
  const int py = ty * TILE + part * A.sr + pix / TILE;
  const bool inside = px < A.w && py < A.h;
  const int start = A.tile_start[tile], tile_end = A.tile_start[tile + 1];
  const int nvisit = part_nvisit(A.wstop, tile, part, A.nsub);
  if (nvisit == 0) return;
  const int chunk_base = chunk * CB;
  const R pcx = (R)px + R(0.5), pcy = (R)py + R(0.5);
  const R wR = (R)A.w, half_w = (R)(A.w / 2.0);
  const R amax = sizeof(R) == 4 ? R(ALPHA_MAX_F) : R(ALPHA_MAX);

  R u[CB];
  const R* dL = (const R*)A.dL;
#pragma unroll
  for (int c = 0; c < CB; ++c) {
    const int64_t cc = chunk_base + c;
    R v = R(0);
    if (inside && cc < A.Cp) {
      const int64_t b = cc / A.C, ch = cc - b * A.C;
      v = dL[((b * A.h + py) * (int64_t)A.w + px) * A.C + ch];
    }
    u[c] = v;
    s_u[c * UP + pix] = v;
  }
  const int p = py * A.w + px;
  R T = inside ? ((const R*)A.T_final)[p] : R(1);
  const int lastp = inside ? A.last[p] : 0;
  R suffix = R(0);

  R* gcoef = (R*)A.gcoef;
  R* ggeo = (R*)A.ggeo;
  const R* coef = (const R*)A.coef;

  for (int bend = nvisit; bend > 0; bend -= NB) {
    const int b0 = bend > NB ? bend - NB : 0;
    const int nb = bend - b0;
    __syncthreads();
    if (tid < nb) {
      const uint32_t idx = (uint32_t)A.pairs[start + b0 + tid];
      // the reference accumulates per tile with g[rows] += ... (fancy
      // indexing, rasterizer.py:302-326): for a Gaussian listed twice in a
      // tile (seam duplicate) only the later copy's row survives -- drop the
      // first copy's contributions the same way
      const int kn = start + b0 + tid + 1;
      const bool first_dup = kn < tile_end && (uint32_t)A.pairs[kn] == idx;
      s_idx[tid] = (int)idx | (first_dup ? (int)0x80000000 : 0);
      if constexpr (sizeof(R) == 4) {
        // conic recovered from the pre-scaled exponent coefficients
        const float4 f0 = __ldg(A.rrec + 2 * (size_t)idx), f1 = __ldg(A.rrec + 2 * (size_t)idx + 1);
        s_fr[2 * tid] = f0;
        s_fr[2 * tid + 1] = f1;
        const float k2 = (float)(-2.0 / LOG2E), k1 = (float)(-1.0 / LOG2E);
        s_rec[tid] = Rec<R>{f0.x, f0.y, f0.z * k2, f0.w * k1, f1.x * k2, exp2f(f1.y)};
      } else {
        s_rec[tid] = load_rec_t<R>(A.rec32, A.rec64, idx);
      }
    }
    for (int e = tid; e < nb * 6 * (DET ? 8 : 1); e += blockDim.x) s_red[e] = R(0);
    __syncthreads();
    // the batch's coef rows: indices from shared memory, every load of a
    // thread issued before its stores (one latency instead of one per row)
    {
      constexpr int PER = (NB * CB + 63) / 64;  // elements per thread at P >= 64
      R cv[PER];
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int e = tid + k * blockDim.x;
        cv[k] = R(0);
        if (e < nb * CB) {
          const int j = e / CB, c = e - j * CB;
          const int64_t cc = chunk_base + c;
          const uint32_t idx = (uint32_t)(s_idx[j] & 0x7fffffff);
          if (cc < A.Cp) cv[k] = coef[(int64_t)idx * A.Cp + cc];
        }
      }
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int e = tid + k * blockDim.x;
        if (e < nb * CB) s_coef[e] = cv[k];
      }
      for (int e = tid + PER * blockDim.x; e < nb * CB; e += blockDim.x) {  // P < 64
        const int j = e / CB, c = e - j * CB;
        const int64_t cc = chunk_base + c;
        const uint32_t idx = (uint32_t)(s_idx[j] & 0x7fffffff);
        s_coef[e] = cc < A.Cp ? coef[(int64_t)idx * A.Cp + cc] : R(0);
      }
    }
    __syncthreads();
    for (int j = nb - 1; j >= 0; --j) {
      const int k = b0 + j;
      R wgt = R(0), g_sig = R(0), gc0 = R(0), gc1 = R(0), gc2 = R(0), gm0 = R(0), gm1 = R(0);
      if (k < lastp) {
        const Rec<R> r = s_rec[j];
        AlphaOut<R> a;
        if constexpr (sizeof(R) == 4) {
          const FastAlpha f = fast_alpha_full(pcx, pcy, s_fr[2 * j], s_fr[2 * j + 1], wR,
                                              1.0f / wR);
          a = AlphaOut<R>{f.alpha, f.raw, f.g, f.dx, f.dy};
        } else {
          a = pixel_alpha<R>(pcx, pcy, r.mx, r.my, r.ca, r.cb, r.cc, r.op, wR, half_w);
        }
        if (a.alpha > R(0)) {
          const R om = R(1) - a.alpha;
          // one correctly rounded reciprocal for both divisions by (1 - alpha)
          R rom;
          if constexpr (sizeof(R) == 4) rom = __frcp_rn(om);
          else rom = R(1) / om;
          const R Tb = sizeof(R) == 4 ? T * rom : T / om;
          wgt = Tb * a.alpha;
          R uc = R(0);
          const R* cf = s_coef + j * CB;
          if constexpr (sizeof(R) == 4 && CB % 8 == 0) {
            // FFMA2 with 4 independent accumulators (8 partial sums): a
            // 4x shorter dependent chain than one running sum
            float2 a2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                            make_float2(0.f, 0.f)};
            const float2* cf2 = reinterpret_cast<const float2*>(cf);
#pragma unroll
            for (int c = 0; c < CB / 2; ++c)
              a2[c & 3] = ffma2(make_float2(u[2 * c], u[2 * c + 1]), cf2[c], a2[c & 3]);
            uc = ((a2[0].x + a2[0].y) + (a2[1].x + a2[1].y)) + ((a2[2].x + a2[2].y) + (a2[3].x + a2[3].y));
          } else if constexpr (sizeof(R) == 4 && CB % 2 == 0) {  // FFMA2: even/odd partial sums
            float2 a2 = make_float2(0.f, 0.f);
            const float2* cf2 = reinterpret_cast<const float2*>(cf);
#pragma unroll
            for (int c = 0; c < CB / 2; ++c)
              a2 = ffma2(make_float2(u[2 * c], u[2 * c + 1]), cf2[c], a2);
            uc = a2.x + a2.y;
          } else {
#pragma unroll
            for (int c = 0; c < CB; ++c) uc += u[c] * cf[c];
          }
          const R dA = Tb * uc - (sizeof(R) == 4 ? suffix * rom : suffix / om);
          suffix += wgt * uc;
          T = Tb;
          if (a.raw < amax) {
            g_sig = dA * a.g;
            const R dq = R(-0.5) * (dA * r.op) * a.g;
            gc0 = dq * a.dx * a.dx;
            gc1 = dq * a.dx * a.dy;
            gc2 = dq * a.dy * a.dy;
            gm0 = -(dq * R(2) * (r.ca * a.dx + r.cb * a.dy));
            gm1 = -(dq * R(2) * (r.cb * a.dx + r.cc * a.dy));
          }
        }
      }
      s_wgt[j * WP + pix] = wgt;
      const bool any = __any_sync(0xffffffffu, g_sig != R(0) || gc0 != R(0) || gc2 != R(0) ||
                                                   gm0 != R(0) || gm1 != R(0));
      if (any) {
        // reduce-scatter of the 6 values (padded to 8) over the warp: 9
        // shuffles instead of 6 x 5; lane 4f (f < 6) ends up with field f
        R v[8] = {gc0, gc1, gc2, gm0, gm1, g_sig, R(0), R(0)};
        {
          const bool hi = lane & 16;
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // keep 4 (by lane bit 4), send 4
            const R send = hi ? v[k] : v[k + 4];
            const R keep = hi ? v[k + 4] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
          }
        }
        {
          const bool hi = lane & 8;
#pragma unroll
          for (int k = 0; k < 2; ++k) {  // keep 2 (by lane bit 3), send 2
            const R send = hi ? v[k] : v[k + 2];
            const R keep = hi ? v[k + 2] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
          }
        }
        {
          const bool hi = lane & 4;
          const R send = hi ? v[0] : v[1];
          const R keep = hi ? v[1] : v[0];
          v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        }
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        const int f = lane >> 2;  // (bit4, bit3, bit2) -> field
        if ((lane & 3) == 0 && f < 6) {
          if constexpr (DET) {  // one slot per warp, summed in warp order
            s_red[(j * 8 + (tid >> 5)) * 6 + f] = v[0];
          } else {
            atomicAdd(s_red + j * 6 + f, v[0]);
          }
        }
      }
    }
    __syncthreads();
    // dL/dcoef for this batch: [nb x CB] = wgt[nb x P] . u[P x CB], register
    // tiles of 4 entries x CT channels (12 shared loads per 32 FMAs)
    {
      constexpr int JT = 4, CT = CB < 8 ? CB : 8;
      constexpr int NCT = CB / CT, NTILE = (NB / JT) * NCT;
      for (int tile = tid; tile < NTILE; tile += blockDim.x) {
        const int j0 = (tile / NCT) * JT, c0 = (tile % NCT) * CT;
        if (j0 >= nb) continue;
        R acc[JT][CT];
#pragma unroll
        for (int a = 0; a < JT; ++a)
#pragma unroll
          for (int b = 0; b < CT; ++b) acc[a][b] = R(0);
        const R* wr = s_wgt + j0 * WP;
        const R* ur = s_u + c0 * UP;
#pragma unroll 4
        for (int q = 0; q < P; ++q) {
          R wv[JT], uv[CT];
#pragma unroll
          for (int a = 0; a < JT; ++a) wv[a] = wr[a * WP + q];
#pragma unroll
          for (int b = 0; b < CT; ++b) uv[b] = ur[b * UP + q];
          if constexpr (sizeof(R) == 4 && CT % 2 == 0) {  // FFMA2 over channel pairs
#pragma unroll
            for (int a = 0; a < JT; ++a)
#pragma unroll
              for (int b = 0; b < CT; b += 2) {
                const float2 r2 = ffma2(make_float2(wv[a], wv[a]), make_float2(uv[b], uv[b + 1]),
                                        make_float2(acc[a][b], acc[a][b + 1]));
                acc[a][b] = r2.x;
                acc[a][b + 1] = r2.y;
              }
          } else {
#pragma unroll
            for (int a = 0; a < JT; ++a)
#pragma unroll
              for (int b = 0; b < CT; ++b) acc[a][b] += wv[a] * uv[b];
          }
        }
#pragma unroll
        for (int a = 0; a < JT; ++a) {
          const int j = j0 + a;
          if (j >= nb) break;
          const int sj = s_idx[j];
#pragma unroll
          for (int b = 0; b < CT; ++b) {
            const int64_t cc = chunk_base + c0 + b;
            if (cc >= A.Cp) continue;
            R v = sj < 0 ? R(0) : acc[a][b];  // first copy of a seam duplicate
            if constexpr (DET) {
              const int64_t k = start + b0 + j;  // list position
              ((R*)A.dgc)[(k * A.nsub + part) * A.Cp + cc] = v;
            } else {
              if (v != R(0)) atomicAdd(gcoef + (int64_t)sj * A.Cp + cc, v);
            }
          }
        }
      }
    }
    for (int o = tid; o < nb * 6; o += blockDim.x) {
      if constexpr (DET) {
        const int j = o / 6, f = o % 6;
        const int nw = P >> 5;
        R v = R(0);
        for (int w = 0; w < nw; ++w) v += s_red[(j * 8 + w) * 6 + f];
        if (s_idx[j] < 0) v = R(0);  // first copy of a seam duplicate
        const int64_t k = start + b0 + j;
        ((R*)A.dgg)[((k * A.nsub + part) * A.nchunks + chunk) * 6 + f] = v;
      } else {
        const R v = s_red[o];
        const int sj = s_idx[o / 6];
        if (v != R(0) && sj >= 0) atomicAdd(ggeo + (int64_t)sj * 8 + (o % 6), v);
      }
    }
  }
}

template <typename R, int CB, int NB, bool DET>
static int launch_bwd_cfg(const BwdArgs& A, int ntiles, cudaStream_t st) {
  const int P = TILE * A.sr;
  constexpr size_t RED = NB * 6 * (DET ? 8 : 1);
  const size_t smem_max = sizeof(R) * ((size_t)CB * 257 + (size_t)NB * 257 + NB * CB + RED) +
                          sizeof(Rec<R>) * NB + sizeof(int) * NB + 32 * NB + 32;
  const size_t smem = sizeof(R) * ((size_t)CB * (P + 1) + (size_t)NB * (P + 1) + NB * CB + RED) +
                      sizeof(Rec<R>) * NB + sizeof(int) * NB + 32 * NB + 32;
  auto kern = k_raster_bwd<R, CB, NB, DET>;
  static bool attr_set = false;  // one per instantiation; keeps capture clean
  if (!attr_set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
    attr_set = true;
  }
  const int chunks = (int)((A.Cp + CB - 1) / CB);
  kern<<<dim3(ntiles * A.nsub, chunks), P, smem, st>>>(A);
  return check_launch("k_raster_bwd");
}

// Deterministic mode, step 2: per Gaussian (one warp), sum the partials of
// every list entry it owns in a fixed order -- tiles in (ty, tx) order over
// the a segment then the b-only tiles (rasterizer.py:117-141), the seam
// duplicate right after its first copy, then sub-tiles, then channel chunks.
// An entry's list position is found by binary search on (f64 key, index),
// the order the tile lists are sorted in.
struct RedArgs {
  const uint64_t* pairs;
  const int* tile_start;
  const int* wstop;
  const uint64_t* key;
  const int4* rect;
  const void* dgc;
  const void* dgg;
  void* gcoef;
  void* ggeo;
  int64_t n, Cp;
  int nchunks, ntx, nsub, ntiles;
  const int* inv;  // [n][ntiles] list positions per tile slot (K3)
};

constexpr int RED_MAXT = DET_MAXT;  // tile slots staged in shared memory per pass

template <typename R>
__global__ void __launch_bounds__(256) k_bwd_reduce(RedArgs A) {
  __shared__ int s_pos[8][RED_MAXT];   // list position per enumerated tile
  __shared__ unsigned char s_vis[8][RED_MAXT];  // bit 4 copy + sub-tile: partial visited
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * 8 + warp;
  if (i >= A.n) return;
  R* gc = (R*)A.gcoef + i * A.Cp;
  R* gg = (R*)A.ggeo + i * 8;
  const uint64_t ki = A.key[i];
  int ntile = 0, na = 0, nbo = 0, y0 = 0, a0 = 0, b1 = -1;
  if (ki != ~0ULL) {
    const int4 r = A.rect[i];
    y0 = r.x & 0xffff;
    const int y1 = r.x >> 16;
    a0 = r.y & 0xffff;
    const int a1 = r.y >> 16;
    b1 = r.z >> 16;  // b segment is [0, b1] (wrapped), empty if b1 < 0
    na = a1 - a0 + 1;
    nbo = b1 >= 0 ? min(b1, a0 - 1) + 1 : 0;  // b tiles outside the a range
    ntile = (y1 - y0 + 1) * (na + nbo);       // <= ntiles (K3's table stride)
  }
  const R* dgc = (const R*)A.dgc;
  const R* dgg = (const R*)A.dgg;
  // slots are taken RED_MAXT at a time (a rectangle can span every tile of
  // a wide frame); each pass adds its fixed-order sum to the running one,
  // so the summation order is canonical for a given frame
  for (int j0 = 0; j0 == 0 || j0 < ntile; j0 += RED_MAXT) {
    const int nj = min(ntile - j0, RED_MAXT);
    __syncwarp();
    for (int jj = lane; jj < nj; jj += 32) {
      const int j = j0 + jj;
      const int ty = y0 + j / (na + nbo), rj = j % (na + nbo);
      const int tx = rj < na ? a0 + rj : rj - na;
      const int t = ty * A.ntx + tx;
      // list position of (Gaussian i, tile t): recorded by K3 when it placed
      // the entry (the first copy of a seam duplicate)
      const int lo = __ldg(A.inv + i * A.ntiles + j);
      const bool twice = rj < na && b1 >= 0 && tx <= b1;  // seam duplicate
      s_pos[warp][jj] = lo;
      // which (copy, sub-tile) partials exist: K5 wrote those inside each
      // sub-tile's visited prefix (wstop, per 32-pixel warp)
      const int ts = A.tile_start[t];
      unsigned vis = 0;
      for (int copy = 0; copy <= (twice ? 1 : 0); ++copy)
        for (int p = 0; p < A.nsub; ++p) {
          const int nv = part_nvisit(A.wstop, t, p, A.nsub);
          if (lo + copy - ts < nv) vis |= 1u << (4 * copy + p);
        }
      s_vis[warp][jj] = (unsigned char)vis;
    }
    __syncwarp();
    // sums in the fixed order (tile slot, copy, sub-tile[, chunk]); the (up to
    // 8) partials of a slot are loaded together
    for (int64_t c0 = 0; c0 < A.Cp; c0 += 32) {
      const int64_t cc = c0 + lane;
      if (cc < A.Cp) {
        R acc = R(0);
        // 4 slots' partials in flight per round (the sum stays in slot order)
        for (int jb = 0; jb < nj; jb += 4) {
          R v[4][8];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int jj = jb + u;
            const unsigned vis = jj < nj ? s_vis[warp][jj] : 0u;
            const int64_t k0 = jj < nj ? s_pos[warp][jj] : 0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              v[u][q] = ((vis >> q) & 1u)
                            ? dgc[((k0 + (q >> 2)) * A.nsub + (q & 3)) * A.Cp + cc]
                            : R(0);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned vis = jb + u < nj ? s_vis[warp][jb + u] : 0u;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if ((vis >> q) & 1u) acc += v[u][q];
          }
        }
        gc[cc] = j0 == 0 ? acc : gc[cc] + acc;
      }
    }
    if (lane < 8) {
      R acc = R(0);
      if (lane < 6 && A.nchunks == 1) {
        // one channel chunk: 4 slots' partials in flight per round, summed
        // in the same (slot, copy/sub-tile) order as the general loop
        for (int jb = 0; jb < nj; jb += 4) {
          R v[4][8];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int jj = jb + u;
            const unsigned vis = jj < nj ? s_vis[warp][jj] : 0u;
            const int64_t k0 = jj < nj ? s_pos[warp][jj] : 0;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              v[u][q] = ((vis >> q) & 1u)
                            ? dgg[((k0 + (q >> 2)) * A.nsub + (q & 3)) * 6 + lane]
                            : R(0);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const unsigned vis = jb + u < nj ? s_vis[warp][jb + u] : 0u;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if ((vis >> q) & 1u) acc += v[u][q];
          }
        }
      } else if (lane < 6) {
        for (int jj = 0; jj < nj; ++jj) {
          const int64_t k0 = s_pos[warp][jj];
          const unsigned vis = s_vis[warp][jj];
          for (int q = 0; q < 8; ++q)
            if ((vis >> q) & 1u)
              for (int ch = 0; ch < A.nchunks; ++ch)
                acc += dgg[(((k0 + (q >> 2)) * A.nsub + (q & 3)) * A.nchunks + ch) * 6 + lane];
        }
      }
      gg[lane] = j0 == 0 ? acc : gg[lane] + acc;
    }
  }
}

int launch_raster_backward(const gsparc_frame_layout& L, char* frame, int n_tx, int C,
                           const void* dL, bool det, cudaStream_t st) {
  BwdArgs A;
  A.pairs = (const uint64_t*)(frame + L.off_pairs);
  A.tile_start = (const int*)(frame + L.off_tile_start);
  A.wstop = (const int*)(frame + L.off_wstop);
  A.rec32 = (const float4*)(frame + L.off_rec32);
  A.rrec = (const float4*)(frame + L.off_rrec);
  A.rec64 = (const double*)(frame + L.off_rec64);
  A.coef = frame + L.off_coef;
  A.dL = dL;
  A.T_final = frame + L.off_T;
  A.last = (const int*)(frame + L.off_last);
  A.gcoef = frame + L.off_gcoef;
  A.ggeo = frame + L.off_ggeo;
  A.dgc = frame + L.off_det_gcoef;
  A.dgg = frame + L.off_det_ggeo;
  A.counters = (const int*)(frame + L.off_counters);
  A.Cp = (int64_t)n_tx * C;
  A.C = C;
  A.w = L.width;
  A.h = L.height;
  A.ntx = L.ntx;
  A.sr = forward_sub_rows(L, A.Cp);
  A.nsub = TILE / A.sr;
  const size_t esz = L.dtype == GSPARC_F64 ? 8 : 4;
  const int CB = L.dtype == GSPARC_F64 ? 4
                 : A.Cp <= 2 ? 2 : A.Cp <= 8 ? 8 : A.Cp <= 16 ? 16 : A.Cp <= 32 ? 32 : 64;
  A.nchunks = (int)((A.Cp + CB - 1) / CB);
  if (det) {
    if (A.nsub > 4 || A.nchunks > (L.channels >= 4 ? (L.channels + 3) / 4 : 1)) {
      set_error("raster_backward: deterministic partial buffers too small");
      return GSPARC_ERR_UNSUPPORTED;
    }
  } else if (cudaMemsetAsync(A.gcoef, 0, esz * (size_t)L.n * (size_t)L.channels, st) !=
                 cudaSuccess ||
             cudaMemsetAsync(A.ggeo, 0, esz * (size_t)L.n * 8, st) != cudaSuccess) {
    return check_launch("bwd memset");
  }
  int rc;
  if (raster_bwd_tc_supported(L, A.Cp)) {
    // both channel contractions on the tensor cores, one CTA per half tile
    A.nsub = 2;
    A.nchunks = 1;
    rc = launch_raster_bwd_tc(L, frame, n_tx, C, dL, det, st);
  } else if (L.dtype == GSPARC_F64) {
    rc = det ? launch_bwd_cfg<double, 4, 32, true>(A, L.ntiles, st)
             : launch_bwd_cfg<double, 4, 32, false>(A, L.ntiles, st);
  } else if (A.Cp <= 2) {
    rc = det ? launch_bwd_cfg<float, 2, 32, true>(A, L.ntiles, st)
             : launch_bwd_cfg<float, 2, 32, false>(A, L.ntiles, st);
  } else if (A.Cp <= 8) {
    rc = det ? launch_bwd_cfg<float, 8, 32, true>(A, L.ntiles, st)
             : launch_bwd_cfg<float, 8, 32, false>(A, L.ntiles, st);
  } else if (A.Cp <= 16) {
    rc = det ? launch_bwd_cfg<float, 16, 32, true>(A, L.ntiles, st)
             : launch_bwd_cfg<float, 16, 32, false>(A, L.ntiles, st);
  } else if (A.Cp <= 32) {
    rc = det ? launch_bwd_cfg<float, 32, 32, true>(A, L.ntiles, st)
             : launch_bwd_cfg<float, 32, 32, false>(A, L.ntiles, st);
  } else {  // one pass of the alpha/T walk per 64 channels
    rc = det ? launch_bwd_cfg<float, 64, 32, true>(A, L.ntiles, st)
             : launch_bwd_cfg<float, 64, 32, false>(A, L.ntiles, st);
  }
  if (rc != GSPARC_OK || !det) return rc;
  RedArgs R;
  R.pairs = A.pairs;
  R.tile_start = A.tile_start;
  R.wstop = A.wstop;
  R.key = (const uint64_t*)(frame + L.off_key);
  R.rect = (const int4*)(frame + L.off_rect);
  R.dgc = A.dgc;
  R.dgg = A.dgg;
  R.gcoef = A.gcoef;
  R.ggeo = A.ggeo;
  R.n = L.n;
  R.Cp = A.Cp;
  R.nchunks = A.nchunks;
  R.ntx = L.ntx;
  R.nsub = A.nsub;
  R.ntiles = L.ntiles;
  R.inv = (const int*)(frame + L.off_det_inv);
  const unsigned blocks = (unsigned)((L.n + 7) / 8);
  if (blocks == 0) return GSPARC_OK;
  if (L.dtype == GSPARC_F64) k_bwd_reduce<double><<<blocks, 256, 0, st>>>(R);
  else k_bwd_reduce<float><<<blocks, 256, 0, st>>>(R);
  return check_launch("k_bwd_reduce");
}

}  // namespace gs
