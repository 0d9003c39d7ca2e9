// K4: front-to-back alpha compositing over hemisphere pixels x channels.
// Replaces do_tile / _tile_alphas (rasterizer.py:169-231).
//
// Work decomposition ("lanes = list entries"): a CTA owns a 16x4-pixel
// sub-tile of a 16x16 tile (4 CTAs per tile) and streams the tile's
// depth-sorted list through shared memory in chunks of CH entries.  Each
// warp takes one pixel at a time and evaluates 32 consecutive list entries
// in its 32 lanes:
//   * alpha: branch-free pixel_alpha() in numpy's exact op order;
//   * transmittance: T_before = T_in * exclusive prefix product of (1-alpha)
//     (warp scan), the reference rule "stop at the first entry with
//     T_before < t_eps, include iff alpha > 0" via ballots
//     (rasterizer.py:209-219), wgt = T_before * alpha;
//   * per-pixel count / last / T_final, live-Gaussian marking.
// Pixels are independent work items, so every SM runs tens of warps
// regardless of how few pixels there are (the former lanes = pixels scan
// left 7 warps per SM on the 32400-pixel image).  The tree-ordered product
// rounds differently from numpy's sequential cumprod (a few ulp); the tests
// count the resulting rare threshold flips like the exp ones.
//
// Channel accumulation (ACC): for <= 4 channels the weight warp reduces
// wgt*coef over its lanes directly (SMALLC); otherwise the weights go to
// shared memory and 4 thread groups x 64 pixels accumulate CC channels
// each with coef rows staged once per chunk.
//
// Passes: AUX writes T_final / count / last / per-warp stops and the live
// list; ACC writes the image.  fused = AUX+ACC; the lazy-MLP path runs AUX,
// evaluates the MLP on the live Gaussians only, then ACC over the visited
// prefix (identical arithmetic, so ACC reproduces AUX's weights bitwise).
#include "common.cuh"
#include "kernels.cuh"

namespace gs {

struct RasterArgs {
  const uint64_t* pairs;
  const int* tile_start;
  int* wstop;              // [ntiles * 8] visited prefix per 2-row strip
  const float4* rec32;
  const double* rec64;
  const void* coef;
  int64_t Cp;  // channels per coef row (n_tx * C)
  int C;       // channels per TX (image last dim)
  void* img;
  void* T_out;
  int* count_out;
  int* last_out;
  int* live;
  int* live_list;
  int* counters;
  int w, h, ntx, ntiles;
  double t_eps;
};

constexpr int RP = 64;       // pixels per CTA (16 x 4 sub-tile)
constexpr int RWARPS = 8;    // warps per CTA
constexpr int RSLOTS = RP / RWARPS;

template <typename R>
__device__ __forceinline__ R shfl_up_r(R v, int d) {
  return __shfl_up_sync(0xffffffffu, v, d);
}
template <typename R>
__device__ __forceinline__ R shfl_r(R v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

// CH: list entries staged per chunk.  CC: channels per group (4 groups) for
// the wide accumulation, or the channel count for SMALLC (reduced by the
// weight warp itself).
template <typename R, int CH, int CC, bool AUX, bool ACC, bool SMALLC>
__global__ void __launch_bounds__(256) k_raster(RasterArgs A) {
  constexpr int G = 4;                        // accumulation groups (wide)
  constexpr int CW = SMALLC ? CC : CC * G;    // staged coef channels
  constexpr bool WIDE = ACC && !SMALLC;
  extern __shared__ __align__(16) unsigned char smraw[];
  Rec<R>* s_rec = (Rec<R>*)smraw;                          // [CH]
  int* s_idx = (int*)(s_rec + CH);                         // [CH]
  int* s_live = s_idx + CH;                                // [CH]
  R* s_coef = (R*)(((uintptr_t)(s_live + CH) + 15) & ~(uintptr_t)15);  // [CH][CW]
  R* s_w = s_coef + (ACC ? CH * CW : 0);                   // [CH][RP+1]
  __shared__ int s_done[RP];
  __shared__ int s_stop[2];

  if (A.counters[GSPARC_CNT_OVERFLOW]) return;
  const int sidx = blockIdx.x, chunk = blockIdx.y;
  const int tile = sidx >> 2, part = sidx & 3;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx_ = tile % A.ntx, ty = tile / A.ntx;
  const int start = A.tile_start[tile];
  const int end = AUX ? A.tile_start[tile + 1]
                      : start + max(A.wstop[tile * 8 + part * 2], A.wstop[tile * 8 + part * 2 + 1]);
  const bool aux_writer = AUX && chunk == 0;
  const R wR = (R)A.w, half_w = (R)(A.w / 2.0);
  const R teps = (R)A.t_eps;
  const int chunk_base = chunk * CW;

  // per-slot pixel state (uniform across the warp's lanes)
  R Tin[RSLOTS];
  int cnt[RSLOTS], last[RSLOTS];
  unsigned done_mask = 0;
  R sacc[RSLOTS][SMALLC ? CC : 1];
#pragma unroll
  for (int s = 0; s < RSLOTS; ++s) {
    Tin[s] = R(1);
    cnt[s] = 0;
    last[s] = 0;
    const int p = warp + RWARPS * s;
    const int px = tx_ * TILE + (p & 15), py = ty * TILE + part * 4 + (p >> 4);
    if (!(px < A.w && py < A.h)) done_mask |= 1u << s;
#pragma unroll
    for (int c = 0; c < (SMALLC ? CC : 1); ++c) sacc[s][c] = R(0);
  }
  // wide accumulation: thread (pix, grp)
  const int apix = tid & (RP - 1), agrp = tid >> 6;
  R acc[WIDE ? CC : 1];
#pragma unroll
  for (int c = 0; c < (WIDE ? CC : 1); ++c) acc[c] = R(0);
  if (tid < RP) s_done[tid] = 0;
  if (tid < 2) s_stop[tid] = 0;

  for (int cb = start; cb < end; cb += CH) {
    const int nch = min(CH, end - cb);
    __syncthreads();
    for (int e = tid; e < CH; e += blockDim.x) {
      if (e < nch) {
        const uint32_t idx = (uint32_t)A.pairs[cb + e];
        s_rec[e] = load_rec_t<R>(A.rec32, A.rec64, idx);
        s_idx[e] = (int)idx;
      }
      if (AUX) s_live[e] = 0;
    }
    if (ACC) {
      __syncthreads();
      const R* coef = (const R*)A.coef;
      for (int q = tid; q < CH * CW; q += blockDim.x) {
        const int e = q / CW, c = q - e * CW;
        const int64_t cc = chunk_base + c;
        R v = R(0);
        if (e < nch && cc < A.Cp) v = coef[(int64_t)s_idx[e] * A.Cp + cc];
        s_coef[q] = v;
      }
    }
    __syncthreads();
    // ---- weights: one pixel per warp; lane l holds entries e0+2l, e0+2l+1
#pragma unroll
    for (int s = 0; s < RSLOTS; ++s) {
      const int p = warp + RWARPS * s;
      const bool pdone = (done_mask >> s) & 1u;
      if (!pdone) {
        const int px = tx_ * TILE + (p & 15), py = ty * TILE + part * 4 + (p >> 4);
        const R pcx = (R)px + R(0.5), pcy = (R)py + R(0.5);
        for (int e0 = 0; e0 < nch; e0 += 64) {
          const int ea = e0 + 2 * lane, eb = ea + 1;
          const bool va = ea < nch, vb = eb < nch;
          R a0 = R(0), a1 = R(0);
          if (va) {
            const Rec<R> r = s_rec[ea];
            a0 = pixel_alpha<R>(pcx, pcy, r.mx, r.my, r.ca, r.cb, r.cc, r.op, wR, half_w).alpha;
          }
          if (vb) {
            const Rec<R> r = s_rec[eb];
            a1 = pixel_alpha<R>(pcx, pcy, r.mx, r.my, r.ca, r.cb, r.cc, r.op, wR, half_w).alpha;
          }
          const R om0 = sub(R(1), a0), om1 = sub(R(1), a1);
          R P = mul(om0, om1);  // lane total
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const R t = shfl_up_r(P, d);
            if (lane >= d) P = mul(t, P);
          }
          R Pex = shfl_up_r(P, 1);
          if (lane == 0) Pex = R(1);
          const R Tb0 = mul(Tin[s], Pex);
          const R Tb1 = mul(Tb0, om0);
          const int lf = (va && Tb0 < teps) ? 2 * lane : ((vb && Tb1 < teps) ? 2 * lane + 1 : 64);
          const int first = __reduce_min_sync(0xffffffffu, lf);
          const bool i0 = va && 2 * lane < first && a0 > R(0);
          const bool i1 = vb && 2 * lane + 1 < first && a1 > R(0);
          const unsigned m0 = __ballot_sync(0xffffffffu, i0);
          const unsigned m1 = __ballot_sync(0xffffffffu, i1);
          const R w0 = i0 ? mul(Tb0, a0) : R(0);
          const R w1 = i1 ? mul(Tb1, a1) : R(0);
          if (m0 | m1) {
            cnt[s] += __popc(m0) + __popc(m1);
            const int l0 = m0 ? 2 * (31 - __clz(m0)) : -1;
            const int l1 = m1 ? 2 * (31 - __clz(m1)) + 1 : -1;
            last[s] = cb - start + e0 + max(l0, l1) + 1;
          }
          if (AUX) {
            if (i0) s_live[ea] = 1;
            if (i1) s_live[eb] = 1;
          }
          if (ACC && SMALLC) {
#pragma unroll
            for (int c = 0; c < CC; ++c) {
              R v = w0 * s_coef[(va ? ea : 0) * CW + c] + w1 * s_coef[(vb ? eb : 0) * CW + c];
              v = warp_sum(v);
              sacc[s][c] += v;
            }
          } else if (WIDE) {
            s_w[ea * (RP + 1) + p] = w0;  // rows past nch are never read
            s_w[eb * (RP + 1) + p] = w1;
          }
          if (first < 64) {
            Tin[s] = first & 1 ? __shfl_sync(0xffffffffu, Tb1, first >> 1)
                               : __shfl_sync(0xffffffffu, Tb0, first >> 1);
            done_mask |= 1u << s;
            if (WIDE) {  // weights of the rest of this chunk are zero
              for (int e2 = e0 + 64 + lane; e2 < nch; e2 += 32) s_w[e2 * (RP + 1) + p] = R(0);
            }
            break;
          }
          Tin[s] = shfl_r(mul(Tin[s], P), 31);
        }
      } else if (WIDE) {
        for (int e = lane; e < nch; e += 32) s_w[e * (RP + 1) + p] = R(0);
      }
      if (lane == 0) s_done[p] = (done_mask >> s) & 1u;
    }
    if (aux_writer) {
      __syncthreads();
      for (int e = tid; e < nch; e += blockDim.x) {
        if (s_live[e]) {
          const int idx = s_idx[e];
          if (A.live[idx] == 0 && atomicExch(A.live + idx, 1) == 0) {
            const int pos = atomicAdd(A.counters + GSPARC_CNT_LIVE, 1);
            A.live_list[pos] = idx;
          }
        }
      }
    }
    if (WIDE) {
      __syncthreads();
      const R* cfg = s_coef + agrp * CC;
      for (int e = 0; e < nch; ++e) {
        const R wj = s_w[e * (RP + 1) + apix];
        if (__any_sync(0xffffffffu, wj != R(0))) {
          const R* cf = cfg + e * CW;
#pragma unroll
          for (int c = 0; c < CC; ++c) acc[c] += wj * cf[c];
        }
      }
    }
    if (__syncthreads_count(tid < RP ? s_done[tid] : 1) == (int)blockDim.x) break;
  }

  // ---- per-pixel outputs
#pragma unroll
  for (int s = 0; s < RSLOTS; ++s) {
    const int p = warp + RWARPS * s;
    const int px = tx_ * TILE + (p & 15), py = ty * TILE + part * 4 + (p >> 4);
    if (px < A.w && py < A.h && lane == 0) {
      const int q = py * A.w + px;
      if (aux_writer) {
        ((R*)A.T_out)[q] = Tin[s];
        A.count_out[q] = cnt[s];
        A.last_out[q] = last[s];
        atomicMax(&s_stop[p >> 5], last[s]);
      }
      if (ACC && SMALLC) {
#pragma unroll
        for (int c = 0; c < CC; ++c) {
          const int64_t cc = chunk_base + c;
          if (cc < A.Cp) {
            const int64_t b = cc / A.C, ch = cc - b * A.C;
            ((R*)A.img)[((b * A.h + py) * (int64_t)A.w + px) * A.C + ch] = sacc[s][c];
          }
        }
      }
    }
  }
  if (WIDE) {
    const int px = tx_ * TILE + (apix & 15), py = ty * TILE + part * 4 + (apix >> 4);
    if (px < A.w && py < A.h) {
#pragma unroll
      for (int c = 0; c < CC; ++c) {
        const int64_t cc = chunk_base + agrp * CC + c;
        if (cc < A.Cp) {
          const int64_t b = cc / A.C, ch = cc - b * A.C;
          ((R*)A.img)[((b * A.h + py) * (int64_t)A.w + px) * A.C + ch] = acc[c];
        }
      }
    }
  }
  if (aux_writer) {
    __syncthreads();
    if (tid < 2) A.wstop[tile * 8 + part * 2 + tid] = s_stop[tid];
  }
}

template <typename R, int CH, int CC, bool AUX, bool ACC, bool SMALLC>
static void launch_cfg(const RasterArgs& A, int chunks, cudaStream_t st) {
  constexpr int CW = SMALLC ? CC : CC * 4;
  const size_t smem = sizeof(Rec<R>) * CH + 2 * sizeof(int) * CH + 16 +
                      (ACC ? sizeof(R) * CH * CW : 0) +
                      ((ACC && !SMALLC) ? sizeof(R) * CH * (RP + 1) : 0);
  auto kern = k_raster<R, CH, CC, AUX, ACC, SMALLC>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  kern<<<dim3(A.ntiles * 4, chunks), 256, smem, st>>>(A);
}

// The raster and its backward split tiles into 4 sub-tiles of 4 rows.
int forward_sub_rows(const gsparc_frame_layout& /*L*/, int64_t /*Cp*/) { return 4; }

int launch_raster_forward(const gsparc_frame_layout& L, char* frame, int n_tx, int C,
                          double t_eps, int pass, void* img, cudaStream_t st) {
  RasterArgs A;
  A.pairs = (const uint64_t*)(frame + L.off_pairs);
  A.tile_start = (const int*)(frame + L.off_tile_start);
  A.wstop = (int*)(frame + L.off_wstop);
  A.rec32 = (const float4*)(frame + L.off_rec32);
  A.rec64 = (const double*)(frame + L.off_rec64);
  A.coef = frame + L.off_coef;
  A.Cp = (int64_t)n_tx * C;
  A.C = C;
  A.img = img;
  A.T_out = frame + L.off_T;
  A.count_out = (int*)(frame + L.off_count);
  A.last_out = (int*)(frame + L.off_last);
  A.live = (int*)(frame + L.off_live);
  A.live_list = (int*)(frame + L.off_live_list);
  A.counters = (int*)(frame + L.off_counters);
  A.w = L.width;
  A.h = L.height;
  A.ntx = L.ntx;
  A.ntiles = L.ntiles;
  A.t_eps = t_eps;
  if (A.Cp > L.channels || A.Cp < 1) {
    set_error("raster: n_tx*C=%lld outside frame channels %lld", (long long)A.Cp,
              (long long)L.channels);
    return GSPARC_ERR_ARG;
  }
  // f32 frames: one pixel per lane, tcgen05 accumulation (raster_px.cu)
  if (L.dtype == GSPARC_F32) return launch_raster_px(L, frame, n_tx, C, t_eps, pass, img, st);
  if (L.dtype == GSPARC_F64) {
    if (pass == 1) {
      launch_cfg<double, 64, 1, true, false, true>(A, 1, st);
    } else {
      const int chunks = (int)((A.Cp + 3) / 4);
      if (A.Cp <= 2) {
        if (pass == 0) launch_cfg<double, 64, 2, true, true, true>(A, 1, st);
        else launch_cfg<double, 64, 2, false, true, true>(A, 1, st);
      } else {
        if (pass == 0) launch_cfg<double, 64, 4, true, true, true>(A, chunks, st);
        else launch_cfg<double, 64, 4, false, true, true>(A, chunks, st);
      }
    }
  }
  return check_launch("k_raster");
}

}  // namespace gs
