// K4: front-to-back alpha compositing over hemisphere pixels x channels.
// Replaces do_tile / _tile_alphas (rasterizer.py:169-231).
//
// One CTA per 16x16 tile (and per channel chunk when channels > 128).  The
// tile's depth-sorted list is consumed in batches staged in shared memory.
// Per pixel, in list order:  T_before < t_eps -> stop;  alpha from
// pixel_alpha() (exact numpy op order);  alpha > 0 -> wgt = T*alpha,
// img += wgt * coef, count++, T *= 1 - alpha  (rasterizer.py:209-219).
// The CTA leaves the list as soon as every pixel has stopped
// (__syncthreads_count), which is the raster's dominant saving on the
// occlusion-dominated scenes.
//
// Channel layout: G thread groups of 256 share the pixels; group 0 computes
// the compositing weights once into shared memory and all G groups
// accumulate CC channels each, so the TX-independent alpha/T work is done
// once for up to 128 channels (C' = n_tx * C).
//
// Passes: AUX writes T_final / count / last and the live-Gaussian list;
// ACC accumulates the image.  Fused = AUX+ACC; the lazy-MLP path runs AUX
// first, evaluates the MLP on live Gaussians only, then ACC.
#include "common.cuh"
#include "kernels.cuh"

namespace gs {

struct RasterArgs {
  const uint64_t* pairs;
  const int* tile_start;
  int* tile_stop;
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
  int w, h, ntx;
  double t_eps;
};

template <typename R, int CC, int G, bool AUX, bool ACC>
__global__ void __launch_bounds__(256 * G) k_raster_fwd(RasterArgs A) {
  constexpr int NB = (G == 1) ? 32 : 16;
  constexpr int CW = CC * G;
  __shared__ Rec<R> s_rec[NB];
  __shared__ int s_idx[NB];
  __shared__ int s_live[NB];
  __shared__ R s_coef[ACC ? NB * CW : 1];
  __shared__ R s_wgt[(ACC && G > 1) ? NB * TILE_PX : 1];
  __shared__ int s_stop;

  if (A.counters[GSPARC_CNT_OVERFLOW]) return;
  const int tile = blockIdx.x, chunk = blockIdx.y;
  const int tid = threadIdx.x, pix = tid & (TILE_PX - 1), grp = tid / TILE_PX;
  const int tx_ = tile % A.ntx, ty = tile / A.ntx;
  const int px = tx_ * TILE + (pix & (TILE - 1)), py = ty * TILE + pix / TILE;
  const bool inside = px < A.w && py < A.h;
  const int start = A.tile_start[tile];
  const int end = AUX ? A.tile_start[tile + 1] : start + A.tile_stop[tile];
  const bool aux_writer = AUX && chunk == 0;
  const R pcx = (R)px + R(0.5), pcy = (R)py + R(0.5);
  const R wR = (R)A.w, half_w = (R)(A.w / 2.0);
  const R teps = (R)A.t_eps;
  const int chunk_base = chunk * CW;

  R T = R(1);
  int cnt = 0, last = 0;
  bool done = !inside || grp != 0;
  R acc[ACC ? CC : 1];
#pragma unroll
  for (int c = 0; c < (ACC ? CC : 1); ++c) acc[c] = R(0);
  if (AUX && tid == 0) s_stop = 0;

  for (int base = start; base < end; base += NB) {
    const int nb = min(NB, end - base);
    __syncthreads();
    if (tid < nb) {
      const uint32_t idx = (uint32_t)A.pairs[base + tid];
      s_idx[tid] = (int)idx;
      s_rec[tid] = load_rec_t<R>(A.rec32, A.rec64, idx);
      if (AUX) s_live[tid] = 0;
    }
    if (ACC) {
      const R* coef = (const R*)A.coef;
      for (int e = tid; e < nb * CW; e += blockDim.x) {
        const int j = e / CW, c = e - j * CW;
        const uint32_t idx = (uint32_t)A.pairs[base + j];
        const int64_t cc = chunk_base + c;
        s_coef[e] = cc < A.Cp ? coef[(int64_t)idx * A.Cp + cc] : R(0);
      }
    }
    __syncthreads();
    if (grp == 0) {
      for (int j = 0; j < nb; ++j) {
        R wgt = R(0);
        if (!done) {
          if (T < teps) {
            done = true;
          } else {
            const Rec<R> r = s_rec[j];
            const AlphaOut<R> a =
                pixel_alpha<R>(pcx, pcy, r.mx, r.my, r.ca, r.cb, r.cc, r.op, wR, half_w);
            if (a.alpha > R(0)) {
              wgt = mul(T, a.alpha);
              if (AUX) {
                ++cnt;
                last = base - start + j + 1;
                s_live[j] = 1;
              }
              if (ACC && G == 1) {
#pragma unroll
                for (int c = 0; c < CC; ++c) acc[c] += wgt * s_coef[j * CW + c];
              }
              T = mul(T, sub(R(1), a.alpha));
            }
          }
        }
        if (ACC && G > 1) s_wgt[j * TILE_PX + pix] = wgt;
      }
      if (!done && T < teps) done = true;
    }
    if (ACC && G > 1) {
      __syncthreads();
      for (int j = 0; j < nb; ++j) {
        const R wj = s_wgt[j * TILE_PX + pix];
        if (wj != R(0)) {
          const R* cf = s_coef + j * CW + grp * CC;
#pragma unroll
          for (int c = 0; c < CC; ++c) acc[c] += wj * cf[c];
        }
      }
    }
    if (aux_writer) {
      __syncthreads();
      if (tid < nb && s_live[tid]) {
        const int idx = s_idx[tid];
        if (atomicExch(A.live + idx, 1) == 0) {
          const int pos = atomicAdd(A.counters + GSPARC_CNT_LIVE, 1);
          A.live_list[pos] = idx;
        }
      }
    }
    if (__syncthreads_count(done) == (int)blockDim.x) break;
  }

  if (aux_writer && grp == 0 && inside) {
    const int p = py * A.w + px;
    ((R*)A.T_out)[p] = T;
    A.count_out[p] = cnt;
    A.last_out[p] = last;
    atomicMax(&s_stop, last);
  }
  if (aux_writer) {
    __syncthreads();
    if (tid == 0) A.tile_stop[tile] = s_stop;
  }
  if (ACC && inside) {
#pragma unroll
    for (int c = 0; c < CC; ++c) {
      const int64_t cc = chunk_base + grp * CC + c;
      if (cc < A.Cp) {
        const int64_t b = cc / A.C, ch = cc - b * A.C;
        ((R*)A.img)[((b * A.h + py) * (int64_t)A.w + px) * A.C + ch] = acc[c];
      }
    }
  }
}

template <typename R, int CC, int G, bool AUX, bool ACC>
static void launch_cfg(const RasterArgs& A, int ntiles, int chunks, cudaStream_t st) {
  dim3 grid(ntiles, chunks);
  k_raster_fwd<R, CC, G, AUX, ACC><<<grid, 256 * G, 0, st>>>(A);
}

template <bool AUX>
static int dispatch_f32(const RasterArgs& A, int ntiles, cudaStream_t st) {
  const int64_t Cp = A.Cp;
  if (Cp <= 2) {
    launch_cfg<float, 2, 1, AUX, true>(A, ntiles, 1, st);
  } else if (Cp <= 4) {
    launch_cfg<float, 4, 1, AUX, true>(A, ntiles, 1, st);
  } else {
    int chunks = (int)((Cp + 127) / 128);
    int per = (int)((Cp + chunks - 1) / chunks);  // channels per CTA
    int cc = ((per + 3) / 4 + 3) / 4 * 4;         // per-group, multiple of 4
    if (cc < 4) cc = 4;
    switch (cc) {
      case 4: launch_cfg<float, 4, 4, AUX, true>(A, ntiles, chunks, st); break;
      case 8: launch_cfg<float, 8, 4, AUX, true>(A, ntiles, chunks, st); break;
      case 12: launch_cfg<float, 12, 4, AUX, true>(A, ntiles, chunks, st); break;
      case 16: launch_cfg<float, 16, 4, AUX, true>(A, ntiles, chunks, st); break;
      case 20: launch_cfg<float, 20, 4, AUX, true>(A, ntiles, chunks, st); break;
      case 24: launch_cfg<float, 24, 4, AUX, true>(A, ntiles, chunks, st); break;
      case 28: launch_cfg<float, 28, 4, AUX, true>(A, ntiles, chunks, st); break;
      default: {
        chunks = (int)((Cp + 127) / 128);
        launch_cfg<float, 32, 4, AUX, true>(A, ntiles, chunks, st);
      }
    }
  }
  return GSPARC_OK;
}

int launch_raster_forward(const gsparc_frame_layout& L, char* frame, int n_tx, int C,
                          double t_eps, int pass, void* img, cudaStream_t st) {
  RasterArgs A;
  A.pairs = (const uint64_t*)(frame + L.off_pairs);
  A.tile_start = (const int*)(frame + L.off_tile_start);
  A.tile_stop = (int*)(frame + L.off_tile_stop);
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
  A.t_eps = t_eps;
  if (A.Cp > L.channels || A.Cp < 1) {
    set_error("raster: n_tx*C=%lld outside frame channels %lld", (long long)A.Cp,
              (long long)L.channels);
    return GSPARC_ERR_ARG;
  }
  if (pass != 2) {
    if (cudaMemsetAsync(A.live, 0, sizeof(int) * L.n, st) != cudaSuccess)
      return check_launch("raster live memset");
  }
  const int T = L.ntiles;
  if (L.dtype == GSPARC_F64) {
    if (pass == 1) {
      launch_cfg<double, 1, 1, true, false>(A, T, 1, st);
    } else {
      int chunks = (int)((A.Cp + 3) / 4);
      if (A.Cp <= 2) {
        if (pass == 0) launch_cfg<double, 2, 1, true, true>(A, T, 1, st);
        else launch_cfg<double, 2, 1, false, true>(A, T, 1, st);
      } else {
        if (pass == 0) launch_cfg<double, 4, 1, true, true>(A, T, chunks, st);
        else launch_cfg<double, 4, 1, false, true>(A, T, chunks, st);
      }
    }
  } else {
    if (pass == 1) launch_cfg<float, 1, 1, true, false>(A, T, 1, st);
    else if (pass == 0) dispatch_f32<true>(A, T, st);
    else dispatch_f32<false>(A, T, st);
  }
  return check_launch("k_raster_fwd");
}

}  // namespace gs
