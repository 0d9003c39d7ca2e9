// K4: front-to-back alpha compositing over hemisphere pixels x channels.
// Replaces do_tile / _tile_alphas (rasterizer.py:169-231).
//
// One CTA per sub-tile (16 x SR pixel rows of a 16x16 tile; SR = 4 gives
// 4 CTAs per tile, so 138 tiles fill 148 SMs several times over and the
// longest list bounds a quarter of the pixels only).  The tile's
// depth-sorted list is consumed in batches of NB entries staged in shared
// memory; per batch:
//   1. alphas: G threads per pixel split the NB entries (branch-free
//      pixel_alpha, exact numpy op order) -> shared memory;
//   2. scan: one thread per pixel applies the reference rule in list
//      order -- stop once T_before < t_eps, include iff alpha > 0,
//      wgt = T*alpha, T *= 1 - alpha, count++ (rasterizer.py:209-219) --
//      and overwrites alpha with wgt;
//   3. accumulate: all G groups add wgt * coef for CC channels each
//      (or, for <= 4 channels, the scan thread accumulates directly).
// The CTA leaves the list once every pixel has stopped (__syncthreads_count).
//
// Passes: AUX writes T_final / count / last / per-sub-tile stop and the live
// Gaussian list; ACC accumulates the image.  fused = AUX+ACC; the lazy-MLP
// path runs AUX first, evaluates the MLP on live Gaussians only, then ACC
// (identical arithmetic, so ACC reproduces AUX's weights bit for bit).
#include "common.cuh"
#include "kernels.cuh"

namespace gs {

struct RasterArgs {
  const uint64_t* pairs;
  const int* tile_start;
  int* sub_stop;  // [ntiles * nsub]
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
  int w, h, ntx, sr, nsub;
  double t_eps;
};

// SCANACC: the scan thread accumulates CC channels itself (small C').
// Otherwise, with ACC, every group accumulates CC channels after the scan.
template <typename R, int CC, int G, int NB, bool AUX, bool ACC, bool SCANACC>
__global__ void __launch_bounds__(256) k_raster_fwd(RasterArgs A) {
  constexpr int CW = SCANACC ? CC : CC * G;  // coef channels staged per CTA
  constexpr int PMAX = 256 / G;
  __shared__ Rec<R> s_rec[NB];
  __shared__ int s_idx[NB];
  __shared__ int s_live[NB];
  __shared__ __align__(16) R s_coef[ACC ? NB * CW : 1];
  __shared__ R s_w[NB * PMAX];  // alpha, then weight
  __shared__ int s_stop;

  if (A.counters[GSPARC_CNT_OVERFLOW]) return;
  const int P = blockDim.x / G;
  const int sidx = blockIdx.x, chunk = blockIdx.y;
  const int tile = sidx / A.nsub, part = sidx - tile * A.nsub;
  const int tid = threadIdx.x, pix = tid % P, grp = tid / P;
  const int tx_ = tile % A.ntx, ty = tile / A.ntx;
  const int px = tx_ * TILE + (pix & (TILE - 1));
  const int py = ty * TILE + part * A.sr + pix / TILE;
  const bool inside = px < A.w && py < A.h;
  const int start = A.tile_start[tile];
  const int end = AUX ? A.tile_start[tile + 1] : start + A.sub_stop[sidx];
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
      for (int e = tid; e < NB * CW; e += blockDim.x) {
        const int j = e / CW, c = e - j * CW;
        const int64_t cc = chunk_base + c;
        R v = R(0);
        if (j < nb && cc < A.Cp) {
          const uint32_t idx = (uint32_t)A.pairs[base + j];
          v = coef[(int64_t)idx * A.Cp + cc];
        }
        s_coef[e] = v;
      }
    }
    __syncthreads();
    // 1. alphas, entries split over the G groups
#pragma unroll
    for (int jj = 0; jj < NB / G; ++jj) {
      const int j = jj * G + grp;
      R a = R(0);
      if (j < nb) {
        const Rec<R> r = s_rec[j];
        a = pixel_alpha<R>(pcx, pcy, r.mx, r.my, r.ca, r.cb, r.cc, r.op, wR, half_w).alpha;
      }
      s_w[j * PMAX + pix] = a;
    }
    __syncthreads();
    // 2. sequential scan in list order (one thread per pixel)
    if (grp == 0) {
#pragma unroll 8
      for (int j = 0; j < NB; ++j) {
        const R a = s_w[j * PMAX + pix];
        R wgt = R(0);
        if (!done) {
          if (T < teps) {
            done = true;
          } else if (a > R(0)) {
            wgt = mul(T, a);
            T = mul(T, sub(R(1), a));
            if (AUX) {
              ++cnt;
              last = base - start + j + 1;
              s_live[j] = 1;
            }
          }
        }
        if (ACC && SCANACC) {
          if (wgt != R(0)) {
#pragma unroll
            for (int c = 0; c < CC; ++c) acc[c] += wgt * s_coef[j * CW + c];
          }
        } else if (ACC) {
          s_w[j * PMAX + pix] = wgt;
        }
      }
      if (!done && T < teps) done = true;
    }
    if (ACC && !SCANACC) {
      __syncthreads();
      // 3. channel accumulation; warp-uniform skip of all-zero weights
      const R* cfg = s_coef + grp * CC;
      for (int j = 0; j < nb; ++j) {
        const R wj = s_w[j * PMAX + pix];
        if (__any_sync(0xffffffffu, wj != R(0))) {
          const R* cf = cfg + j * CW;
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
    if (tid == 0) A.sub_stop[sidx] = s_stop;
  }
  if (ACC && inside && (SCANACC ? grp == 0 : true)) {
    const int g0 = SCANACC ? 0 : grp;
#pragma unroll
    for (int c = 0; c < CC; ++c) {
      const int64_t cc = chunk_base + g0 * CC + c;
      if (cc < A.Cp) {
        const int64_t b = cc / A.C, ch = cc - b * A.C;
        ((R*)A.img)[((b * A.h + py) * (int64_t)A.w + px) * A.C + ch] = acc[c];
      }
    }
  }
}

template <typename R, int CC, int G, int NB, bool AUX, bool ACC, bool SCANACC>
static void launch_cfg(const RasterArgs& A, int nsubs, int chunks, cudaStream_t st) {
  dim3 grid(nsubs, chunks);
  k_raster_fwd<R, CC, G, NB, AUX, ACC, SCANACC><<<grid, TILE * A.sr * G, 0, st>>>(A);
}

template <bool AUX>
static int dispatch_f32(const RasterArgs& A, int nsubs, cudaStream_t st) {
  const int64_t Cp = A.Cp;
  if (Cp <= 2) {
    launch_cfg<float, 2, 4, 32, AUX, true, true>(A, nsubs, 1, st);
  } else if (Cp <= 4) {
    launch_cfg<float, 4, 4, 32, AUX, true, true>(A, nsubs, 1, st);
  } else {
    int chunks = (int)((Cp + 127) / 128);
    int per = (int)((Cp + chunks - 1) / chunks);  // channels per CTA
    int cc = ((per + 3) / 4 + 3) / 4 * 4;         // per group, multiple of 4
    if (cc < 4) cc = 4;
    switch (cc) {
      case 4: launch_cfg<float, 4, 4, 32, AUX, true, false>(A, nsubs, chunks, st); break;
      case 8: launch_cfg<float, 8, 4, 32, AUX, true, false>(A, nsubs, chunks, st); break;
      case 12: launch_cfg<float, 12, 4, 32, AUX, true, false>(A, nsubs, chunks, st); break;
      case 16: launch_cfg<float, 16, 4, 32, AUX, true, false>(A, nsubs, chunks, st); break;
      case 20: launch_cfg<float, 20, 4, 32, AUX, true, false>(A, nsubs, chunks, st); break;
      case 24: launch_cfg<float, 24, 4, 32, AUX, true, false>(A, nsubs, chunks, st); break;
      case 28: launch_cfg<float, 28, 4, 32, AUX, true, false>(A, nsubs, chunks, st); break;
      default: {
        chunks = (int)((Cp + 127) / 128);
        launch_cfg<float, 32, 4, 32, AUX, true, false>(A, nsubs, chunks, st);
      }
    }
  }
  return GSPARC_OK;
}

// Sub-tile rows: 4 -> 64-pixel CTAs of 4 thread groups (256 threads).  The
// backward reuses the same split (it reads the per-sub-tile stops).
int forward_sub_rows(const gsparc_frame_layout& /*L*/, int64_t /*Cp*/) { return 4; }

int launch_raster_forward(const gsparc_frame_layout& L, char* frame, int n_tx, int C,
                          double t_eps, int pass, void* img, cudaStream_t st) {
  RasterArgs A;
  A.pairs = (const uint64_t*)(frame + L.off_pairs);
  A.tile_start = (const int*)(frame + L.off_tile_start);
  A.sub_stop = (int*)(frame + L.off_tile_stop);
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
  A.sr = forward_sub_rows(L, A.Cp);
  A.nsub = TILE / A.sr;
  const int nsubs = L.ntiles * A.nsub;
  if (pass != 2) {
    if (cudaMemsetAsync(A.live, 0, sizeof(int) * L.n, st) != cudaSuccess)
      return check_launch("raster live memset");
  }
  if (L.dtype == GSPARC_F64) {
    if (pass == 1) {
      launch_cfg<double, 1, 4, 16, true, false, true>(A, nsubs, 1, st);
    } else {
      const int chunks = (int)((A.Cp + 3) / 4);
      if (A.Cp <= 2) {
        if (pass == 0) launch_cfg<double, 2, 4, 16, true, true, true>(A, nsubs, 1, st);
        else launch_cfg<double, 2, 4, 16, false, true, true>(A, nsubs, 1, st);
      } else {
        if (pass == 0) launch_cfg<double, 4, 4, 16, true, true, true>(A, nsubs, chunks, st);
        else launch_cfg<double, 4, 4, 16, false, true, true>(A, nsubs, chunks, st);
      }
    }
  } else {
    if (pass == 1) launch_cfg<float, 1, 4, 32, true, false, true>(A, nsubs, 1, st);
    else if (pass == 0) dispatch_f32<true>(A, nsubs, st);
    else dispatch_f32<false>(A, nsubs, st);
  }
  return check_launch("k_raster_fwd");
}

}  // namespace gs
