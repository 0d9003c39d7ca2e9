// K7: training loss on device.  Replaces image.magnitude /
// magnitude_backward (image.py:46-61) and optimize.combined_loss with the
// exact SSIM adjoint (optimize.py:67-188):
//   loss_b = (1-lam) mean|p-g| + lam (1 - mean_c SSIM_c)
// SSIM: 11-tap Gaussian window (sigma 1.5), separable, scipy 'reflect'
// (half-sample symmetric) padding; gradient through the adjoint filter
// (zero-padded correlation folded back at the borders, optimize.py:97-115).
// f64 throughout (variance terms cancel).  Pipeline, one thread per pixel:
//   h-blur of (x, y, xx, yy, xy) -> v-blur + SSIM map + adjoint seeds
//   -> adjoint v -> adjoint h + L1 term + magnitude chain -> dimg.
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace gs {

// optimize.py:81-87: x = arange(11) - 5; w = exp(-(x/1.5)^2/2) / sum
static void make_window(double* w) {
  double s = 0.0;
  for (int t = 0; t < 11; ++t) {
    double x = (double)t - 5.0;
    w[t] = exp(-0.5 * ((x / 1.5) * (x / 1.5)));
    s += w[t];
  }
  for (int t = 0; t < 11; ++t) w[t] /= s;
}

template <typename T>
struct LossArgsT {
  double win[11];
  const T* img;
  const T* gt;
  T* dimg;
  double* H5;    // [5][NI][S][h][w]
  double* G3;    // [3][NI][S][h][w]
  double* A3;    // [3][NI][S][h][w]
  double* XY;    // [2][NI][S][h][w] prediction and ground truth (f64)
  double* sums;  // [NI * S][LOSS_RB][3] per-plane partial (ssim, l1, sq) sums
  double* V3;    // [3][tot] per-pixel (ssim, l1, sq) terms
  double* stats; // [NI][GSPARC_LOSS_STATS]
  int NI, S, C, h, w, sup;
  double lam;
};

constexpr int LOSS_RB = 16;  // CTAs per (image, channel) plane in k_loss_reduce

__device__ __forceinline__ int refl(int j, int n) {
  if (j < 0) return -j - 1;
  if (j >= n) return 2 * n - 1 - j;
  return j;
}

template <typename T>
__device__ __forceinline__ double pred_at(const LossArgsT<T>& A, int b, int s, int r, int c) {
  const T* z = A.img + (((int64_t)b * A.h + r) * A.w + c) * A.C;
  if (A.sup == 0) {  // C == 2: one (re, im) pair load
    using T2 = typename std::conditional<sizeof(T) == 4, float2, double2>::type;
    const T2 zz = *(const T2*)z;
    return hypot((double)zz.x, (double)zz.y);
  }
  return (double)z[s];
}
template <typename T>
__device__ __forceinline__ double gt_at(const LossArgsT<T>& A, int b, int s, int r, int c) {
  return (double)A.gt[(((int64_t)b * A.h + r) * A.w + c) * A.S + s];
}

// prediction (|z| for magnitude supervision) and ground truth once per pixel
// (the blur reads each 11 times); indices fit 32 bits (checked on launch)
template <typename T>
__global__ void k_loss_prep(LossArgsT<T> A) {
  const int plane = A.h * A.w, tot = A.NI * A.S * plane;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tot) return;
  const int c = e % A.w, r = (e / A.w) % A.h, bs = e / plane;
  const int s = bs % A.S, b = bs / A.S;
  A.XY[e] = pred_at(A, b, s, r, c);
  A.XY[tot + e] = gt_at(A, b, s, r, c);
}

template <typename T>
__global__ void k_loss_h(LossArgsT<T> A) {
  const int plane = A.h * A.w, tot = A.NI * A.S * plane;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tot) return;
  const int c = e % A.w;
  const int rowbase = e - c;
  double a[5] = {0, 0, 0, 0, 0};
#pragma unroll
  for (int t = 0; t < 11; ++t) {
    const int cc = refl(c + t - 5, A.w);
    const double x = A.XY[rowbase + cc], y = A.XY[tot + rowbase + cc];
    const double wt = A.win[t];
    a[0] += wt * x;
    a[1] += wt * y;
    a[2] += wt * (x * x);
    a[3] += wt * (y * y);
    a[4] += wt * (x * y);
  }
  for (int k = 0; k < 5; ++k) A.H5[(int64_t)k * tot + e] = a[k];
}

template <typename T>
__global__ void k_loss_v(LossArgsT<T> A) {
  const int plane = A.h * A.w, tot = A.NI * A.S * plane;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  double ssim_v = 0.0, l1_v = 0.0, sq_v = 0.0;
  if (e < tot) {
    const int c = e % A.w, r = (e / A.w) % A.h;
    const int bs = e / plane;
    const int64_t rowbase = (int64_t)bs * plane;
    double m[5] = {0, 0, 0, 0, 0};
    for (int t = 0; t < 11; ++t) {
      const int rr = refl(r + t - 5, A.h);
      const double wt = A.win[t];
      for (int k = 0; k < 5; ++k) m[k] += wt * A.H5[(int64_t)k * tot + rowbase + (int64_t)rr * A.w + c];
    }
    const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
    const double mx = m[0], my = m[1];
    const double vx = m[2] - mx * mx, vy = m[3] - my * my, vxy = m[4] - mx * my;
    const double a1 = 2 * mx * my + c1, a2 = 2 * vxy + c2;
    const double b1 = mx * mx + my * my + c1, b2 = vx + vy + c2;
    const double sv = (a1 * a2) / (b1 * b2);
    const double da1 = a2 / (b1 * b2), da2 = a1 / (b1 * b2);
    const double db1 = -sv / b1, db2 = -sv / b2;
    A.G3[e] = 2 * my * da1 - 2 * my * da2 + 2 * mx * db1 - 2 * mx * db2;
    A.G3[(int64_t)tot + e] = db2;
    A.G3[2 * (int64_t)tot + e] = 2 * da2;
    ssim_v = sv;
    const double x = A.XY[e], y = A.XY[tot + e];
    l1_v = fabs(x - y);
    sq_v = (x - y) * (x - y);
  }
  // per-pixel terms; summed per (image, channel) plane in a fixed order by
  // k_loss_reduce (no float atomics: the reported losses are bit-stable)
  if (e < tot) {
    A.V3[e] = ssim_v;
    A.V3[(int64_t)tot + e] = l1_v;
    A.V3[2 * (int64_t)tot + e] = sq_v;
  }
}

// LOSS_RB CTAs per plane: fixed strided per-thread sums and a fixed shuffle
// tree per CTA; k_loss_finalize adds the CTA partials in order
template <typename T>
__global__ void __launch_bounds__(256) k_loss_reduce(LossArgsT<T> A) {
  __shared__ double s_part[8][3];
  const int64_t plane = (int64_t)A.h * A.w, tot = (int64_t)A.NI * A.S * plane;
  const int64_t p = blockIdx.x / LOSS_RB;
  const int rb = blockIdx.x % LOSS_RB;
  double v[3] = {0.0, 0.0, 0.0};
  for (int64_t i = rb * blockDim.x + threadIdx.x; i < plane; i += LOSS_RB * blockDim.x) {
    const int64_t e = p * plane + i;
    v[0] += A.V3[e];
    v[1] += A.V3[tot + e];
    v[2] += A.V3[2 * tot + e];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    v[k] = warp_sum(v[k]);
    if (lane == 0) s_part[warp][k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_part[w][threadIdx.x];
    A.sums[(p * LOSS_RB + rb) * 3 + threadIdx.x] = t;  // plane p = b * S + s
  }
}

// adjoint along rows: out[r] = G(r) + [r<5] G(-r-1) + [r>=h-5] G(2h-1-r),
// G(j) = sum_t w[t] g[j+t-5] (g = 0 outside [0,h))
template <typename T>
__device__ __forceinline__ double adj_line(const LossArgsT<T>& A, const double* g, int stride, int n,
                                          int i) {
  if (i >= 5 && i + 5 < n) {  // interior: all 11 taps in range, no fold-back
    const double* gi = g + (int64_t)(i - 5) * stride;
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < 11; ++t) acc += A.win[t] * gi[(int64_t)t * stride];
    return acc;
  }
  auto G = [&](int j) {
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < 11; ++t) {
      const int q = j + t - 5;
      if (q >= 0 && q < n) acc += A.win[t] * g[(int64_t)q * stride];
    }
    return acc;
  };
  double out = G(i);
  if (i < 5) out += G(-i - 1);
  if (i >= n - 5) out += G(2 * n - 1 - i);
  return out;
}

template <typename T>
__global__ void k_loss_adj_v(LossArgsT<T> A) {
  const int plane = A.h * A.w, tot = A.NI * A.S * plane;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tot) return;
  const int c = e % A.w, r = (e / A.w) % A.h;
  const int bs = e / plane;
  for (int k = 0; k < 3; ++k)
    A.A3[(int64_t)k * tot + e] =
        adj_line(A, A.G3 + (int64_t)k * tot + (int64_t)bs * plane + c, A.w, A.h, r);
}

template <typename T>
__global__ void k_loss_adj_h(LossArgsT<T> A) {
  const int plane = A.h * A.w, tot = A.NI * A.S * plane;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= tot) return;
  const int c = e % A.w, r = (e / A.w) % A.h;
  const int bs = e / plane;
  const int s = bs % A.S, b = bs / A.S;
  const double* rowp = A.A3 + (int64_t)bs * plane + (int64_t)r * A.w;
  const double amx = adj_line(A, rowp, 1, A.w, c);
  const double ab2 = adj_line(A, rowp + tot, 1, A.w, c);
  const double aa2 = adj_line(A, rowp + 2 * tot, 1, A.w, c);
  const double x = A.XY[e], y = A.XY[tot + e];
  const double n = (double)plane;
  const double gssim = (amx + 2 * x * ab2 + y * aa2) / n;
  const double diff = x - y;
  const double sgn = diff > 0 ? 1.0 : (diff < 0 ? -1.0 : 0.0);
  const double gp = (1.0 - A.lam) * sgn / (n * A.S) - A.lam * gssim / A.S;
  T* dz = A.dimg + (((int64_t)b * A.h + r) * A.w + c) * A.C;
  if (A.sup == 0) {
    const T* z = A.img + (((int64_t)b * A.h + r) * A.w + c) * A.C;
    const double re = z[0], im = z[1];
    const double m = hypot(re, im);
    const double k = m > 0.0 ? gp / m : 0.0;
    dz[0] = (T)(re * k);
    dz[1] = (T)(im * k);
  } else {
    dz[s] = (T)gp;
  }
}

template <typename T>
__global__ void k_loss_finalize(LossArgsT<T> A) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= A.NI) return;
  const double* sm = A.sums + (int64_t)b * A.S * LOSS_RB * 3;
  const double n = (double)A.h * A.w;
  double ss = 0.0, l1s = 0.0, sqs = 0.0, ss0 = 0.0, sq0 = 0.0;
  for (int s = 0; s < A.S; ++s) {
    double t[3] = {0.0, 0.0, 0.0};
    for (int rb = 0; rb < LOSS_RB; ++rb)
      for (int k = 0; k < 3; ++k) t[k] += sm[(s * LOSS_RB + rb) * 3 + k];
    ss += t[0] / n;
    l1s += t[1];
    sqs += t[2];
    if (s == 0) {
      ss0 = t[0] / n;
      sq0 = t[2] / n;
    }
  }
  ss /= A.S;
  const double l1 = l1s / (n * A.S);
  double* o = A.stats + (int64_t)GSPARC_LOSS_STATS * b;
  o[0] = (1.0 - A.lam) * l1 + A.lam * (1.0 - ss);
  o[1] = l1;
  o[2] = ss;
  o[3] = sqs / (n * A.S);
  // channel 0 only: the reference's train_step logs ssim/psnr of
  // pred[:,:,0] vs gt[:,:,0] (optimize.py:281,293)
  o[4] = ss0;
  o[5] = sq0;
}

// ---------------------------------------------------------------- banded K7
// Two kernels over (column band of LB output columns, image plane), each
// staging its band plus a 5-column halo for all rows in shared memory:
//   k_loss_band_fwd: x/y (|z| for magnitude supervision, reflect-padded
//     columns) -> h-blur of (x, y, xx, yy, xy) -> v-blur (reflect rows) ->
//     SSIM and its three adjoint seeds (written to G3) + the band's
//     fixed-order (ssim, l1, sq) partial sums;
//   k_loss_band_adj: G3 (zero outside the image) -> adjoint v-blur (rows
//     folded back at the borders) -> adjoint h-blur (columns folded) ->
//     L1 term + magnitude chain -> dL/dimg.
// Same arithmetic (f64, taps in order) as the per-pixel kernels above, two
// launches instead of six.
// 40-column bands: 9 bands x 32 planes = 288 CTAs of one per SM (2 waves
// on 148 SMs) at 90x360, where 32 columns gave 384 (2.6 waves)
constexpr int LB = 40;        // output columns per band (the last band is padded)
constexpr int RB = 1024 / LB; // band rows per pass
constexpr int XW = LB + 10;   // staged columns: the band + a 5-column halo each side

__host__ __device__ inline int loss_nbands(int w) { return (w + LB - 1) / LB; }
__host__ __device__ inline size_t loss_band_smem(int h) {
  return sizeof(double) * (size_t)h * (size_t)(2 * XW + 5 * LB);
}
__host__ __device__ inline size_t loss_adj_smem(int h) {
  return sizeof(double) * (size_t)h * (size_t)(6 * XW);
}
constexpr size_t LOSS_SMEM_MAX = 224 * 1024;  // + the static reduction buffer <= 227 KB

// 11-tap window sum over a strided line with every tap in range
__device__ __forceinline__ double tap11(const double (&wv)[11], const double* g, int stride) {
  double acc = 0.0;
#pragma unroll
  for (int t = 0; t < 11; ++t) acc += wv[t] * g[t * stride];
  return acc;
}

// out(i) = G(i) + [i < 5] G(-i-1) + [i >= n-5] G(2n-1-i), G(j) = sum_t w[t]
// g[j+t-5] (g = 0 outside [0, n)); line element q at g[(q - q0) * stride]
__device__ __forceinline__ double adj_fold(const double (&wv)[11], const double* g, int stride,
                                          int q0, int n, int i) {
  if (i >= 5 && i + 5 < n) return tap11(wv, g + (i - 5 - q0) * stride, stride);
  auto G = [&](int j) {
    double acc = 0.0;
#pragma unroll
    for (int t = 0; t < 11; ++t) {
      const int q = j + t - 5;
      if (q >= 0 && q < n) acc += wv[t] * g[(q - q0) * stride];
    }
    return acc;
  };
  double out = G(i);
  if (i < 5) out += G(-i - 1);
  if (i >= n - 5) out += G(2 * n - 1 - i);
  return out;
}

template <typename T>
__global__ void __launch_bounds__(1024) k_loss_band_fwd(LossArgsT<T> A) {
  extern __shared__ double lsm[];
  const int h = A.h, w = A.w;
  const int p = blockIdx.y, b = p / A.S, s = p - b * A.S;
  const int c0 = blockIdx.x * LB;
  double wv[11];
#pragma unroll
  for (int t = 0; t < 11; ++t) wv[t] = A.win[t];
  double* X = lsm;              // [h][XW]
  double* Y = X + h * XW;       // [h][XW]
  double* H5 = Y + h * XW;      // [5][h][LB]
  // x / y with reflect-padded columns (columns past the image in a padded
  // last band are staged too; their outputs are never written)
  // 2-D thread maps fixed per thread (no index divisions in the loops):
  // staged rows of XW columns (RS rows per pass) and band rows of LB columns
  // (RB rows per pass)
  constexpr int RS = 1024 / XW;
  const int sx = threadIdx.x % XW, sy = threadIdx.x / XW;
  const int bx = threadIdx.x % LB, by = threadIdx.x / LB;
  if (sy < RS) {
    const int col = refl(min(c0 - 5 + sx, 2 * w - 1), w);
#pragma unroll 4
    for (int r = sy; r < h; r += RS) {
      X[r * XW + sx] = pred_at(A, b, s, r, col);
      Y[r * XW + sx] = gt_at(A, b, s, r, col);
    }
  }
  __syncthreads();
  const int HW = h * LB;
  for (int r = by; r < h && by < RB; r += RB) {
    const int c = bx, e = r * LB + c;
    double a[5] = {0, 0, 0, 0, 0};
    const double* xr = X + r * XW + c;
    const double* yr = Y + r * XW + c;
#pragma unroll
    for (int t = 0; t < 11; ++t) {
      const double x = xr[t], y = yr[t], wt = wv[t];
      a[0] += wt * x;
      a[1] += wt * y;
      a[2] += wt * (x * x);
      a[3] += wt * (y * y);
      a[4] += wt * (x * y);
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) H5[k * HW + e] = a[k];
  }
  __syncthreads();
  const int64_t plane = (int64_t)h * w, tot = (int64_t)A.NI * A.S * plane;
  double v3[3] = {0.0, 0.0, 0.0};
  for (int r = by; r < h && by < RB; r += RB) {
    const int c = bx;
    if (c0 + c >= w) continue;
    double m[5] = {0, 0, 0, 0, 0};
    if (r >= 5 && r + 5 < h) {  // interior rows: straight taps
      const double* hc = H5 + (r - 5) * LB + c;
#pragma unroll
      for (int t = 0; t < 11; ++t) {
#pragma unroll
        for (int k = 0; k < 5; ++k) m[k] += wv[t] * hc[k * HW + t * LB];
      }
    } else {
#pragma unroll
      for (int t = 0; t < 11; ++t) {
        const double* hc = H5 + refl(r + t - 5, h) * LB + c;
#pragma unroll
        for (int k = 0; k < 5; ++k) m[k] += wv[t] * hc[k * HW];
      }
    }
    const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
    const double mx = m[0], my = m[1];
    const double vx = m[2] - mx * mx, vy = m[3] - my * my, vxy = m[4] - mx * my;
    const double a1 = 2 * mx * my + c1, a2 = 2 * vxy + c2;
    const double b1 = mx * mx + my * my + c1, b2 = vx + vy + c2;
    // one f64 division per pixel instead of five (1/(b1 b2) and its
    // products give 1/b1 = b2 / (b1 b2), 1/b2 = b1 / (b1 b2))
    const double ib = 1.0 / (b1 * b2);
    const double sv = (a1 * a2) * ib;
    const double da1 = a2 * ib, da2 = a1 * ib;
    const double db1 = -sv * (b2 * ib), db2 = -sv * (b1 * ib);
    const int64_t pe = (int64_t)p * plane + (int64_t)r * w + c0 + c;
    A.G3[pe] = 2 * my * da1 - 2 * my * da2 + 2 * mx * db1 - 2 * mx * db2;
    A.G3[tot + pe] = db2;
    A.G3[2 * tot + pe] = 2 * da2;
    const double x = X[r * XW + c + 5], y = Y[r * XW + c + 5];
    v3[0] += sv;
    v3[1] += fabs(x - y);
    v3[2] += (x - y) * (x - y);
  }
  // fixed-order CTA reduction: warp trees, then warps in order
  __shared__ double s_part[32][3];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    v3[k] = warp_sum(v3[k]);
    if (lane == 0) s_part[warp][k] = v3[k];
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int wq = 0; wq < (int)(blockDim.x >> 5); ++wq) t += s_part[wq][threadIdx.x];
    A.sums[((int64_t)p * gridDim.x + blockIdx.x) * 3 + threadIdx.x] = t;
  }
}

template <typename T>
__global__ void __launch_bounds__(1024) k_loss_band_adj(LossArgsT<T> A) {
  extern __shared__ double lsm[];
  const int h = A.h, w = A.w;
  const int p = blockIdx.y, b = p / A.S, s = p - b * A.S;
  const int c0 = blockIdx.x * LB;
  const int64_t plane = (int64_t)h * w, tot = (int64_t)A.NI * A.S * plane;
  double wv[11];
#pragma unroll
  for (int t = 0; t < 11; ++t) wv[t] = A.win[t];
  double* G = lsm;                 // [3][h][XW], columns c0-5 .. c0+LB+5
  double* Av = G + 3 * h * XW;     // [3][h][XW]
  const int HX = h * XW;
  constexpr int RS = 1024 / XW;  // staged rows per pass
  const int sx = threadIdx.x % XW, sy = threadIdx.x / XW;
  const int bx = threadIdx.x % LB, by = threadIdx.x / LB;
  if (sy < RS) {
    const int col = c0 - 5 + sx;
    const bool in = col >= 0 && col < w;
    const double* g3 = A.G3 + (int64_t)p * plane + col;
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll 4
      for (int r = sy; r < h; r += RS)
        G[k * HX + r * XW + sx] = in ? g3[k * tot + (int64_t)r * w] : 0.0;
  }
  __syncthreads();
  // adjoint along rows for every staged column (rows complete in smem)
  if (sy < RS) {
#pragma unroll
    for (int k = 0; k < 3; ++k)
      for (int r = sy; r < h; r += RS)
        Av[k * HX + r * XW + sx] = adj_fold(wv, G + k * HX + sx, XW, 0, h, r);
  }
  __syncthreads();
  const double n = (double)plane;
  const double inv_n = 1.0 / n, k_l1 = (1.0 - A.lam) / (n * A.S), k_ss = A.lam / A.S;
  for (int r = by; r < h && by < RB; r += RB) {
    const int c = bx, col = c0 + c;
    if (col >= w) continue;
    const double* row = Av + r * XW;
    // line index q = image column; element at (q - (c0 - 5))
    const double amx = adj_fold(wv, row, 1, c0 - 5, w, col);
    const double ab2 = adj_fold(wv, row + HX, 1, c0 - 5, w, col);
    const double aa2 = adj_fold(wv, row + 2 * HX, 1, c0 - 5, w, col);
    const double x = pred_at(A, b, s, r, col), y = gt_at(A, b, s, r, col);
    const double gssim = (amx + 2 * x * ab2 + y * aa2) * inv_n;
    const double diff = x - y;
    const double sgn = diff > 0 ? 1.0 : (diff < 0 ? -1.0 : 0.0);
    const double gp = sgn * k_l1 - k_ss * gssim;
    T* dz = A.dimg + (((int64_t)b * h + r) * w + col) * A.C;
    if (A.sup == 0) {  // (re, im) pairs: one 2-element load and store per pixel
      using T2 = typename std::conditional<sizeof(T) == 4, float2, double2>::type;
      const T2 zz = *(const T2*)(A.img + (((int64_t)b * h + r) * w + col) * A.C);
      const double re = zz.x, im = zz.y;
      const double m = hypot(re, im);
      const double kk = m > 0.0 ? gp / m : 0.0;
      T2 o;
      o.x = (T)(re * kk);
      o.y = (T)(im * kk);
      *(T2*)dz = o;
    } else {
      dz[s] = (T)gp;
    }
  }
}

template <typename T>
__global__ void k_loss_band_finalize(LossArgsT<T> A, int nbands) {
  // one warp per image: lanes take the band partials (all loads in flight),
  // then a fixed butterfly -- the same order on every run
  const int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (b >= A.NI) return;
  const double n = (double)A.h * A.w;
  double ss = 0.0, l1s = 0.0, sqs = 0.0, ss0 = 0.0, sq0 = 0.0;
  for (int s = 0; s < A.S; ++s) {
    const double* sm = A.sums + ((int64_t)b * A.S + s) * nbands * 3;
    double t[3] = {0.0, 0.0, 0.0};
    for (int k = lane; k < nbands; k += 32)
      for (int q = 0; q < 3; ++q) t[q] += sm[k * 3 + q];
    for (int q = 0; q < 3; ++q) t[q] = warp_sum(t[q]);
    ss += t[0] / n;
    l1s += t[1];
    sqs += t[2];
    if (s == 0) {
      ss0 = t[0] / n;
      sq0 = t[2] / n;
    }
  }
  if (lane) return;
  ss /= A.S;
  const double l1 = l1s / (n * A.S);
  double* o = A.stats + (int64_t)GSPARC_LOSS_STATS * b;
  o[0] = (1.0 - A.lam) * l1 + A.lam * (1.0 - ss);
  o[1] = l1;
  o[2] = ss;
  o[3] = sqs / (n * A.S);
  o[4] = ss0;  // channel 0 (optimize.py:281,293)
  o[5] = sq0;
}

int64_t loss_scratch_bytes(int NI, int h, int w, int C) {
  const int64_t tot = (int64_t)NI * C * h * w;  // upper bound: S <= C
  return (int64_t)sizeof(double) * (16 * tot + (int64_t)NI * C * 3 * LOSS_RB) + 256;
}

template <typename T>
static int run_loss(const T* img, const T* gt, int NI, int h, int w, int C, int sup, double lam,
                    T* dimg, double* stats, void* scratch, cudaStream_t st) {
  LossArgsT<T> A;
  make_window(A.win);
  A.img = img;
  A.gt = gt;
  A.dimg = dimg;
  A.NI = NI;
  A.S = sup == 0 ? 1 : C;
  A.C = C;
  A.h = h;
  A.w = w;
  A.sup = sup;
  A.lam = lam;
  A.stats = stats;
  const int64_t tot = (int64_t)NI * A.S * h * w;
  double* base = (double*)scratch;
  A.H5 = base;
  A.G3 = A.H5 + 5 * tot;
  A.A3 = A.G3 + 3 * tot;
  A.V3 = A.A3 + 3 * tot;
  A.XY = A.V3 + 3 * tot;
  A.sums = A.XY + 2 * tot;
  if (tot >= (int64_t)1 << 31) {
    set_error("loss: %lld pixels x channels exceed 2^31", (long long)tot);
    return GSPARC_ERR_UNSUPPORTED;
  }
  if (loss_band_smem(h) <= LOSS_SMEM_MAX && loss_adj_smem(h) <= LOSS_SMEM_MAX) {
    // banded path: G3 + per-band partial sums in the same scratch
    const int nb = loss_nbands(w);
    A.G3 = base;
    A.sums = base + 3 * tot;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_loss_band_fwd<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)LOSS_SMEM_MAX);
      cudaFuncSetAttribute(k_loss_band_adj<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)LOSS_SMEM_MAX);
      attr = true;
    }
    const dim3 grid((unsigned)nb, (unsigned)(NI * A.S));
    k_loss_band_fwd<T><<<grid, 1024, loss_band_smem(h), st>>>(A);
    k_loss_band_adj<T><<<grid, 1024, loss_adj_smem(h), st>>>(A);
    k_loss_band_finalize<T><<<(NI + 3) / 4, 128, 0, st>>>(A, nb);
    return check_launch("k_loss_band");
  }
  const unsigned blocks = (unsigned)((tot + 255) / 256);
  k_loss_prep<T><<<blocks, 256, 0, st>>>(A);
  k_loss_h<T><<<blocks, 256, 0, st>>>(A);
  k_loss_v<T><<<blocks, 256, 0, st>>>(A);
  k_loss_reduce<T><<<(unsigned)(NI * A.S * LOSS_RB), 256, 0, st>>>(A);
  k_loss_adj_v<T><<<blocks, 256, 0, st>>>(A);
  k_loss_adj_h<T><<<blocks, 256, 0, st>>>(A);
  k_loss_finalize<T><<<(NI + 127) / 128, 128, 0, st>>>(A);
  return check_launch("k_loss");
}

int launch_loss(const void* img, const void* gt, int dtype, int NI, int h, int w, int C, int sup,
                double lam, void* dimg, double* stats, void* scratch, int64_t scratch_bytes,
                cudaStream_t st) {
  if (sup == 0 && C != 2) {
    set_error("loss: magnitude supervision needs 2 channels, got %d", C);
    return GSPARC_ERR_ARG;
  }
  if (h < 6 || w < 6) {
    set_error("loss: image must be at least 6x6 for the 11-tap reflect window");
    return GSPARC_ERR_ARG;
  }
  if (scratch_bytes < loss_scratch_bytes(NI, h, w, C)) {
    set_error("loss: scratch too small");
    return GSPARC_ERR_ARG;
  }
  if (dtype == GSPARC_F64)
    return run_loss<double>((const double*)img, (const double*)gt, NI, h, w, C, sup, lam,
                            (double*)dimg, stats, scratch, st);
  return run_loss<float>((const float*)img, (const float*)gt, NI, h, w, C, sup, lam,
                         (float*)dimg, stats, scratch, st);
}

}  // namespace gs
