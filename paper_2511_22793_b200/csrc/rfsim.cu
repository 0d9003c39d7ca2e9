// K9 / K10: dataset-side kernels around the render path.
//
// K9  ground-truth spectra: the closed-form multipath oracle of
//     rfsim.ground_truth_spectrum (rfsim.py:75-99) for a batch of
//     transmitters.  One CTA row per TX; the per-(emitter, TX) terms
//     (unit direction, complex path amplitude, 1/(2 spread^2)) are computed
//     once per CTA into shared memory, then every thread owns pixels.
//     f64 throughout, in the reference's operation order (no FMA
//     contraction); cos/sin/acos/exp are CUDA's f64 routines (<= 1-2 ulp
//     from glibc), and the reference's `dirs @ unit` is a BLAS dgemv whose
//     summation order is not specified, so parity is tolerance based.
// K10 RSSI energies: rfsim.rssi_from_spectrum (rfsim.py:227-243) for a
//     batch of images sharing one pixel selection (the selection is the
//     reference's own PCG64 `choice`, drawn on the host): energy_b =
//     sum_{s in sel} |img_b[s]|^2 in f64, reduced in a fixed order (one CTA
//     per image), so the dB value needs 8 bytes of D2H per image instead of
//     the image.
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"

namespace gs {

constexpr int GT_T = 256;
constexpr int GT_EMAX = 256;  // emitters staged in shared memory per CTA

struct GtArgs {
  const gsparc_emitter* em;
  int ne;
  double rx[3];
  double wavelength;
  const double* tx;  // [B,3]
  int w, h;
  double scale;  // <= 0: none
  int out_f64;
  void* out;  // [B,h,w]
};

__global__ void __launch_bounds__(GT_T) k_gt_spectrum(GtArgs A) {
  __shared__ double s_u[GT_EMAX][3];     // unit direction rx -> emitter
  __shared__ double s_amp[GT_EMAX][2];   // gain * free-space amplitude (re, im)
  __shared__ double s_den[GT_EMAX];      // 2 spread^2
  __shared__ int s_ok[GT_EMAX];          // emitter not at the receiver
  const int b = blockIdx.y;
  const double* txb = A.tx + 3 * b;
  for (int e = threadIdx.x; e < A.ne; e += blockDim.x) {
    const gsparc_emitter E = A.em[e];
    // to_em = em.position - rx; r_em = |to_em| (rfsim.py:86-87)
    const double t0 = sub(E.position[0], A.rx[0]), t1 = sub(E.position[1], A.rx[1]),
                 t2 = sub(E.position[2], A.rx[2]);
    const double r_em = __dsqrt_rn(add(add(mul(t0, t0), mul(t1, t1)), mul(t2, t2)));
    s_ok[e] = r_em >= 1e-9;  // rfsim.py:88-90 (skipped with a warning)
    s_u[e][0] = t0 / r_em;
    s_u[e][1] = t1 / r_em;
    s_u[e][2] = t2 / r_em;
    // path = |em - tx| + r_em (rfsim.py:91)
    const double d0 = sub(E.position[0], txb[0]), d1 = sub(E.position[1], txb[1]),
                 d2 = sub(E.position[2], txb[2]);
    const double path = add(__dsqrt_rn(add(add(mul(d0, d0), mul(d1, d1)), mul(d2, d2))), r_em);
    // free_space_amplitude (rfsim.py:65-71): (l / (4 pi d)) exp(-2j pi d / l)
    const double pi = 3.141592653589793;
    const double mag = A.wavelength / mul(4.0 * pi, path);
    const double ph = mul(-2.0 * pi, path) / A.wavelength;
    double sn, cs;
    sincos(ph, &sn, &cs);
    const double fr = mul(mag, cs), fi = mul(mag, sn);
    // em.gain * amplitude, complex product (rfsim.py:92)
    s_amp[e][0] = sub(mul(E.gain_re, fr), mul(E.gain_im, fi));
    s_amp[e][1] = add(mul(E.gain_re, fi), mul(E.gain_im, fr));
    s_den[e] = 2.0 * mul(E.angular_spread, E.angular_spread);
  }
  __syncthreads();
  const int npx = A.w * A.h;
  const double pi = 3.141592653589793;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < npx; p += gridDim.x * blockDim.x) {
    const int v = p / A.w, u = p - v * A.w;
    // pixel_to_direction (geometry.py:83-95)
    const double az = mul(sub(add((double)u, 0.5) * 2.0 / (double)A.w, 1.0), pi);
    const double el = mul(add((double)v, 0.5), pi / 2.0) / (double)A.h;
    const double ce = cos(el);
    const double dx = mul(ce, sin(az)), dy = sin(el), dz = mul(ce, cos(az));
    double fre = 0.0, fim = 0.0;
    for (int e = 0; e < A.ne; ++e) {
      if (!s_ok[e]) continue;
      double c = add(add(mul(dx, s_u[e][0]), mul(dy, s_u[e][1])), mul(dz, s_u[e][2]));
      c = fmin(fmax(c, -1.0), 1.0);
      const double ang = acos(c);
      const double k = exp(mul(-ang, ang) / s_den[e]);
      fre = add(fre, mul(s_amp[e][0], k));
      fim = add(fim, mul(s_amp[e][1], k));
    }
    double m = hypot(fre, fim);  // np.abs (rfsim.py:96)
    if (A.scale > 0.0) m = m / A.scale;
    const int64_t o = (int64_t)b * npx + p;
    if (A.out_f64) ((double*)A.out)[o] = m;
    else ((float*)A.out)[o] = (float)m;
  }
}

int launch_gt_spectrum(const gsparc_emitter* em_dev, int ne, const double* rx, double wavelength,
                       const double* tx_dev, int B, int w, int h, double scale, int out_dtype,
                       void* out, cudaStream_t st) {
  if (ne < 1 || ne > GT_EMAX || B < 1 || w < 1 || h < 1 || !em_dev || !tx_dev || !out || !rx ||
      !(wavelength > 0.0) || (out_dtype != GSPARC_F32 && out_dtype != GSPARC_F64)) {
    set_error("gt_spectrum: invalid arguments (1 <= emitters <= %d, wavelength > 0)", GT_EMAX);
    return GSPARC_ERR_ARG;
  }
  GtArgs A;
  A.em = em_dev;
  A.ne = ne;
  for (int k = 0; k < 3; ++k) A.rx[k] = rx[k];
  A.wavelength = wavelength;
  A.tx = tx_dev;
  A.w = w;
  A.h = h;
  A.scale = scale;
  A.out_f64 = out_dtype == GSPARC_F64;
  A.out = out;
  const int npx = w * h;
  const int gx = min((npx + GT_T - 1) / GT_T, 64);
  k_gt_spectrum<<<dim3(gx, B), GT_T, 0, st>>>(A);
  return check_launch("k_gt_spectrum");
}

// ------------------------------------------------------------------ K10
constexpr int RS_THREADS = 512;

template <typename R>
__global__ void __launch_bounds__(RS_THREADS) k_rssi_energy(const R* img, int64_t npx, int C,
                                                           const int64_t* sel, int64_t nsel,
                                                           double* energy) {
  __shared__ double s_part[RS_THREADS / 32];
  const int b = blockIdx.x;
  const R* im = img + (int64_t)b * npx * C;
  double acc = 0.0;
  for (int64_t s = threadIdx.x; s < nsel; s += blockDim.x) {
    const int64_t q = sel[s];
    const double re = (double)im[q * C];
    double e = mul(re, re);  // rfsim.py:236-239
    if (C == 2) {
      const double imv = (double)im[q * C + 1];
      e = add(e, mul(imv, imv));
    }
    acc = add(acc, e);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < RS_THREADS / 32 ? s_part[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) energy[b] = v;
  }
}

int launch_rssi_energy(const void* img, int dtype, int B, int h, int w, int C, const int64_t* sel,
                       int64_t nsel, double* energy, cudaStream_t st) {
  if (!img || !sel || !energy || B < 1 || h < 1 || w < 1 || (C != 1 && C != 2) || nsel < 1 ||
      (dtype != GSPARC_F32 && dtype != GSPARC_F64)) {
    set_error("rssi_energy: invalid arguments (C must be 1 or 2)");
    return GSPARC_ERR_ARG;
  }
  const int64_t npx = (int64_t)h * w;
  if (dtype == GSPARC_F64)
    k_rssi_energy<double><<<B, RS_THREADS, 0, st>>>((const double*)img, npx, C, sel, nsel, energy);
  else
    k_rssi_energy<float><<<B, RS_THREADS, 0, st>>>((const float*)img, npx, C, sel, nsel, energy);
  return check_launch("k_rssi_energy");
}

}  // namespace gs
