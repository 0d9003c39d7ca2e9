// K8: Adam with per-group learning rates, annealed position LR and
// quaternion renormalisation.  Replaces optimize.adam_step
// (optimize.py:234-259), optimize.position_lr (optimize.py:205-213) and the
// ParamGradients.check_finite gate (rasterizer.py:63-66): if any gradient is
// non-finite no parameter moves and the bitmask of offending groups is
// published in counters[GSPARC_CNT_NONFINITE] (bit g = group g), which the
// host turns into FloatingPointError naming the first group.
// The zero-based step lives on the device so the whole train step can be
// captured in a CUDA graph.
#include "common.cuh"
#include "kernels.cuh"

namespace gs {

struct AdamArgs {
  double* pos;
  double* ls;
  double* rot;
  double* op;
  float* mlp;
  const float* g;
  float* m;
  float* v;
  int64_t* step;
  int* counters;
  int64_t n;
  int P;
  gsparc_adam_config cfg;
};

__device__ __forceinline__ int group_of(int64_t e, int64_t n) {
  if (e < 3 * n) return 0;
  if (e < 6 * n) return 1;
  if (e < 10 * n) return 2;
  if (e < 11 * n) return 3;
  return 4;
}

__global__ void k_check_finite(AdamArgs A, int64_t total) {
  int bad = 0;
  // float4 over the flat buffer (group boundaries resolved per element)
  const int64_t n4 = total >> 2;
  const float4* g4 = reinterpret_cast<const float4*>(A.g);
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n4;
       q += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = g4[q];
    const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (!isfinite(x[k])) bad |= 1 << group_of(4 * q + k, A.n);
  }
  for (int64_t e = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (!isfinite(A.g[e])) bad |= 1 << group_of(e, A.n);
  }
  bad = __reduce_or_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicOr(A.counters + GSPARC_CNT_NONFINITE, bad);
}

__device__ double position_lr_dev(double step, const gsparc_adam_config& c) {
  double t = step / c.position_lr_max_steps;
  t = fmin(fmax(t, 0.0), 1.0);
  const double lr = exp((1.0 - t) * log(c.position_lr_init) + t * log(c.position_lr_final));
  double ramp = step / (0.01 * c.position_lr_max_steps);
  ramp = fmin(fmax(ramp, 0.0), 1.0);
  const double delay = c.position_lr_delay_mult +
                       (1.0 - c.position_lr_delay_mult) * sin(0.5 * 3.141592653589793 * ramp);
  return delay * lr;
}

__device__ __forceinline__ double adam_upd(double g, float& m, float& v, double lr, double b1,
                                           double b2, double bc1, double bc2, double eps) {
  const double mm = b1 * (double)m + (1.0 - b1) * g;
  const double vv = b2 * (double)v + (1.0 - b2) * g * g;
  m = (float)mm;
  v = (float)vv;
  return lr * (mm / bc1) / (sqrt(vv / bc2) + eps);
}

// Blocks [0, geo_blocks): the geometry (f64): a thread per position,
// log-scale and opacity element, a thread per Gaussian's rotation; the
// remaining blocks: the MLP weights, 4 per thread.
__global__ void k_adam(AdamArgs A, int64_t total, int geo_blocks) {
  // a frame whose pair buffer overflowed produced no valid gradient
  if (A.counters[GSPARC_CNT_NONFINITE] || A.counters[GSPARC_CNT_OVERFLOW]) return;
  // step scalars once per CTA: the two bias corrections on two threads, the
  // position schedule (f64 exp/log/sin) on a third and only in the geometry
  // blocks (the MLP blocks' CTAs start their loads sooner)
  __shared__ double s_sc[3];
  if (threadIdx.x < 3) {
    const int64_t step = *A.step;
    const double t = (double)(step + 1);
    if (threadIdx.x == 0) s_sc[0] = 1.0 - pow(A.cfg.beta1, t);
    if (threadIdx.x == 1) s_sc[1] = 1.0 - pow(A.cfg.beta2, t);
    if (threadIdx.x == 2 && (int)blockIdx.x < geo_blocks)
      s_sc[2] = position_lr_dev((double)step, A.cfg);
  }
  __syncthreads();
  const double b1 = A.cfg.beta1, b2 = A.cfg.beta2, eps = A.cfg.eps;
  const double bc1 = s_sc[0], bc2 = s_sc[1];
  const int64_t n = A.n;
  if ((int)blockIdx.x < geo_blocks) {
    // geometry, f64: thread per position / log-scale / opacity element
    // (t < 7n), thread per Gaussian for the rotations (renormalised right
    // after their update, scene.py:117-122)
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < 3 * n) {
      A.pos[t] -= adam_upd((double)A.g[t], A.m[t], A.v[t], s_sc[2], b1, b2, bc1, bc2, eps);
    } else if (t < 6 * n) {
      A.ls[t - 3 * n] -=
          adam_upd((double)A.g[t], A.m[t], A.v[t], A.cfg.scaling_lr, b1, b2, bc1, bc2, eps);
    } else if (t < 7 * n) {
      const int64_t i = t - 6 * n, e = 10 * n + i;
      A.op[i] -= adam_upd((double)A.g[e], A.m[e], A.v[e], A.cfg.opacity_lr, b1, b2, bc1, bc2, eps);
    } else if (t < 8 * n) {
      const int64_t i = t - 7 * n;
      double q[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t e = 6 * n + 4 * i + k;
        q[k] = A.rot[4 * i + k] -
               adam_upd((double)A.g[e], A.m[e], A.v[e], A.cfg.rotation_lr, b1, b2, bc1, bc2, eps);
      }
      const double nr = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
      if (nr > 0.0) {
        for (int k = 0; k < 4; ++k) A.rot[4 * i + k] = q[k] / nr;
      } else {
        for (int k = 0; k < 4; ++k) A.rot[4 * i + k] = q[k];
        atomicOr(A.counters + GSPARC_CNT_NONFINITE, 1 << 5);
      }
    }
    return;
  }
  // MLP weights: flat range [11n, total), 4 consecutive elements per thread
  const int64_t base = 11 * n;
  const int64_t cnt = total - base;
  const int64_t q = ((int64_t)blockIdx.x - geo_blocks) * blockDim.x + threadIdx.x;
  const int64_t e0 = base + 4 * q;
  if (4 * q >= cnt) return;
  const double lr = A.cfg.mlp_lr;
  // all loads of the 4 elements first, then 4 independent f64 chains
  const int kn = (int)min((int64_t)4, cnt - 4 * q);
  float gv[4], mv[4], vv[4], wv[4];
  // 16-byte vectors when the MLP block of the flat buffer is aligned
  // (11 n % 4 == 0) and all four elements exist
  const bool vec = ((base & 3) == 0) && kn == 4;
  if (vec) {
    const float4 g4 = *reinterpret_cast<const float4*>(A.g + e0);
    const float4 m4 = *reinterpret_cast<const float4*>(A.m + e0);
    const float4 v4 = *reinterpret_cast<const float4*>(A.v + e0);
    const float4 w4 = *reinterpret_cast<const float4*>(A.mlp + (e0 - base));
    gv[0] = g4.x; gv[1] = g4.y; gv[2] = g4.z; gv[3] = g4.w;
    mv[0] = m4.x; mv[1] = m4.y; mv[2] = m4.z; mv[3] = m4.w;
    vv[0] = v4.x; vv[1] = v4.y; vv[2] = v4.z; vv[3] = v4.w;
    wv[0] = w4.x; wv[1] = w4.y; wv[2] = w4.z; wv[3] = w4.w;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < kn) {
        gv[k] = A.g[e0 + k];
        mv[k] = A.m[e0 + k];
        vv[k] = A.v[e0 + k];
        wv[k] = A.mlp[e0 + k - base];
      }
    }
  }
  // f32 moments and update for the f32 weights (the stored m, v are f32;
  // the update's f32 rounding, ~1e-7 relative, is far inside the 1e-6
  // parameter tolerance); the f64 geometry above keeps f64 arithmetic
  const float b1f = (float)b1, b2f = (float)b2, ib1 = (float)(1.0 / bc1),
              ib2 = (float)(1.0 / bc2), lrf = (float)lr, epsf = (float)eps;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (k < kn) {
      const float g = gv[k];
      const float mm = b1f * mv[k] + (1.f - b1f) * g;
      const float v2 = b2f * vv[k] + (1.f - b2f) * g * g;
      mv[k] = mm;
      vv[k] = v2;
      wv[k] -= lrf * (mm * ib1) / (sqrtf(v2 * ib2) + epsf);
    }
  }
  if (vec) {
    *reinterpret_cast<float4*>(A.m + e0) = make_float4(mv[0], mv[1], mv[2], mv[3]);
    *reinterpret_cast<float4*>(A.v + e0) = make_float4(vv[0], vv[1], vv[2], vv[3]);
    *reinterpret_cast<float4*>(A.mlp + (e0 - base)) = make_float4(wv[0], wv[1], wv[2], wv[3]);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < kn) {
        A.m[e0 + k] = mv[k];
        A.v[e0 + k] = vv[k];
        A.mlp[e0 + k - base] = wv[k];
      }
    }
  }
}

__global__ void k_adam_finish(AdamArgs A) {
  const bool skip = A.counters[GSPARC_CNT_NONFINITE] != 0 || A.counters[GSPARC_CNT_OVERFLOW] != 0;
  if (!skip) *A.step += 1;
}

int launch_adam(double* pos, double* ls, double* rot, double* op, float* mlp, int64_t n, int P,
                const float* g, float* m, float* v, int64_t* step, int* counters,
                const gsparc_adam_config& cfg, cudaStream_t st) {
  AdamArgs A{pos, ls, rot, op, mlp, g, m, v, step, counters, n, P, cfg};
  const int64_t total = n * (11 + (int64_t)P);
  if (cudaMemsetAsync(counters + GSPARC_CNT_NONFINITE, 0, sizeof(int), st) != cudaSuccess)
    return check_launch("adam memset");
  int blocks = (int)((total / 4 + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_check_finite<<<blocks, 256, 0, st>>>(A, total);
  const int geo_blocks = (int)((8 * n + 255) / 256);
  const int64_t mlp4 = (n * (int64_t)P + 3) / 4;
  const int mlp_blocks = (int)((mlp4 + 255) / 256);
  if (geo_blocks + mlp_blocks > 0) k_adam<<<geo_blocks + mlp_blocks, 256, 0, st>>>(A, total, geo_blocks);
  k_adam_finish<<<1, 1, 0, st>>>(A);
  return check_launch("k_adam");
}

}  // namespace gs
