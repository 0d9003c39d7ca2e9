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
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float g = A.g[e];
    if (!isfinite(g)) bad |= 1 << group_of(e, A.n);
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

__global__ void k_adam(AdamArgs A, int64_t total) {
  // a frame whose pair buffer overflowed produced no valid gradient
  if (A.counters[GSPARC_CNT_NONFINITE] || A.counters[GSPARC_CNT_OVERFLOW]) return;
  // step scalars (pow, exp/log/sin of the position schedule) once per CTA
  __shared__ double s_sc[3];
  if (threadIdx.x == 0) {
    const int64_t step = *A.step;
    const double t = (double)(step + 1);
    s_sc[0] = 1.0 - pow(A.cfg.beta1, t);
    s_sc[1] = 1.0 - pow(A.cfg.beta2, t);
    s_sc[2] = position_lr_dev((double)step, A.cfg);
  }
  __syncthreads();
  const double b1 = A.cfg.beta1, b2 = A.cfg.beta2, eps = A.cfg.eps;
  const double bc1 = s_sc[0], bc2 = s_sc[1];
  const double lrs[5] = {s_sc[2], A.cfg.scaling_lr, A.cfg.rotation_lr, A.cfg.opacity_lr,
                         A.cfg.mlp_lr};
  const int64_t n = A.n;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int grp = group_of(e, n);
    const double g = (double)A.g[e];
    double m = b1 * (double)A.m[e] + (1.0 - b1) * g;
    double v = b2 * (double)A.v[e] + (1.0 - b2) * g * g;
    A.m[e] = (float)m;
    A.v[e] = (float)v;
    const double upd = lrs[grp] * (m / bc1) / (sqrt(v / bc2) + eps);
    switch (grp) {
      case 0: A.pos[e] -= upd; break;
      case 1: A.ls[e - 3 * n] -= upd; break;
      case 2: A.rot[e - 6 * n] -= upd; break;
      case 3: A.op[e - 10 * n] -= upd; break;
      default: A.mlp[e - 11 * n] = (float)((double)A.mlp[e - 11 * n] - upd); break;
    }
  }
}

__global__ void k_adam_finish(AdamArgs A) {
  const bool skip = A.counters[GSPARC_CNT_NONFINITE] != 0 || A.counters[GSPARC_CNT_OVERFLOW] != 0;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (!skip && i < A.n) {  // normalize_quaternions (scene.py:117-122)
    double* q = A.rot + 4 * i;
    const double nr = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    if (nr > 0.0) {
      q[0] /= nr;
      q[1] /= nr;
      q[2] /= nr;
      q[3] /= nr;
    } else {
      atomicOr(A.counters + GSPARC_CNT_NONFINITE, 1 << 5);
    }
  }
  if (!skip && i == 0) *A.step += 1;
}

int launch_adam(double* pos, double* ls, double* rot, double* op, float* mlp, int64_t n, int P,
                const float* g, float* m, float* v, int64_t* step, int* counters,
                const gsparc_adam_config& cfg, cudaStream_t st) {
  AdamArgs A{pos, ls, rot, op, mlp, g, m, v, step, counters, n, P, cfg};
  const int64_t total = n * (11 + (int64_t)P);
  if (cudaMemsetAsync(counters + GSPARC_CNT_NONFINITE, 0, sizeof(int), st) != cudaSuccess)
    return check_launch("adam memset");
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  k_check_finite<<<blocks, 256, 0, st>>>(A, total);
  k_adam<<<blocks, 256, 0, st>>>(A, total);
  k_adam_finish<<<(unsigned)((n + 255) / 256 > 0 ? (n + 255) / 256 : 1), 256, 0, st>>>(A);
  return check_launch("k_adam");
}

}  // namespace gs
