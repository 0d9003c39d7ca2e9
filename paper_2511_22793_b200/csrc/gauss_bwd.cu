// K6: per-Gaussian backward chain, one warp per Gaussian.
// Replaces rasterizer.py:328-377 with geometry.equirect_jacobian_deriv
// (geometry.py:152-180), scene.rotation_backward (scene.py:142-173),
// mlp.batch_mlp_backward (mlp.py:48-70) and mlp.direction_angles_backward
// (mlp.py:92-103).  Inputs are the screen-space accumulators of K5
// (dL/dcoef per TX, dL/d conic, dL/d mean2d, dL/d sigma); the chain runs in
// f64 and writes the flat gradient buffer
//   positions(n,3) | log_scales(n,3) | rotations(n,4) | raw_opacities(n) |
//   mlp_weights(n,P)
// (the ParamGradients groups of rasterizer.py:39-61), overwriting it.
// Culled Gaussians, and on f32 frames those no pixel included, get exact
// zeros.  TX batches sum their gradients.
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace gs {

struct GBwdArgs {
  gsparc_cloud cloud;
  Pose pose;
  GeoConst gc;
  const double* tx;
  int B;
  const uint64_t* key;
  const float4* rec32;
  const double* rec64;
  const void* gcoef;  // [n, Cp] frame dtype
  const void* ggeo;   // [n, 8] frame dtype
  void* grad;         // flat, grad dtype
  int64_t Cp;
  int P;
  int lane_tx;  // (5,16,C<=16) head: lane-per-TX MLP backward
  // f32 frames: pass A's live flags (the Gaussian was included at some
  // pixel); a Gaussian no pixel included has dL/dcoef = 0 for every TX and
  // zero screen-space gradients, so every parameter gradient is exactly 0
  const int* live;
};

constexpr int LANE_TX_JMAX = 12;  // flat MLP rows up to 384 parameters

template <typename G>
__device__ __forceinline__ void put(G* base, int64_t k, double v) {
  base[k] = (G)v;
}

// FR: frame / weight precision (float or double); G: gradient dtype.
template <typename FR, typename G>
__global__ void __launch_bounds__(128, 4) k_gauss_bwd(GBwdArgs A) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int C = A.cloud.mlp_out, H = A.cloud.mlp_hidden, I = A.cloud.mlp_in, P = A.P;
  // per-warp scratch: x[8] hid[32] pre[32] gpre[32] gs[C] acc[P] (the
  // weight gradients summed over TX, in f64 shared memory)
  double* sw = (double*)smraw +
               (size_t)warp * (A.lane_tx ? (size_t)32 * (2 * 17 + 6 + C + 1) : (size_t)(8 + 96 + C + P));
  double* s_x = sw;
  double* s_hid = sw + 8;
  double* s_pre = sw + 40;
  double* s_gpre = sw + 72;
  double* s_gs = sw + 104;
  double* s_acc = s_gs + C;
  if (i >= A.cloud.n) return;
  const int64_t n = A.cloud.n;
  G* g = (G*)A.grad;
  G* g_pos = g;
  G* g_ls = g + 3 * n;
  G* g_rot = g + 6 * n;
  G* g_op = g + 10 * n;
  G* g_w = g + 11 * n + i * (int64_t)P;
  if (A.key[i] == ~0ULL || (A.live && !A.live[i])) {  // culled, or included nowhere
    if (lane < 3) put(g_pos, 3 * i + lane, 0.0);
    if (lane < 3) put(g_ls, 3 * i + lane, 0.0);
    if (lane < 4) put(g_rot, 4 * i + lane, 0.0);
    if (lane == 0) put(g_op, i, 0.0);
    for (int e = lane; e < P; e += 32) g_w[e] = (G)0;
    return;
  }
  double theta, phi;
  if constexpr (sizeof(FR) == 4) {
    const float4 r = A.rec32[2 * i + 1];
    theta = r.z;
    phi = r.w;
  } else {
    theta = A.rec64[8 * i + 6];
    phi = A.rec64[8 * i + 7];
  }
  const FR* w = (sizeof(FR) == 4) ? (const FR*)(A.cloud.mlp_weights + i * (int64_t)P)
                                  : (const FR*)(A.cloud.mlp_weights64 + i * (int64_t)P);
  const FR* W1 = w;
  const FR* b1 = w + H * I;
  const FR* W2 = b1 + H;
  const FR* b2 = W2 + C * H;
  const FR* gcoef = (const FR*)A.gcoef + i * A.Cp;
  const double* pos = A.cloud.positions + 3 * i;
  double g_theta = 0.0, g_phi = 0.0, gpd0 = 0.0, gpd1 = 0.0, gpd2 = 0.0;
  if (A.lane_tx) {
    // ---- MLP backward, lane = TX (mlp.py:48-70 for the (5,16,C) head).
    // Each lane runs its transmitter's forward + backward in registers;
    // the weight gradients sum_b gpre_b (x) x_b, gs_b (x) hid_b are then
    // 32-term dots over the lanes' rows staged in shared memory, owned by
    // lane e (mod 32) of the flat parameter row, accumulated in registers.
    // MT: f32 for the training path (f32 frame and gradients: the sums run
    // over <= 32 TX, ~1e-7 relative), f64 otherwise (the drop-in's f64
    // gradients follow the reference's f64 mlp.batch_mlp_backward)
    using MT = std::conditional_t<sizeof(FR) == 4 && sizeof(G) == 4, float, double>;
    constexpr int H16 = 16, I5 = 5, JMAX = LANE_TX_JMAX;
    MT* t_gp = reinterpret_cast<MT*>(smraw) +
               (size_t)warp * 32 * (2 * (H16 + 1) + I5 + 1 + C + 1);  // [32][17] dL/d pre
    MT* t_hid = t_gp + 32 * (H16 + 1);  // [32][17] hidden
    MT* t_x = t_hid + 32 * (H16 + 1);   // [32][6]  inputs
    MT* t_gs = t_x + 32 * (I5 + 1);     // [32][C+1] dL/d s
    const int CP1 = C + 1;
    MT acc[JMAX];
#pragma unroll
    for (int j = 0; j < JMAX; ++j) acc[j] = MT(0);
    MT gth = 0, gph = 0, gq0 = 0, gq1 = 0, gq2 = 0;
    for (int b0 = 0; b0 < A.B; b0 += 32) {
      const int b = b0 + lane;
      const bool vb = b < A.B;
      MT x[I5], hid[H16], gh[H16];
      x[3] = (MT)theta;
      x[4] = (MT)phi;
      MT d0 = 0, d1 = 0, d2 = 0, draw = 1, d = 1;
      if (vb) {
        const double* txb = A.tx + 3 * b;
        x[0] = (MT)(FR)txb[0];
        x[1] = (MT)(FR)txb[1];
        x[2] = (MT)(FR)txb[2];
        d0 = (MT)(pos[0] - txb[0]);
        d1 = (MT)(pos[1] - txb[1]);
        d2 = (MT)(pos[2] - txb[2]);
        draw = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
        d = draw < (MT)NEAR_PLANE ? (MT)NEAR_PLANE : draw;
      } else {
        x[0] = x[1] = x[2] = MT(0);
      }
#pragma unroll
      for (int h = 0; h < H16; ++h) {
        MT v = 0;
#pragma unroll
        for (int k = 0; k < I5; ++k) v += (MT)W1[h * I5 + k] * x[k];
        v += (MT)b1[h];
        hid[h] = v > MT(0) ? v : MT(0);
        gh[h] = 0;
      }
      MT gd_part = 0;
      for (int c = 0; c < C; ++c) {
        MT sc = 0;
#pragma unroll
        for (int h = 0; h < H16; ++h) sc += (MT)W2[c * H16 + h] * hid[h];
        sc += (MT)b2[c];
        const MT gcv = vb ? (MT)gcoef[(int64_t)b * C + c] : MT(0);
        const MT gsc = gcv / d;
        gd_part -= gcv * sc;
#pragma unroll
        for (int h = 0; h < H16; ++h) gh[h] += (MT)W2[c * H16 + h] * gsc;
        t_gs[lane * CP1 + c] = gsc;
      }
      const MT g_d = gd_part / (d * d);
      if (vb && !(draw < (MT)NEAR_PLANE)) {  // rasterizer.py:366-368
        gq0 += g_d * d0 / d;
        gq1 += g_d * d1 / d;
        gq2 += g_d * d2 / d;
      }
#pragma unroll
      for (int h = 0; h < H16; ++h) {
        const MT gp = hid[h] > MT(0) ? gh[h] : MT(0);  // relu' (pre > 0 <=> hid > 0)
        gth += (MT)W1[h * I5 + 3] * gp;
        gph += (MT)W1[h * I5 + 4] * gp;
        t_gp[lane * (H16 + 1) + h] = gp;
        t_hid[lane * (H16 + 1) + h] = vb ? hid[h] : MT(0);
      }
#pragma unroll
      for (int k = 0; k < I5; ++k) t_x[lane * (I5 + 1) + k] = x[k];
      __syncwarp();
      const int nl = min(32, A.B - b0);
#pragma unroll
      for (int j = 0; j < JMAX; ++j) {
        const int e = lane + 32 * j;
        if (e >= P) break;
        MT v = 0;
        if (e < H16 * I5) {
          const int h = e / I5, k = e - h * I5;
          for (int l = 0; l < nl; ++l) v += t_gp[l * (H16 + 1) + h] * t_x[l * (I5 + 1) + k];
        } else if (e < H16 * I5 + H16) {
          const int h = e - H16 * I5;
          for (int l = 0; l < nl; ++l) v += t_gp[l * (H16 + 1) + h];
        } else if (e < H16 * I5 + H16 + C * H16) {
          const int f = e - H16 * I5 - H16, c = f / H16, h = f - c * H16;
          for (int l = 0; l < nl; ++l) v += t_gs[l * CP1 + c] * t_hid[l * (H16 + 1) + h];
        } else {
          const int c = e - H16 * I5 - H16 - C * H16;
          for (int l = 0; l < nl; ++l) v += t_gs[l * CP1 + c];
        }
        acc[j] += v;
      }
      __syncwarp();
    }
#pragma unroll
    for (int j = 0; j < JMAX; ++j) {
      const int e = lane + 32 * j;
      if (e < P) g_w[e] = (G)acc[j];
    }
    g_theta = warp_sum(gth);
    g_phi = warp_sum(gph);
    gpd0 = warp_sum(gq0);
    gpd1 = warp_sum(gq1);
    gpd2 = warp_sum(gq2);
  } else {
  for (int e = lane; e < P; e += 32) s_acc[e] = 0.0;
    double acc_gpre = 0.0;  // lane h: sum over TX of dL/d pre_h
  
    for (int b = 0; b < A.B; ++b) {
      const double* txb = A.tx + 3 * b;
      if (lane < 5) s_x[lane] = lane < 3 ? (double)(FR)txb[lane] : (lane == 3 ? theta : phi);
      __syncwarp();
      if (lane < H) {
        double pre = 0.0;
        for (int k = 0; k < I; ++k) pre += (double)W1[lane * I + k] * s_x[k];
        pre += (double)b1[lane];
        s_pre[lane] = pre;
        s_hid[lane] = pre > 0.0 ? pre : 0.0;
      }
      __syncwarp();
      const double d0 = pos[0] - txb[0], d1 = pos[1] - txb[1], d2 = pos[2] - txb[2];
      const double draw = sqrt(d0 * d0 + d1 * d1 + d2 * d2);
      const double d = draw < NEAR_PLANE ? NEAR_PLANE : draw;
      // s_c, g_s = dL/dcoef / d,  g_d = -sum_c dL/dcoef_c * s_c / d^2
      double gd_part = 0.0;
      for (int c = lane; c < C; c += 32) {
        double s = 0.0;
        for (int h = 0; h < H; ++h) s += (double)W2[c * H + h] * s_hid[h];
        s += (double)b2[c];
        const double gcv = (double)gcoef[(int64_t)b * C + c];
        s_gs[c] = gcv / d;
        gd_part -= gcv * s;
      }
      const double g_d = warp_sum(gd_part) / (d * d);
      __syncwarp();
      if (lane < H) {
        double gh = 0.0;
        for (int c = 0; c < C; ++c) gh += (double)W2[c * H + lane] * s_gs[c];
        s_gpre[lane] = s_pre[lane] > 0.0 ? gh : 0.0;
        acc_gpre += s_gpre[lane];
      }
      __syncwarp();
      if (lane == 0) {
        if (!(draw < NEAR_PLANE)) {  // rasterizer.py:366-368
          gpd0 += g_d * d0 / d;
          gpd1 += g_d * d1 / d;
          gpd2 += g_d * d2 / d;
        }
      }
      // weight gradients: W1 | b1 | W2 | b2 (mlp.py:58-66), summed over TX
      for (int e = lane; e < P; e += 32) {
        double v;
        if (e < H * I) {
          v = s_gpre[e / I] * s_x[e % I];
        } else if (e < H * I + H) {
          v = s_gpre[e - H * I];
        } else if (e < H * I + H + C * H) {
          const int f = e - H * I - H;
          v = s_gs[f / H] * s_hid[f % H];
        } else {
          v = s_gs[e - H * I - H - C * H];
        }
        s_acc[e] += v;
      }
      __syncwarp();
    }
    for (int e = lane; e < P; e += 32) g_w[e] = (G)s_acc[e];
    // angle gradients: sum_h W1[h, 3|4] * sum_b gpre_b[h] (mlp.py:58-70)
    {
      const double a3 = lane < H ? (double)W1[lane * I + 3] * acc_gpre : 0.0;
      const double a4 = lane < H ? (double)W1[lane * I + 4] * acc_gpre : 0.0;
      g_theta = warp_sum(a3);
      g_phi = warp_sum(a4);
    }
  }
  // the per-Gaussian geometry chain runs in k_gauss_geo (thread per
  // Gaussian); its MLP-side inputs are parked in this Gaussian's own
  // g_pos / g_ls slots, which that kernel overwrites
  if (lane == 0) {
    put(g_pos, 3 * i + 0, gpd0);
    put(g_pos, 3 * i + 1, gpd1);
    put(g_pos, 3 * i + 2, gpd2);
    put(g_ls, 3 * i + 0, g_theta);
    put(g_ls, 3 * i + 1, g_phi);
  }
}

// K6b: the per-Gaussian geometry chain (f64), one thread per Gaussian.
template <typename FR, typename G>
__global__ void __launch_bounds__(128) k_gauss_geo(GBwdArgs A) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.cloud.n) return;
  if (A.key[i] == ~0ULL || (A.live && !A.live[i])) return;  // zeros written by k_gauss_bwd
  const int64_t n = A.cloud.n;
  G* g = (G*)A.grad;
  G* g_pos = g;
  G* g_ls = g + 3 * n;
  G* g_rot = g + 6 * n;
  G* g_op = g + 10 * n;
  const double* pos = A.cloud.positions + 3 * i;
  const double gpd0 = (double)g_pos[3 * i + 0], gpd1 = (double)g_pos[3 * i + 1],
               gpd2 = (double)g_pos[3 * i + 2];
  const double g_theta = (double)g_ls[3 * i + 0], g_phi = (double)g_ls[3 * i + 1];
  const double* W = A.pose.W;
  const double p0 = pos[0] - A.pose.rx[0], p1 = pos[1] - A.pose.rx[1], p2 = pos[2] - A.pose.rx[2];
  const double x = p0 * W[0] + p1 * W[1] + p2 * W[2];
  const double y = p0 * W[3] + p1 * W[4] + p2 * W[5];
  const double z = p0 * W[6] + p1 * W[7] + p2 * W[8];
  const double r2u = x * x + y * y + z * z;
  const double ru = sqrt(r2u);
  const double el = asin(fmin(fmax(y / ru, -1.0), 1.0));
  double jx = x, jy = y, jz = z;
  if (el > A.gc.pole_lim) {  // _clamp_pole (geometry.py:98-113)
    const double az = atan2(x, z);
    const double tr = ru * A.gc.cos_lim;
    jx = tr * sin(az);
    jy = ru * A.gc.sin_lim;
    jz = tr * cos(az);
  }
  const double rho2 = jx * jx + jz * jz;
  const double rho = sqrt(rho2);
  const double r2 = rho2 + jy * jy;
  const double r4 = r2 * r2;
  const double ca = A.gc.ca, ce = A.gc.ce;
  double J[2][3];
  J[0][0] = ca * jz / rho2;
  J[0][1] = 0.0;
  J[0][2] = -ca * jx / rho2;
  J[1][0] = -ce * jx * jy / (r2 * rho);
  J[1][1] = ce * rho / r2;
  J[1][2] = -ce * jy * jz / (r2 * rho);
  // Hessian H[k][a][b] (geometry.py:167-179)
  double Hs[2][3][3] = {};
  const double rho4 = rho2 * rho2;
  Hs[0][0][0] = ca * (-2.0 * jx * jz / rho4);
  Hs[0][0][2] = Hs[0][2][0] = ca * (jx * jx - jz * jz) / rho4;
  Hs[0][2][2] = ca * (2.0 * jx * jz / rho4);
  const double Acoef = 2.0 / (r4 * rho) + 1.0 / (r2 * rho * rho2);
  Hs[1][0][0] = ce * (-jy / (r2 * rho) + jx * jx * jy * Acoef);
  Hs[1][0][1] = Hs[1][1][0] = ce * (-jx * (r2 - 2.0 * jy * jy) / (r4 * rho));
  Hs[1][0][2] = Hs[1][2][0] = ce * (jx * jy * jz * Acoef);
  Hs[1][1][1] = ce * (-2.0 * rho * jy / r4);
  Hs[1][1][2] = Hs[1][2][1] = ce * (jz * (jy * jy - rho2) / (rho * r4));
  Hs[1][2][2] = ce * (-jy / (r2 * rho) + jz * jz * jy * Acoef);

  // Sigma, R, scales (scene.py:84-88)
  const double* qr = A.cloud.rotations + 4 * i;
  const double qn = sqrt(qr[0] * qr[0] + qr[1] * qr[1] + qr[2] * qr[2] + qr[3] * qr[3]);
  const double qw = qr[0] / qn, qx = qr[1] / qn, qy = qr[2] / qn, qz = qr[3] / qn;
  double R[3][3];
  R[0][0] = 1 - 2 * (qy * qy + qz * qz);
  R[0][1] = 2 * (qx * qy - qw * qz);
  R[0][2] = 2 * (qx * qz + qw * qy);
  R[1][0] = 2 * (qx * qy + qw * qz);
  R[1][1] = 1 - 2 * (qx * qx + qz * qz);
  R[1][2] = 2 * (qy * qz - qw * qx);
  R[2][0] = 2 * (qx * qz - qw * qy);
  R[2][1] = 2 * (qy * qz + qw * qx);
  R[2][2] = 1 - 2 * (qx * qx + qy * qy);
  const double* ls = A.cloud.log_scales + 3 * i;
  const double sc[3] = {exp(ls[0]), exp(ls[1]), exp(ls[2])};
  double M[3][3], S[3][3], M3[3][3], tmp[3][3];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) M[a][c] = R[a][c] * sc[c];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) S[a][c] = M[a][0] * M[c][0] + M[a][1] * M[c][1] + M[a][2] * M[c][2];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c)
      tmp[a][c] = W[3 * a] * S[0][c] + W[3 * a + 1] * S[1][c] + W[3 * a + 2] * S[2][c];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c)
      M3[a][c] = tmp[a][0] * W[3 * c] + tmp[a][1] * W[3 * c + 1] + tmp[a][2] * W[3 * c + 2];
  // conic from cov2d
  double JM[2][3];
  for (int a = 0; a < 2; ++a)
    for (int c = 0; c < 3; ++c)
      JM[a][c] = J[a][0] * M3[0][c] + J[a][1] * M3[1][c] + J[a][2] * M3[2][c];
  double cov[2][2];
  for (int a = 0; a < 2; ++a)
    for (int c = 0; c < 2; ++c)
      cov[a][c] = JM[a][0] * J[c][0] + JM[a][1] * J[c][1] + JM[a][2] * J[c][2];
  const double ka = cov[0][0] + COV2D_REG, kb = 0.5 * (cov[0][1] + cov[1][0]),
               kc = cov[1][1] + COV2D_REG;
  const double det = ka * kc - kb * kb;
  const double Am[2][2] = {{kc / det, -kb / det}, {-kb / det, ka / det}};

  const FR* gg = (const FR*)A.ggeo + 8 * i;
  const double GA[2][2] = {{(double)gg[0], (double)gg[1]}, {(double)gg[1], (double)gg[2]}};
  const double gm0 = gg[3], gm1 = gg[4], gsig = gg[5];
  // G_cov2d = -A G_A A
  double AG[2][2], G2[2][2];
  for (int a = 0; a < 2; ++a)
    for (int c = 0; c < 2; ++c) AG[a][c] = Am[a][0] * GA[0][c] + Am[a][1] * GA[1][c];
  for (int a = 0; a < 2; ++a)
    for (int c = 0; c < 2; ++c) G2[a][c] = -(AG[a][0] * Am[0][c] + AG[a][1] * Am[1][c]);
  // G_M3 = J^T G2 J ; G_J = 2 G2 J M3
  double GJt[2][3], GM3[3][3], GJ[2][3];
  for (int a = 0; a < 2; ++a)
    for (int c = 0; c < 3; ++c) GJt[a][c] = G2[a][0] * J[0][c] + G2[a][1] * J[1][c];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c) GM3[a][c] = J[0][a] * GJt[0][c] + J[1][a] * GJt[1][c];
  for (int a = 0; a < 2; ++a)
    for (int c = 0; c < 3; ++c)
      GJ[a][c] = 2.0 * (GJt[a][0] * M3[0][c] + GJt[a][1] * M3[1][c] + GJt[a][2] * M3[2][c]);
  double gmu[3] = {0.0, 0.0, 0.0};
  for (int q = 0; q < 3; ++q)
    for (int k = 0; k < 2; ++k)
      for (int c = 0; c < 3; ++c) gmu[q] += GJ[k][c] * Hs[k][c][q];
  // G_Sigma = W^T G_M3 W ; G_M = 2 G_Sigma M
  double GS[3][3], GM[3][3];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c)
      tmp[a][c] = GM3[0][c] * W[a] + GM3[1][c] * W[3 + a] + GM3[2][c] * W[6 + a];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c)
      GS[a][c] = tmp[a][0] * W[c] + tmp[a][1] * W[3 + c] + tmp[a][2] * W[6 + c];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c)
      GM[a][c] = 2.0 * (GS[a][0] * M[0][c] + GS[a][1] * M[1][c] + GS[a][2] * M[2][c]);
  double gls[3], GR[3][3];
  for (int c = 0; c < 3; ++c) {
    gls[c] = (R[0][c] * GM[0][c] + R[1][c] * GM[1][c] + R[2][c] * GM[2][c]) * sc[c];
    for (int a = 0; a < 3; ++a) GR[a][c] = GM[a][c] * sc[c];
  }
  // rotation_backward (scene.py:142-173)
  double gw = 2 * (-qz * GR[0][1] + qy * GR[0][2] + qz * GR[1][0] - qx * GR[1][2] -
                   qy * GR[2][0] + qx * GR[2][1]);
  double gxq = 2 * (qy * GR[0][1] + qz * GR[0][2] + qy * GR[1][0] - 2 * qx * GR[1][1] -
                    qw * GR[1][2] + qz * GR[2][0] + qw * GR[2][1] - 2 * qx * GR[2][2]);
  double gyq = 2 * (-2 * qy * GR[0][0] + qx * GR[0][1] + qw * GR[0][2] + qx * GR[1][0] +
                    qz * GR[1][2] - qw * GR[2][0] + qz * GR[2][1] - 2 * qy * GR[2][2]);
  double gzq = 2 * (-2 * qz * GR[0][0] - qw * GR[0][1] + qx * GR[0][2] + qw * GR[1][0] -
                    2 * qz * GR[1][1] + qy * GR[1][2] + qx * GR[2][0] + qy * GR[2][1]);
  const double dotq = gw * qw + gxq * qx + gyq * qy + gzq * qz;
  const double gq[4] = {(gw - qw * dotq) / qn, (gxq - qx * dotq) / qn, (gyq - qy * dotq) / qn,
                        (gzq - qz * dotq) / qn};
  // angles backward (mlp.py:92-103), unclamped mu_v
  {
    const double rho2u = x * x + z * z;
    const double rhou = sqrt(rho2u);
    const double r2a = rho2u + y * y;
    gmu[0] += g_theta * (z / rho2u) + g_phi * (-x * y / (r2a * rhou));
    gmu[1] += g_phi * (rhou / r2a);
    gmu[2] += g_theta * (-x / rho2u) + g_phi * (-y * z / (r2a * rhou));
  }
  // projected-mean path: J^T g_mean2d
  for (int q = 0; q < 3; ++q) gmu[q] += J[0][q] * gm0 + J[1][q] * gm1;
  // g_pos = g_mu W + distance path
  double gp[3];
  for (int c = 0; c < 3; ++c) gp[c] = gmu[0] * W[c] + gmu[1] * W[3 + c] + gmu[2] * W[6 + c];
  gp[0] += gpd0;
  gp[1] += gpd1;
  gp[2] += gpd2;
  // opacity logit
  const double logit = A.cloud.raw_opacities[i];
  double sig;
  if (logit >= 0.0) {
    sig = 1.0 / (1.0 + exp(-logit));
  } else {
    const double e = exp(logit);
    sig = e / (1.0 + e);
  }
  for (int c = 0; c < 3; ++c) {
    put(g_pos, 3 * i + c, gp[c]);
    put(g_ls, 3 * i + c, gls[c]);
  }
  for (int c = 0; c < 4; ++c) put(g_rot, 4 * i + c, gq[c]);
  put(g_op, i, gsig * sig * (1.0 - sig));
}

int launch_gauss_backward(const gsparc_cloud& cloud, const gsparc_view& view, const double* tx,
                          int B, const gsparc_frame_layout& L, char* frame, void* grad,
                          int grad_dtype, cudaStream_t st) {
  GBwdArgs A;
  A.cloud = cloud;
  for (int k = 0; k < 3; ++k) A.pose.rx[k] = view.rx[k];
  for (int k = 0; k < 9; ++k) A.pose.W[k] = view.rotation[k];
  A.gc = make_geo_const(L.width, L.height);
  A.tx = tx;
  A.B = B;
  A.key = (const uint64_t*)(frame + L.off_key);
  A.rec32 = (const float4*)(frame + L.off_rec32);
  A.rec64 = (const double*)(frame + L.off_rec64);
  A.gcoef = frame + L.off_gcoef;
  A.ggeo = frame + L.off_ggeo;
  A.live = L.dtype == GSPARC_F32 ? (const int*)(frame + L.off_live) : nullptr;
  A.grad = grad;
  A.Cp = L.channels;
  A.P = cloud.mlp_in * cloud.mlp_hidden + cloud.mlp_hidden + cloud.mlp_hidden * cloud.mlp_out +
        cloud.mlp_out;
  if (cloud.mlp_hidden > 32 || cloud.mlp_in > 8) {
    set_error("gaussian backward: hidden<=32, inputs<=8 supported");
    return GSPARC_ERR_UNSUPPORTED;
  }
  if (cloud.n == 0) return GSPARC_OK;
  const int threads = 128;
  A.lane_tx = cloud.mlp_in == 5 && cloud.mlp_hidden == 16 && cloud.mlp_out <= 16 &&
              A.P <= 32 * LANE_TX_JMAX;
  const size_t per_warp =
      A.lane_tx ? (size_t)32 * (2 * 17 + 6 + cloud.mlp_out + 1)
                : (size_t)(8 + 96 + cloud.mlp_out + A.P);
  // the lane-per-TX path stages f32 rows for f32 frames and gradients
  const size_t elem = (A.lane_tx && L.dtype == GSPARC_F32 && grad_dtype == GSPARC_F32)
                          ? sizeof(float) : sizeof(double);
  const size_t smem = elem * (threads / 32) * per_warp;
  if (smem > 227 * 1024) {
    set_error("gaussian backward: %d MLP parameters exceed shared memory", A.P);
    return GSPARC_ERR_UNSUPPORTED;
  }
  static size_t attr[4] = {0, 0, 0, 0};
  auto opt_in = [&](auto kern, int slot) {
    if (attr[slot] < smem) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr[slot] = smem;
    }
  };
  opt_in(k_gauss_bwd<double, double>, 0);
  opt_in(k_gauss_bwd<double, float>, 1);
  opt_in(k_gauss_bwd<float, double>, 2);
  opt_in(k_gauss_bwd<float, float>, 3);
  const unsigned blocks = (unsigned)((cloud.n * 32 + threads - 1) / threads);
  const unsigned gblocks = (unsigned)((cloud.n + 127) / 128);
  if (L.dtype == GSPARC_F64) {
    if (grad_dtype == GSPARC_F64) {
      k_gauss_bwd<double, double><<<blocks, threads, smem, st>>>(A);
      k_gauss_geo<double, double><<<gblocks, 128, 0, st>>>(A);
    } else {
      k_gauss_bwd<double, float><<<blocks, threads, smem, st>>>(A);
      k_gauss_geo<double, float><<<gblocks, 128, 0, st>>>(A);
    }
  } else {
    if (grad_dtype == GSPARC_F64) {
      k_gauss_bwd<float, double><<<blocks, threads, smem, st>>>(A);
      k_gauss_geo<float, double><<<gblocks, 128, 0, st>>>(A);
    } else {
      k_gauss_bwd<float, float><<<blocks, threads, smem, st>>>(A);
      k_gauss_geo<float, float><<<gblocks, 128, 0, st>>>(A);
    }
  }
  return check_launch("k_gauss_bwd");
}

}  // namespace gs
