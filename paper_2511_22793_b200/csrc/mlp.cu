// K1: per-Gaussian emitter MLP with 1/d attenuation, batched over TX.
// Replaces mlp.direction_angles (mlp.py:83-89), mlp.batch_mlp_forward
// (mlp.py:40-45), the near-plane distance clamp (rasterizer.py:103-105) and
// coef = s / d_tx (rasterizer.py:200).  theta/phi are TX-independent and were
// produced by K2 (rec32/rec64).  Output coef[i, b*C + c] (frame dtype).
//
// Two mappings:
//   narrow: one thread per (Gaussian, TX); for small heads (C <= 8) where the
//           130-float weight row is L1-resident across the TX threads.
//   wide:   one warp per Gaussian; W2 (C x 16) streamed with coalesced float4
//           loads (lane l reads float4 #l of the row block), partial dots
//           reduced over the 4 lanes that share an output row.  This is the
//           HBM-bound path of the 52-subcarrier config (7.5 KB per Gaussian).
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"

namespace gs {

long long* dbg_rows(int which);

struct MlpArgs {
  const float* w32;
  const double* w64;
  const double* pos;
  const double* tx;  // [B,3]
  const float4* rec32;
  const double* rec64;
  const uint64_t* key;
  const int* live_list;  // live Gaussians (K4 pass A); nullptr -> all kept
  const int* counters;
  void* coef;
  int64_t n;
  int stream_ctas;  // > 0: started during pass A (PDL); entries appear as its CTAs finish
  long long* dbg;   // experiments: per-CTA start/end stamps (GSPARC_MLP_DBG)
  int B, C, H, I, P;
  int64_t Cp;  // B*C
};

__device__ __forceinline__ double tx_distance(const double* pos, const double* tx) {
  double d0 = sub(pos[0], tx[0]), d1 = sub(pos[1], tx[1]), d2 = sub(pos[2], tx[2]);
  double d = __dsqrt_rn(add(add(mul(d0, d0), mul(d1, d1)), mul(d2, d2)));
  return d < NEAR_PLANE ? NEAR_PLANE : d;  // rasterizer.py:103-105
}

// (5, 16, C) head with few outputs (C <= 8, e.g. the 2-channel RSSI model
// batched over TX): thread per (Gaussian, TX), a warp = one Gaussian's
// weights (broadcast loads) for 32 transmitters; loops unrolled, hidden layer
// in registers.
template <int C>
__global__ void __launch_bounds__(256) k_mlp_narrow516(MlpArgs A) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gi = t / A.B;
  const int b = (int)(t % A.B);
  const int64_t count = A.live_list ? A.counters[GSPARC_CNT_LIVE] : A.n;
  if (gi >= count) return;
  const int64_t i = A.live_list ? A.live_list[gi] : gi;
  if (!A.live_list && A.key[i] == ~0ULL) return;
  const float4 r = A.rec32[2 * i + 1];
  const double* txb = A.tx + 3 * b;
  const float x[5] = {(float)txb[0], (float)txb[1], (float)txb[2], r.z, r.w};
  constexpr int H = 16, I = 5;
  const float* w = A.w32 + i * (int64_t)A.P;
  float hid[H];
#pragma unroll
  for (int h = 0; h < H; ++h) {
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < I; ++k) acc += w[h * I + k] * x[k];
    acc += w[H * I + h];
    hid[h] = acc > 0.f ? acc : 0.f;
  }
  const float* w2 = w + H * I + H;
  const float* b2 = w2 + C * H;
  const double d = tx_distance(A.pos + 3 * i, txb);
  float* out = (float*)A.coef + i * A.Cp + (int64_t)b * C;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    float acc = 0.f;
#pragma unroll
    for (int h = 0; h < H; ++h) acc += w2[c * H + h] * hid[h];
    acc += b2[c];
    out[c] = (float)((double)acc / d);
  }
}

template <typename R>
__global__ void __launch_bounds__(256) k_mlp_narrow(MlpArgs A) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gi = t / A.B;
  const int b = (int)(t % A.B);
  const int64_t count = A.live_list ? A.counters[GSPARC_CNT_LIVE] : A.n;
  if (gi >= count) return;
  const int64_t i = A.live_list ? A.live_list[gi] : gi;
  if (!A.live_list && A.key[i] == ~0ULL) return;
  R theta, phi;
  if constexpr (sizeof(R) == 4) {
    float4 r = A.rec32[2 * i + 1];
    theta = r.z;
    phi = r.w;
  } else {
    theta = A.rec64[8 * i + 6];
    phi = A.rec64[8 * i + 7];
  }
  const double* txb = A.tx + 3 * b;
  R x[5] = {(R)txb[0], (R)txb[1], (R)txb[2], theta, phi};
  const int H = A.H, I = A.I, C = A.C;
  float hid32[32];
  double hid64[32];
  if constexpr (sizeof(R) == 4) {
    const float* w = A.w32 + i * (int64_t)A.P;
    for (int h = 0; h < H; ++h) {
      float acc = 0.f;
      for (int k = 0; k < I; ++k) acc += w[h * I + k] * x[k];
      acc += w[H * I + h];
      hid32[h] = acc > 0.f ? acc : 0.f;
    }
    const float* w2 = w + H * I + H;
    const float* b2 = w2 + C * H;
    double d = tx_distance(A.pos + 3 * i, txb);
    const int64_t o0 = i * A.Cp + (int64_t)b * C;
    float* out = (float*)A.coef + o0;
    for (int c = 0; c < C; ++c) {
      float acc = 0.f;
      for (int h = 0; h < H; ++h) acc += w2[c * H + h] * hid32[h];
      acc += b2[c];
      out[c] = (float)((double)acc / d);
    }
  } else {
    const double* w = A.w64 + i * (int64_t)A.P;
    for (int h = 0; h < H; ++h) {
      double acc = 0.0;
      for (int k = 0; k < I; ++k) acc += w[h * I + k] * x[k];
      acc += w[H * I + h];
      hid64[h] = acc > 0.0 ? acc : 0.0;
    }
    const double* w2 = w + H * I + H;
    const double* b2 = w2 + C * H;
    double d = tx_distance(A.pos + 3 * i, txb);
    double* out = (double*)A.coef + i * A.Cp + (int64_t)b * C;
    for (int c = 0; c < C; ++c) {
      double acc = 0.0;
      for (int h = 0; h < H; ++h) acc += w2[c * H + h] * hid64[h];
      acc += b2[c];
      out[c] = acc / d;
    }
  }
}

// Wide head, f32 weights, H == 16, I == 5, C % 4 == 0.
// Every load of the Gaussian (its W1/b1 row, W2 and b2, theta/phi) is issued
// before any arithmetic, so one warp has up to 8 KB in flight and pays one
// memory latency per 128 output channels (C > 128 streams W2 in parts).
__device__ __forceinline__ void mlp_wide_one(const MlpArgs& A, int64_t i, int lane) {
  constexpr int MAXV = 16;  // float4 per lane per part: 128 channels
  const float* w = A.w32 + i * (int64_t)A.P;
  const int C = A.C;
  const int nvec = 4 * C;
  const int hu = lane & 15;
  const float4 r1 = __ldg(A.rec32 + 2 * i + 1);
  float w1[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) w1[k] = __ldg(w + hu * 5 + k);
  const float b1 = __ldg(w + 80 + hu);
  const float4* w2v = reinterpret_cast<const float4*>(w + 96);
  const float* b2 = w + 96 + 16 * C;
  const int q = lane & 3;
  const double* pp = A.pos + 3 * i;
  const double pv[3] = {__ldg(pp), __ldg(pp + 1), __ldg(pp + 2)};  // issued with the weights
  for (int part = 0; part * MAXV * 32 < nvec; ++part) {
    float4 v[MAXV];
    float bv[MAXV];
#pragma unroll
    for (int u = 0; u < MAXV; ++u) {
      const int f = (part * MAXV + u) * 32 + lane;
      v[u] = f < nvec ? __ldg(w2v + f) : make_float4(0.f, 0.f, 0.f, 0.f);
      bv[u] = (f < nvec && (lane & 3) == 0) ? __ldg(b2 + (f >> 2)) : 0.f;
    }
    for (int b = 0; b < A.B; ++b) {
      const double* txb = A.tx + 3 * b;
      float x[5] = {(float)txb[0], (float)txb[1], (float)txb[2], r1.z, r1.w};
      float pre = 0.f;
#pragma unroll
      for (int k = 0; k < 5; ++k) pre += w1[k] * x[k];
      pre += b1;
      const float hid = pre > 0.f ? pre : 0.f;
      const float h0 = __shfl_sync(0xffffffffu, hid, 4 * q + 0);
      const float h1 = __shfl_sync(0xffffffffu, hid, 4 * q + 1);
      const float h2 = __shfl_sync(0xffffffffu, hid, 4 * q + 2);
      const float h3 = __shfl_sync(0xffffffffu, hid, 4 * q + 3);
      // s / d_tx (rasterizer.py:200): one f64 reciprocal per (Gaussian, TX);
      // x * (1/d) differs from x / d by <= 1 ulp in f64, invisible after the
      // cast to f32 except on exact rounding ties
      const double rd = 1.0 / tx_distance(pv, txb);
      float* out = (float*)A.coef + i * A.Cp + (int64_t)b * C;
#pragma unroll
      for (int u = 0; u < MAXV; ++u) {
        const int f = (part * MAXV + u) * 32 + lane;
        if ((part * MAXV + u) * 32 >= nvec) break;
        float acc = v[u].x * h0 + v[u].y * h1 + v[u].z * h2 + v[u].w * h3;
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        if (q == 0 && f < nvec) out[f >> 2] = (float)((double)(acc + bv[u]) * rd);
      }
    }
  }
}

__global__ void __launch_bounds__(256, 2) k_mlp_wide(MlpArgs A) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (A.dbg && threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 14] = gtimer();
  // pass B with several channel chunks (> 256 columns, config 5: thousands
  // of CTAs) is scheduled from the MLP's start -- its first CTAs' prologues
  // then overlap the whole MLP (measured 2% faster there); with one chunk
  // only once pass A has finished (below)
  if (A.stream_ctas && A.Cp > 256) pdl_trigger();
  if (A.live_list && A.stream_ctas) {
    // streaming: the list is -1 where pass A has not written yet (K2 clears
    // it); a warp takes entries wid, wid + nwarps, ... as they appear, and
    // stops at the first empty entry once every pass-A CTA has finished
    for (int64_t gi = wid; gi < A.n; gi += nwarps) {
      int v = __ldcv(A.live_list + gi);
      long long spins = 0;
      while (v < 0) {
        if (flag_acquire(A.counters + GSPARC_CNT_PXA_DONE) >= A.stream_ctas ||
            __ldcv(A.counters + GSPARC_CNT_OVERFLOW)) {
          v = __ldcv(A.live_list + gi);
          break;
        }
        __nanosleep(256);
        if (++spins > (1ll << 22)) break;  // bounded (pass A never ran): leave
        v = __ldcv(A.live_list + gi);
      }
      if (v < 0) break;
      mlp_wide_one(A, v, lane);
      if (A.dbg && lane == 0) atomicMax(A.dbg + blockIdx.x * 16 + 13, (long long)gtimer());
    }
    // this warp found the end of the live list (pass A has finished): pass B
    // may now be scheduled and run its prologue beside the MLP's last
    // Gaussians (it waits for this grid).  Not earlier -- its CTAs would sit
    // on SMs pass A still needs -- and not in the other modes, where a pass A
    // launched next would read coef early.
    pdl_trigger();
    if (A.dbg) {
      __syncthreads();
      if (threadIdx.x == 0) A.dbg[blockIdx.x * 16 + 15] = gtimer();
    }
    pdl_wait();  // complete only after pass A has
    return;
  }
  if (A.live_list) {  // one warp per live Gaussian, all in flight
    // the list entry is read speculatively together with the count (the
    // list has room for n entries), saving one dependent round trip
    const int first = wid < A.n ? __ldcg(A.live_list + wid) : 0;
    const int64_t count = __ldcg(A.counters + GSPARC_CNT_LIVE);
    for (int64_t gi = wid; gi < count; gi += nwarps)
      mlp_wide_one(A, gi == wid ? first : __ldcg(A.live_list + gi), lane);
    return;
  }
  for (int64_t gi = wid; gi < A.n; gi += nwarps) {
    if (A.key[gi] == ~0ULL) continue;
    mlp_wide_one(A, gi, lane);
  }
}

int launch_mlp(const gsparc_cloud& cloud, const double* tx, int B, bool live_only,
               const gsparc_frame_layout& L, char* frame, cudaStream_t st, int stream_ctas) {
  MlpArgs A;
  A.stream_ctas = 0;
  A.dbg = experiment_env("GSPARC_MLP_DBG") ? dbg_rows(3) + 16 * 2048 : nullptr;  // experiments only
  A.w32 = cloud.mlp_weights;
  A.w64 = cloud.mlp_weights64;
  A.pos = cloud.positions;
  A.tx = tx;
  A.rec32 = (const float4*)(frame + L.off_rec32);
  A.rec64 = (const double*)(frame + L.off_rec64);
  A.key = (const uint64_t*)(frame + L.off_key);
  A.live_list = live_only ? (const int*)(frame + L.off_live_list) : nullptr;
  A.counters = (const int*)(frame + L.off_counters);
  A.coef = frame + L.off_coef;
  A.n = cloud.n;
  A.B = B;
  A.C = cloud.mlp_out;
  A.H = cloud.mlp_hidden;
  A.I = cloud.mlp_in;
  A.P = cloud.mlp_in * cloud.mlp_hidden + cloud.mlp_hidden + cloud.mlp_hidden * cloud.mlp_out +
        cloud.mlp_out;
  A.Cp = (int64_t)B * cloud.mlp_out;
  if (A.Cp > L.channels) {
    set_error("mlp: n_tx*mlp_out=%lld exceeds frame channels %lld", (long long)A.Cp,
              (long long)L.channels);
    return GSPARC_ERR_ARG;
  }
  if (A.H > 32 || A.I > 5) {
    set_error("mlp: hidden<=32 and inputs==5 supported (got %d, %d)", A.H, A.I);
    return GSPARC_ERR_UNSUPPORTED;
  }
  if (cloud.n == 0) return GSPARC_OK;
  if (L.dtype == GSPARC_F64) {
    if (!A.w64) {
      set_error("mlp: f64 frame needs cloud.mlp_weights64");
      return GSPARC_ERR_ARG;
    }
    int64_t threads = cloud.n * B;
    k_mlp_narrow<double><<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(A);
  } else if (A.C % 4 == 0 && A.C >= 16 && A.H == 16 && A.I == 5) {
    int64_t threads = cloud.n * 32;
    int64_t blocks = (threads + 255) / 256;
    // live list: one wave (2 CTAs per SM), grid-stride over the list; most
    // renders have fewer live Gaussians than resident warps
    if (live_only && blocks > 148 * 2) blocks = 148 * 2;
    static const int stream_blocks =
        experiment_env("GSPARC_MLP_SBLOCKS") ? atoi(experiment_env("GSPARC_MLP_SBLOCKS")) : 148;
    if (live_only && stream_ctas > 0 && !getenv("GSPARC_NO_PDL")) {
      // one CTA per SM: all resident next to pass A's two CTAs, so no entry
      // waits for a CTA that can only start when pass A leaves
      if (stream_blocks > 0 && blocks > stream_blocks) blocks = stream_blocks;
      // programmatic dependent launch behind pass A (which triggers at its
      // start): the MLP runs while pass A's last CTAs finish
      A.stream_ctas = stream_ctas;
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      cfg.gridDim = dim3((unsigned)blocks);
      cfg.blockDim = dim3(256);
      cfg.stream = st;
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, k_mlp_wide, A);
    } else {
      k_mlp_wide<<<(unsigned)blocks, 256, 0, st>>>(A);
    }
  } else {
    int64_t threads = cloud.n * B;
    const unsigned blocks = (unsigned)((threads + 255) / 256);
    if (A.H == 16 && A.I == 5 && A.C == 2) {
      k_mlp_narrow516<2><<<blocks, 256, 0, st>>>(A);
    } else if (A.H == 16 && A.I == 5 && A.C == 4) {
      k_mlp_narrow516<4><<<blocks, 256, 0, st>>>(A);
    } else if (A.H == 16 && A.I == 5 && A.C == 8) {
      k_mlp_narrow516<8><<<blocks, 256, 0, st>>>(A);
    } else {
      k_mlp_narrow<float><<<blocks, 256, 0, st>>>(A);
    }
  }
  return check_launch("k_mlp");
}

}  // namespace gs
