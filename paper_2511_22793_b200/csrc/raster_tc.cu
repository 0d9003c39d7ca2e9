// K4 (lazy path): weights pass + tensor-core accumulation pass.
// Replaces do_tile / _tile_alphas (rasterizer.py:169-231) for wide channel
// counts (C' = n_tx * C > 4, e.g. 52 OFDM subcarriers).
//
// Both passes walk a half tile (16 x 8 = 128 pixels) and consume the tile's
// depth-sorted list in 32-entry chunks with the same arithmetic:
//   lanes = entries: alpha via pixel_alpha(), T_before = T_in * exclusive
//   warp prefix product of (1 - alpha), stop at the first entry with
//   T_before < t_eps, include iff alpha > 0, wgt = T_before * alpha
//   (rasterizer.py:209-219).
// Pass A (k_raster_a) keeps only count / last / T_final, the per-strip
// visited prefix and the live-Gaussian list (the MLP then runs on live
// Gaussians only).  Pass B (k_raster_b) turns every chunk into one K=32 slice
// of a GEMM
//     img[128 px, C'] += W[128 px, 32 entries] . coef[32 entries, C']
// executed by tcgen05.mma (kind::tf32, accumulator in TMEM).  fp32 accuracy
// comes from the 3xTF32 split  W.c ~ Wh.ch + Wh.cl + Wl.ch  (hi = f32 with
// the 13 low mantissa bits cleared, lo = x - hi).  W and coef^T are written
// by the CUDA cores straight into the K-major SWIZZLE_128B layout; chunks are
// double buffered so the weights of chunk i+1 overlap the MMAs of chunk i.
#include "common.cuh"
#include "kernels.cuh"

namespace gs {

struct TcArgs {
  const int* tile_start;
  int* wstop;               // [ntiles * 8] visited prefix per 2-row strip
  const float4* pair_rec;   // list-ordered f32 records (K3)
  const float* coef;        // [n, Cp]
  const int* live;
  int* live_list;
  int* counters;
  float* img;               // [B, h, w, C]
  float* T_out;
  int* count_out;
  int* last_out;
  int64_t Cp;
  int C, w, h, ntx, ntiles;
  float t_eps;
};

constexpr int TC_P = 128;      // pixels per CTA (MMA M)
constexpr int TC_WARPS = 16;
constexpr int TC_K = 32;       // entries per chunk (MMA K slice)

// one 32-entry chunk for one pixel, lanes = entries.  Returns the lane's
// weight; updates the pixel state (uniform across lanes).
struct PixState {
  float T;
  int cnt, last;
  bool done;
};

__device__ __forceinline__ float chunk_weight(const float4* s_rec, int nvalid, int lane, float pcx,
                                              float pcy, float wR, float half_w, float teps,
                                              int list_pos0, PixState& st, bool& inc_out) {
  // a finished pixel sees no valid entries (branch free, so two pixels'
  // chains interleave); its state is left untouched
  const bool live_px = !st.done;
  const bool valid = lane < nvalid && live_px;
  float a = 0.f;
  if (valid) {
    const float4 r0 = s_rec[2 * lane], r1 = s_rec[2 * lane + 1];
    a = pixel_alpha<float>(pcx, pcy, r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, wR, half_w).alpha;
  }
  float P = sub(1.f, a);
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const float t = __shfl_up_sync(0xffffffffu, P, d);
    if (lane >= d) P = mul(t, P);
  }
  float Pex = __shfl_up_sync(0xffffffffu, P, 1);
  if (lane == 0) Pex = 1.f;
  const float Tb = mul(st.T, Pex);
  const unsigned stopm = __ballot_sync(0xffffffffu, valid && Tb < teps);
  const int first = stopm ? __ffs(stopm) - 1 : 32;
  const bool inc = valid && lane < first && a > 0.f;
  const unsigned incm = __ballot_sync(0xffffffffu, inc);
  if (incm) {
    st.cnt += __popc(incm);
    st.last = list_pos0 + (31 - __clz(incm)) + 1;
  }
  const float Tfirst = __shfl_sync(0xffffffffu, Tb, first & 31);
  const float Tall = __shfl_sync(0xffffffffu, mul(st.T, P), 31);
  if (live_px) {
    st.T = first < 32 ? Tfirst : Tall;
    st.done = first < 32;
  }
  inc_out = inc;
  return inc ? mul(Tb, a) : 0.f;
}

// Same chunk, four pixels per warp: the 8 lanes of group g = lane >> 3 own
// one pixel, lane j = lane & 7 owns entries 4j .. 4j+3 (sequential product
// inside the lane, 8-lane scan across lanes).  About half the instructions
// per (pixel, entry) of the one-pixel-per-warp form.
// Records of a chunk in shared memory as structure-of-arrays: field f of
// entry e at soa[f * stride + e]; lane j reads its four entries of a field
// with one conflict-free 16-byte load.
__device__ __forceinline__ void chunk_weight4(const float* soa, int stride, int nvalid, int lane,
                                              float pcx, float pcy, float wR, float half_w,
                                              float teps, int list_pos0, PixState& st,
                                              float (&w)[4], unsigned& incbits) {
  const int j = lane & 7;
  const bool live_px = !st.done;
  float a[4], om[4];
  bool v[4];
  const float4 fmx = *(const float4*)(soa + 0 * stride + 4 * j);
  const float4 fmy = *(const float4*)(soa + 1 * stride + 4 * j);
  const float4 fca = *(const float4*)(soa + 2 * stride + 4 * j);
  const float4 fcb = *(const float4*)(soa + 3 * stride + 4 * j);
  const float4 fcc = *(const float4*)(soa + 4 * stride + 4 * j);
  const float4 fop = *(const float4*)(soa + 5 * stride + 4 * j);
  const float mx[4] = {fmx.x, fmx.y, fmx.z, fmx.w}, my[4] = {fmy.x, fmy.y, fmy.z, fmy.w};
  const float ca[4] = {fca.x, fca.y, fca.z, fca.w}, cb[4] = {fcb.x, fcb.y, fcb.z, fcb.w};
  const float cc[4] = {fcc.x, fcc.y, fcc.z, fcc.w}, op[4] = {fop.x, fop.y, fop.z, fop.w};
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int e = 4 * j + u;
    v[u] = live_px && e < nvalid;
    a[u] = 0.f;
    if (v[u]) {
      a[u] = pixel_alpha<float>(pcx, pcy, mx[u], my[u], ca[u], cb[u], cc[u], op[u], wR, half_w)
                 .alpha;
    }
    om[u] = sub(1.f, a[u]);
  }
  const float L = mul(mul(mul(om[0], om[1]), om[2]), om[3]);
  float P = L;
#pragma unroll
  for (int d = 1; d < 8; d <<= 1) {
    const float t = __shfl_up_sync(0xffffffffu, P, d, 8);
    if (j >= d) P = mul(t, P);
  }
  float Pex = __shfl_up_sync(0xffffffffu, P, 1, 8);
  if (j == 0) Pex = 1.f;
  float Tb[4];
  Tb[0] = mul(st.T, Pex);
  Tb[1] = mul(Tb[0], om[0]);
  Tb[2] = mul(Tb[1], om[1]);
  Tb[3] = mul(Tb[2], om[2]);
  int first = 32;
#pragma unroll
  for (int u = 3; u >= 0; --u)
    if (v[u] && Tb[u] < teps) first = 4 * j + u;
#pragma unroll
  for (int d = 1; d < 8; d <<= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, d, 8));
  int c = 0, m = -1;
  unsigned bits = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const bool inc = v[u] && (4 * j + u) < first && a[u] > 0.f;
    w[u] = inc ? mul(Tb[u], a[u]) : 0.f;
    c += inc;
    m = inc ? 4 * j + u : m;
    bits |= (unsigned)inc << u;
  }
#pragma unroll
  for (int d = 1; d < 8; d <<= 1) {
    c += __shfl_xor_sync(0xffffffffu, c, d, 8);
    m = max(m, __shfl_xor_sync(0xffffffffu, m, d, 8));
  }
  if (c) {
    st.cnt += c;
    st.last = list_pos0 + m + 1;
  }
  // transmittance handed to the next chunk
  const int fu = first & 3;
  const float Tsel = fu == 0 ? Tb[0] : fu == 1 ? Tb[1] : fu == 2 ? Tb[2] : Tb[3];
  const float Tfirst = __shfl_sync(0xffffffffu, Tsel, (first >> 2) & 7, 8);
  const float Tall = __shfl_sync(0xffffffffu, mul(st.T, P), 7, 8);
  if (live_px) {
    st.T = first < 32 ? Tfirst : Tall;
    st.done = first < 32;
  }
  incbits = bits;
}

__device__ __forceinline__ void pixel_xy(int tile, int half, int p, int ntx, int& px, int& py) {
  const int tx_ = tile % ntx, ty = tile / ntx;
  px = tx_ * TILE + (p & 15);
  py = ty * TILE + half * 8 + (p >> 4);
}

// ------------------------------------------------------------- pass A
// 128 entries staged per barrier; 16 warps x 8 pixels each.
__global__ void __launch_bounds__(512) k_raster_a(TcArgs A) {
  constexpr int SUP = 4 * TC_K;
  __shared__ __align__(16) float s_soa[6 * SUP];
  __shared__ int s_sidx[SUP];
  __shared__ int s_live[SUP];
  __shared__ float s_T[TC_P];
  __shared__ int s_cnt[TC_P], s_last[TC_P], s_done[TC_P];
  __shared__ int s_stop[4];
  if (A.counters[GSPARC_CNT_OVERFLOW]) return;
  const int tile = blockIdx.x >> 1, half = blockIdx.x & 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int start = A.tile_start[tile], end = A.tile_start[tile + 1];
  const float wR = (float)A.w, half_w = (float)(A.w / 2.0), teps = A.t_eps;
  if (tid < TC_P) {
    int px, py;
    pixel_xy(tile, half, tid, A.ntx, px, py);
    s_T[tid] = 1.f;
    s_cnt[tid] = 0;
    s_last[tid] = 0;
    s_done[tid] = !(px < A.w && py < A.h);
  }
  if (tid < 4) s_stop[tid] = 0;
  for (int cb = start; cb < end; cb += SUP) {
    const int nsup = min(SUP, end - cb);
    __syncthreads();
    if (tid < SUP) {
      float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
      if (tid < nsup) {
        r0 = __ldg(A.pair_rec + 2 * (size_t)(cb + tid));
        r1 = __ldg(A.pair_rec + 2 * (size_t)(cb + tid) + 1);
      }
      s_soa[0 * SUP + tid] = r0.x;
      s_soa[1 * SUP + tid] = r0.y;
      s_soa[2 * SUP + tid] = r0.z;
      s_soa[3 * SUP + tid] = r0.w;
      s_soa[4 * SUP + tid] = r1.x;
      s_soa[5 * SUP + tid] = r1.y;
      s_sidx[tid] = __float_as_int(r1.z);
      s_live[tid] = 0;
    }
    __syncthreads();
    {
      // lane group g = lane >> 3 owns pixel warp + 16 g (set 0) and
      // warp + 16 (g + 4) (set 1); both sets advance together (ILP)
      const int g = lane >> 3;
      const int p0 = warp + TC_WARPS * g, p1 = warp + TC_WARPS * (g + 4);
      int px0, py0, px1, py1;
      pixel_xy(tile, half, p0, A.ntx, px0, py0);
      pixel_xy(tile, half, p1, A.ntx, px1, py1);
      PixState st0{s_T[p0], s_cnt[p0], s_last[p0], s_done[p0] != 0};
      PixState st1{s_T[p1], s_cnt[p1], s_last[p1], s_done[p1] != 0};
      for (int k0 = 0; k0 < nsup; k0 += TC_K) {
        if (__all_sync(0xffffffffu, st0.done && st1.done)) break;
        const int nv = min(TC_K, nsup - k0);
        float w0[4], w1[4];
        unsigned b0, b1;
        chunk_weight4(s_soa + k0, SUP, nv, lane, (float)px0 + 0.5f, (float)py0 + 0.5f, wR,
                      half_w, teps, cb - start + k0, st0, w0, b0);
        chunk_weight4(s_soa + k0, SUP, nv, lane, (float)px1 + 0.5f, (float)py1 + 0.5f, wR,
                      half_w, teps, cb - start + k0, st1, w1, b1);
        const unsigned b = b0 | b1;
        if (b) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if ((b >> u) & 1u) s_live[k0 + 4 * (lane & 7) + u] = 1;
        }
      }
      if ((lane & 7) == 0) {
        s_T[p0] = st0.T;
        s_cnt[p0] = st0.cnt;
        s_last[p0] = st0.last;
        s_done[p0] = st0.done;
        s_T[p1] = st1.T;
        s_cnt[p1] = st1.cnt;
        s_last[p1] = st1.last;
        s_done[p1] = st1.done;
      }
    }
    __syncthreads();
    if (tid < nsup && s_live[tid]) {
      const int idx = s_sidx[tid];
      if (A.live[idx] == 0 && atomicExch((int*)A.live + idx, 1) == 0) {
        const int pos = atomicAdd(A.counters + GSPARC_CNT_LIVE, 1);
        A.live_list[pos] = idx;
      }
    }
    if (__syncthreads_count(tid < TC_P ? s_done[tid] : 1) == (int)blockDim.x) break;
  }
  __syncthreads();
  if (tid < TC_P) {
    int px, py;
    pixel_xy(tile, half, tid, A.ntx, px, py);
    if (px < A.w && py < A.h) {
      const int q = py * A.w + px;
      A.T_out[q] = s_T[tid];
      A.count_out[q] = s_cnt[tid];
      A.last_out[q] = s_last[tid];
      atomicMax(&s_stop[tid >> 5], s_last[tid]);
    }
  }
  __syncthreads();
  if (tid < 4) A.wstop[tile * 8 + half * 4 + tid] = s_stop[tid];
}

// ------------------------------------------------------------- pass B
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// K-major SWIZZLE_128B UMMA descriptor: rows of 128 B, 8-row atoms 1024 B
// apart (SBO), LBO unused, version 1, layout type 2.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                 // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;       // SBO
  d |= (uint64_t)1 << 46;                 // version (sm100)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}

// byte offset of element (row r, k) of a [rows][32] f32 K-major SW128 tile
__device__ __forceinline__ uint32_t sw128_off(int r, int k) {
  return (uint32_t)(r * 128 + ((((k >> 2) ^ (r & 7)) << 4) | ((k & 3) << 2)));
}

__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity));
}

// NP: channel columns per CTA (multiple of 8, <= 256); the channel axis is
// split over blockIdx.y.  Single operand stage: the weights of chunk c and
// the coef values of chunk c are computed / loaded into registers while the
// MMAs of chunk c-1 run, then stored once those MMAs have retired, so a CTA
// needs ~60 KB of shared memory and three CTAs share an SM.
template <int NP>
__global__ void __launch_bounds__(512, 2) k_raster_b(TcArgs A) {
  constexpr int A_BYTES = TC_P * 128;  // 16 KB per operand copy
  constexpr int B_BYTES = NP * 128;
  constexpr uint32_t TMEM_COLS = NP <= 32 ? 32 : NP <= 64 ? 64 : NP <= 128 ? 128 : 256;
  constexpr int NQ = (NP * TC_K + 511) / 512;  // coef values per thread
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  unsigned char* Ahi = sm;
  unsigned char* Alo = sm + A_BYTES;
  unsigned char* Bhi = sm + 2 * A_BYTES;
  unsigned char* Blo = sm + 2 * A_BYTES + B_BYTES;
  __shared__ __align__(16) float s_soa[6 * TC_K];
  __shared__ int s_cidx[3][TC_K];
  __shared__ float s_T[TC_P];
  __shared__ int s_done[TC_P];
  __shared__ __align__(8) uint64_t s_bar;
  __shared__ uint32_t s_tmem;

  if (A.counters[GSPARC_CNT_OVERFLOW]) return;
  const int tile = blockIdx.x >> 1, half = blockIdx.x & 1;
  const int col0 = blockIdx.y * NP;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int start = A.tile_start[tile];
  int vis = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) vis = max(vis, A.wstop[tile * 8 + half * 4 + q]);
  const int end = start + vis;
  const int nch_total = (vis + TC_K - 1) / TC_K;
  const float wR = (float)A.w, half_w = (float)(A.w / 2.0), teps = A.t_eps;

  if (tid < TC_P) {
    int px, py;
    pixel_xy(tile, half, tid, A.ntx, px, py);
    s_T[tid] = 1.f;
    s_done[tid] = !(px < A.w && py < A.h);
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::);
  }
  // list indices of chunk c (threads < 32).  No live mask is needed: coef
  // rows of Gaussians that are not live were either zero-initialised with
  // the frame or written by an earlier render, so they are finite and meet a
  // weight of exactly zero.
  auto idx_of = [&](int c) -> int {
    int v = -1;
    if (tid < TC_K) {
      const int jj = start + c * TC_K + tid;
      if (c < nch_total && jj < end) v = __float_as_int(__ldg(&A.pair_rec[2 * (size_t)jj + 1].z));
    }
    return v;
  };
  float pre[NQ];
  float4 prec0 = make_float4(0.f, 0.f, 0.f, 0.f), prec1 = prec0;
  auto prefetch = [&](int c) {  // coef values + records of chunk c -> registers
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      const int q = tid + 512 * u;
      float v = 0.f;
      if (q < NP * TC_K && c < nch_total) {
        const int k = q / NP, n = q - k * NP;
        const int idx = s_cidx[c % 3][k];
        const int64_t cc = col0 + n;
        if (idx >= 0 && cc < A.Cp) v = __ldg(A.coef + (int64_t)idx * A.Cp + cc);
      }
      pre[u] = v;
    }
    if (tid < TC_K && c < nch_total) {
      const int jj = start + c * TC_K + tid;
      const bool ok = jj < end;
      prec0 = ok ? __ldg(A.pair_rec + 2 * (size_t)jj) : make_float4(0.f, 0.f, 0.f, 0.f);
      prec1 = ok ? __ldg(A.pair_rec + 2 * (size_t)jj + 1) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  if (tid < TC_K) {
    s_cidx[0][tid] = idx_of(0);
    s_cidx[1][tid] = idx_of(1);
  }
  int ridx = idx_of(2);  // register-carried: stored one iteration later
  asm volatile("tcgen05.fence::before_thread_sync;" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::);
  const uint32_t tmem = s_tmem;
  // instruction descriptor: D f32, A/B tf32, K-major both, N = NP, M = 128
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NP >> 3) << 17) |
                         ((uint32_t)(TC_P >> 4) << 24);
  prefetch(0);

  const int g = lane >> 3, j = lane & 7;
  const int p0 = warp + TC_WARPS * g, p1 = warp + TC_WARPS * (g + 4);
  int px0, py0, px1, py1;
  pixel_xy(tile, half, p0, A.ntx, px0, py0);
  pixel_xy(tile, half, p1, A.ntx, px1, py1);
  PixState st0{1.f, 0, 0, s_done[p0] != 0};
  PixState st1{1.f, 0, 0, s_done[p1] != 0};

  int nchunks = 0;
  for (int c = 0; c < nch_total; ++c) {
    const int nk = min(TC_K, end - (start + c * TC_K));
    // records of chunk c (the previous chunk's readers passed barrier 2)
    if (tid < TC_K) {
      s_cidx[(c + 2) % 3][tid] = ridx;
      s_soa[0 * TC_K + tid] = prec0.x;
      s_soa[1 * TC_K + tid] = prec0.y;
      s_soa[2 * TC_K + tid] = prec0.z;
      s_soa[3 * TC_K + tid] = prec0.w;
      s_soa[4 * TC_K + tid] = prec1.x;
      s_soa[5 * TC_K + tid] = prec1.y;
    }
    __syncthreads();
    // weights of chunk c in registers
    float w0[4], w1[4];
    unsigned b0, b1;
    chunk_weight4(s_soa, TC_K, nk, lane, (float)px0 + 0.5f, (float)py0 + 0.5f, wR, half_w, teps,
                  0, st0, w0, b0);
    chunk_weight4(s_soa, TC_K, nk, lane, (float)px1 + 0.5f, (float)py1 + 0.5f, wR, half_w, teps,
                  0, st1, w1, b1);
    const bool all_done = (j == 0) && st0.done && st1.done;
    // operands of chunk c-1 are free once its MMAs retired
    if (c >= 1) mbar_wait(smem_u32(&s_bar), (c - 1) & 1);
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      const int q = tid + 512 * u;
      if (q < NP * TC_K) {
        const int k = q / NP, n = q - k * NP;
        const float v = pre[u];
        const float hi = tf32_hi(v);
        const uint32_t off = sw128_off(n, k);
        *(float*)(Bhi + off) = hi;
        *(float*)(Blo + off) = v - hi;
      }
    }
    {
      float4 h = make_float4(tf32_hi(w0[0]), tf32_hi(w0[1]), tf32_hi(w0[2]), tf32_hi(w0[3]));
      float4 l = make_float4(w0[0] - h.x, w0[1] - h.y, w0[2] - h.z, w0[3] - h.w);
      const uint32_t o0 = (uint32_t)(p0 * 128 + ((j ^ (p0 & 7)) << 4));
      *(float4*)(Ahi + o0) = h;
      *(float4*)(Alo + o0) = l;
      h = make_float4(tf32_hi(w1[0]), tf32_hi(w1[1]), tf32_hi(w1[2]), tf32_hi(w1[3]));
      l = make_float4(w1[0] - h.x, w1[1] - h.y, w1[2] - h.z, w1[3] - h.w);
      const uint32_t o1 = (uint32_t)(p1 * 128 + ((j ^ (p1 & 7)) << 4));
      *(float4*)(Ahi + o1) = h;
      *(float4*)(Alo + o1) = l;
    }
    // next chunk's loads fly while this chunk's MMAs run
    prefetch(c + 1);
    ridx = idx_of(c + 3);
    asm volatile("fence.proxy.async.shared::cta;" ::);
    const int ndone = __syncthreads_count(all_done);
    if (tid == 512 - 32) {  // the MMA issuer lives in the last warp
      asm volatile("tcgen05.fence::after_thread_sync;" ::);
      const uint32_t a_hi = smem_u32(Ahi), a_lo = smem_u32(Alo);
      const uint32_t b_hi = smem_u32(Bhi), b_lo = smem_u32(Blo);
#pragma unroll
      for (int ks = 0; ks < TC_K / 8; ++ks) {
        const uint32_t koff = ks * 32;  // 8 tf32 = 32 bytes along K
        const uint32_t acc0 = (c > 0 || ks > 0) ? 1u : 0u;
        mma_tf32(tmem, umma_desc_sw128(a_hi + koff), umma_desc_sw128(b_hi + koff), idesc, acc0);
        mma_tf32(tmem, umma_desc_sw128(a_hi + koff), umma_desc_sw128(b_lo + koff), idesc, 1u);
        mma_tf32(tmem, umma_desc_sw128(a_lo + koff), umma_desc_sw128(b_hi + koff), idesc, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::
                       "r"(smem_u32(&s_bar)));
    }
    nchunks = c + 1;
    if (ndone == TC_P / 2) break;  // 16 warps x 4 groups x 2 pixels
  }
  if (nchunks >= 1) mbar_wait(smem_u32(&s_bar), (nchunks - 1) & 1);
  asm volatile("tcgen05.fence::after_thread_sync;" ::);
  // epilogue: warps 0..3 read TMEM lanes 32w..32w+31 (= pixels)
  if (warp < 4) {
    const int p = warp * 32 + lane;
    int px, py;
    pixel_xy(tile, half, p, A.ntx, px, py);
    const bool inside = px < A.w && py < A.h;
#pragma unroll 1
    for (int c0 = 0; c0 < NP; c0 += 8) {
      uint32_t v[8];
      if (nchunks > 0) {
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
              "=r"(v[7])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::);
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = 0u;
      }
      if (inside) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int64_t cc = col0 + c0 + q;
          if (cc < A.Cp) {
            const int64_t b = cc / A.C, ch = cc - b * A.C;
            A.img[((b * A.h + py) * (int64_t)A.w + px) * A.C + ch] = __uint_as_float(v[q]);
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::);
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS));
  }
}

template <int NP>
static void launch_b(const TcArgs& A, int chunks, cudaStream_t st) {
  constexpr int STAGE = 2 * TC_P * 128 + 2 * NP * 128;
  const size_t smem = STAGE + 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_raster_b<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_raster_b<NP><<<dim3(A.ntiles * 2, chunks), 512, smem, st>>>(A);
}

int launch_raster_tc(const gsparc_frame_layout& L, char* frame, int n_tx, int C, double t_eps,
                     int pass, void* img, cudaStream_t st) {
  TcArgs A;
  A.tile_start = (const int*)(frame + L.off_tile_start);
  A.wstop = (int*)(frame + L.off_wstop);
  A.pair_rec = (const float4*)(frame + L.off_pair_rec);
  A.coef = (const float*)(frame + L.off_coef);
  A.live = (const int*)(frame + L.off_live);
  A.live_list = (int*)(frame + L.off_live_list);
  A.counters = (int*)(frame + L.off_counters);
  A.img = (float*)img;
  A.T_out = (float*)(frame + L.off_T);
  A.count_out = (int*)(frame + L.off_count);
  A.last_out = (int*)(frame + L.off_last);
  A.Cp = (int64_t)n_tx * C;
  A.C = C;
  A.w = L.width;
  A.h = L.height;
  A.ntx = L.ntx;
  A.ntiles = L.ntiles;
  A.t_eps = (float)t_eps;
  if (pass == 1) {
    if (cudaMemsetAsync(frame + L.off_live, 0, sizeof(int) * L.n, st) != cudaSuccess)
      return check_launch("raster_a live memset");
    k_raster_a<<<L.ntiles * 2, 512, 0, st>>>(A);
    return check_launch("k_raster_a");
  }
  // pass 2: channel columns per CTA (<= 256, multiple of 8)
  const int64_t Cp = A.Cp;
  const int chunks = (int)((Cp + 255) / 256);
  const int64_t per = (Cp + chunks - 1) / chunks;
  if (per <= 32) launch_b<32>(A, chunks, st);
  else if (per <= 64) launch_b<64>(A, chunks, st);
  else if (per <= 104) launch_b<104>(A, chunks, st);
  else if (per <= 128) launch_b<128>(A, chunks, st);
  else launch_b<256>(A, chunks, st);
  return check_launch("k_raster_b");
}

}  // namespace gs
