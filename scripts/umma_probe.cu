// Probe of tcgen05.mma kind::tf32 with A in TMEM and B MN-major in shared
// memory (the operand layouts raster_px.cu's pass B relies on).  Builds
// D[128, N] = A[128, 32] . B[32, N] with exactly representable values and
// reports the max error per descriptor variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o /tmp/probe scripts/umma_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int N>
__global__ void probe(const float* A, const float* B, float* D, int variant) {
  constexpr int NA = (N + 31) / 32;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = (unsigned char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // B[k][n] -> MN-major SW128: atom (k/8, n/32) at (k/8)*NA*1024 + (n/32)*1024,
  // row k%8 (128 B), 16 B chunk ((n%32)/4) ^ (k%8)
  for (int e = tid; e < 32 * NA * 32; e += blockDim.x) {
    const int k = e / (NA * 32), n = e % (NA * 32);
    float v = n < N ? B[k * N + n] : 0.f;
    uint32_t off;
    if (variant == 4 && false) {
    } else if (variant == 4) {  // K-major SW128 control: row n, 128 B of k
      off = (uint32_t)(n * 128 + ((((k >> 2) ^ (n & 7)) << 4) | ((k & 3) << 2)));
    } else if (variant == 6 || variant == 7) {  // SW128_BASE32B: 4 k-rows x 128 B atoms
      const uint32_t w = (uint32_t)((n & 31) * 4);
      off = (uint32_t)((k >> 2) * (NA * 512) + (n >> 5) * 512 + (k & 3) * 128 +
                       ((((w >> 5) ^ (k & 3)) << 5) | (w & 31)));
    } else if (variant == 2 || variant == 3) {  // no swizzle, core = 8 k-rows x 16 B (4 n)
      off = (uint32_t)((n / 4) * 128 * 4 + (k / 8) * 128 + (k % 8) * 16 + (n % 4) * 4);
    } else {
      off = (uint32_t)((k >> 3) * (NA * 1024) + (n >> 5) * 1024 + (k & 7) * 128 +
                       ((((n & 31) >> 2) ^ (k & 7)) << 4) + (n & 3) * 4);
    }
    *(float*)(sm + off) = v;
  }
  // A rows in smem too (K-major SW128) at sm + 64 KB, for variant 5
  for (int e = tid; e < 128 * 32; e += blockDim.x) {
    const int m = e / 32, k = e % 32;
    *(float*)(sm + 65536 + m * 128 + ((((k >> 2) ^ (m & 7)) << 4) | ((k & 3) << 2))) = A[e];
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = s_tmem;
  // A rows -> TMEM columns [128, 160), lane = row
  {
    const int m = warp * 32 + lane;
    uint32_t v[32];
    for (int k = 0; k < 32; ++k) v[k] = __float_as_uint(A[m * 32 + k]);
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 128;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16};" ::"r"(ta),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
        "r"(v[15]));
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16};" ::"r"(ta + 16),
        "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]),
        "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]),
        "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t bmaj = variant == 4 ? 0u : 1u;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (bmaj << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint32_t b0 = smem_u32(sm);
    for (int ks = 0; ks < 4; ++ks) {
      uint64_t d = 0;
      uint32_t start, lbo, sbo, layout;
      if (variant == 0) {  // LBO = N-atom stride, SBO = K-group stride
        start = b0 + ks * NA * 1024;
        lbo = 1024;
        sbo = NA * 1024;
        layout = 2;
      } else if (variant == 1) {  // swapped
        start = b0 + ks * NA * 1024;
        lbo = NA * 1024;
        sbo = 1024;
        layout = 2;
      } else if (variant == 6 || variant == 7) {
        start = b0 + ks * 2 * NA * 512;
        lbo = variant == 6 ? 512 : NA * 512;
        sbo = variant == 6 ? NA * 512 : 512;
        layout = 1;
      } else if (variant == 4) {
        start = b0 + ks * 32;
        lbo = 16;
        sbo = 1024;
        layout = 2;
      } else {  // no swizzle: core (k8 x 4n), n-cores stride 512, k-groups stride 128
        start = b0 + ks * 128;
        lbo = 128 * 4;
        sbo = 128;
        layout = 0;
        if (variant == 3) {
          lbo = 128;
          sbo = 512;
        }
      }
      d |= (uint64_t)((start >> 4) & 0x3FFF);
      d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
      d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
      d |= (uint64_t)1 << 46;
      d |= (uint64_t)layout << 61;
      const uint32_t acc = ks > 0 ? 1u : 0u;
      if (variant == 5) {
        uint64_t da = 0;
        const uint32_t sa = b0 + 65536 + ks * 32;
        da |= (uint64_t)((sa >> 4) & 0x3FFF);
        da |= (uint64_t)1 << 16;
        da |= (uint64_t)(1024 >> 4) << 32;
        da |= (uint64_t)1 << 46;
        da |= (uint64_t)2 << 61;
        uint64_t db = 0;
        const uint32_t sb = b0 + ks * NA * 1024;
        db |= (uint64_t)((sb >> 4) & 0x3FFF);
        db |= (uint64_t)(1024 >> 4) << 16;
        db |= (uint64_t)((NA * 1024 >> 4) & 0x3FFF) << 32;
        db |= (uint64_t)1 << 46;
        db |= (uint64_t)2 << 61;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
        continue;
      }
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem),
          "r"(tmem + 128 + 8 * ks), "l"(d), "r"(idesc), "r"(acc));
    }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&bar)));
  }
  {
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
        "@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int m = warp * 32 + lane;
  for (int n0 = 0; n0 < N; n0 += 8) {
    uint32_t v[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16) + n0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) D[m * N + n0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int N>
void run() {
  float *A, *B, *D;
  cudaMallocManaged(&A, 128 * 32 * 4);
  cudaMallocManaged(&B, 32 * N * 4);
  cudaMallocManaged(&D, 128 * N * 4);
  for (int m = 0; m < 128; ++m)
    for (int k = 0; k < 32; ++k) A[m * 32 + k] = (float)((m * 7 + k * 3) % 11 - 5);
  for (int k = 0; k < 32; ++k)
    for (int n = 0; n < N; ++n) B[k * N + n] = (float)((k * 5 + n * 2) % 9 - 4);
  const int smem = 65536 + 128 * 128 + 1024;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int variant = 0; variant < 8; ++variant) {
    for (int i = 0; i < 128 * N; ++i) D[i] = -999.f;
    probe<N><<<1, 128, smem>>>(A, B, D, variant);
    cudaError_t e = cudaDeviceSynchronize();
    double err = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double r = 0;
        for (int k = 0; k < 32; ++k) r += (double)A[m * 32 + k] * B[k * N + n];
        err = fmax(err, fabs(r - D[m * N + n]));
      }
    printf("N=%d variant %d: %s max err %g (D[0]=%g D[1]=%g)\n", N, variant,
           cudaGetErrorString(e), err, D[0], D[1]);
    if (e != cudaSuccess) exit(1);
  }
}

int main() {
  run<64>();
  run<104>();
  run<128>();
  return 0;
}
