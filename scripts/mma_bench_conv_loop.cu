// In-situ-like MMA issue loop: runtime trip counts, taps (ks x ks) x ks-steps,
// per-stage base; compare with fully unrolled constant offsets.
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__global__ void bench(int ks_, int Tp, int nks, int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_ptr;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_ptr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = threadIdx.x; i < 220 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;"); asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_ptr;
  if (warp == 1) {
    const int R = 160, NP = 64, r = ks_ / 2, kch = 2 * nks * 2;  // two sources of nks K-steps
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (8u << 17) | (8u << 24);
    const uint64_t a_desc0 = desc(0, R * 16, 128);
    const uint64_t b_desc0 = desc(smem_u32(smem), NP * 16, 128);
    const uint32_t As = smem_u32(smem + 150 * 1024);
    long long t0 = clock64();
    int nmma = 0;
    for (int it = 0; it < tiles; ++it) {
      const uint32_t d = tmem + (it & 1) * NP;
      for (int src = 0; src < 2; ++src) {
        const uint32_t a_stage = ((As + (it & 1) * 20480) >> 4) + 16;
        uint32_t b_tap = (uint32_t)(src * nks * 2) * NP;
        for (int ta = 0; ta < ks_; ++ta)
          for (int tb = 0; tb < ks_; ++tb) {
            uint64_t ad = a_desc0 + (a_stage + (ta - r) * Tp + (tb - r));
            uint64_t bd = b_desc0 + b_tap;
            const uint32_t first = (src | ta | tb) == 0;
#pragma unroll 4
            for (int k = 0; k < nks; ++k) {
              mma(d, ad, bd, idesc, !(first && k == 0));
              ad += 2 * R; bd += 2 * NP; ++nmma;
            }
            b_tap += (uint32_t)kch * NP;
          }
      }
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)));
    if (threadIdx.x == 32) { out[0] = clock64() - t0; out[1] = nmma; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int KS, int NKS>
__global__ void bench_t(int Tp, int tiles, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_ptr;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_ptr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  for (int i = threadIdx.x; i < 220 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;"); asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads(); asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_ptr;
  if (warp == 1) {
    constexpr int R = 160, NP = 64, r = KS / 2, kch = 2 * NKS * 2;
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (8u << 17) | (8u << 24);
    const uint64_t a_desc0 = desc(0, R * 16, 128);
    const uint64_t b_desc0 = desc(smem_u32(smem), NP * 16, 128);
    const uint32_t As = smem_u32(smem + 150 * 1024);
    int shifts[KS * KS];
#pragma unroll
    for (int ta = 0; ta < KS; ++ta)
#pragma unroll
      for (int tb = 0; tb < KS; ++tb) shifts[ta * KS + tb] = (ta - r) * Tp + (tb - r);
    long long t0 = clock64();
    int nmma = 0;
    for (int it = 0; it < tiles; ++it) {
      const uint32_t d = tmem + (it & 1) * NP;
#pragma unroll
      for (int src = 0; src < 2; ++src) {
        const uint64_t a_stage = a_desc0 + (((As + (it & 1) * 20480) >> 4) + 16);
#pragma unroll
        for (int tap = 0; tap < KS * KS; ++tap) {
#pragma unroll
          for (int k = 0; k < NKS; ++k) {
            mma(d, a_stage + shifts[tap] + k * 2 * R, b_desc0 + (uint32_t)((tap * kch + src * NKS * 2 + 2 * k) * NP),
                idesc, (src | tap | k) != 0);
            ++nmma;
          }
        }
      }
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)));
    if (threadIdx.x == 32) { out[0] = clock64() - t0; out[1] = nmma; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}
int main() {
  long long* d; cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int nthreads : {64, 320}) {
    long long h[2];
    for (int rep = 0; rep < 3; ++rep) { bench<<<1, nthreads, 220 * 1024>>>(3, 15, 4, 16, d); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); }
    printf("threads=%d: %.1f cycles/MMA over %lld MMAs (%s)\n", nthreads, (double)h[0] / h[1], h[1], cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(bench_t<3, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  {
    long long h[2];
    for (int rep = 0; rep < 3; ++rep) { bench_t<3, 4><<<1, 320, 220 * 1024>>>(15, 16, d); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); }
    printf("templated unrolled: %.1f cycles/MMA over %lld MMAs (%s)\n", (double)h[0] / h[1], h[1], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
