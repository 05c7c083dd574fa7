// Microbenchmark: cycles per tcgen05.mma.cta_group::1.kind::f16 (M=128, K=16,
// bf16 operands from shared memory) depending on the operand layout and on
// how the A/B descriptors change between consecutive MMAs.  One CTA, one
// issuing thread, 576 back-to-back MMAs, timed to the commit barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/mma_bench scripts/mma_bench.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

// layout 0: no swizzle, rows 16 B apart ([K/8][rows][8]); layout 2: SWIZZLE_128B
// K-major (rows 128 B = 64 K, 8-row atoms of 1 KB).
// walk: 0 fixed, 1 A walks conv taps/k-chunks, 2 B walks, 3 both walk,
//       4 both walk K only (GEMM-like, aligned)
__global__ void bench(int layout, int n, int walk, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_ptr;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tmem_ptr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_ptr;
  if (warp == 0) {  // whole warp runs the loop, elect.sync picks the issuing lane
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 96 * 1024);
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
    const uint32_t R = 160;  // A rows per k-chunk plane (conv tile + halo)
    uint64_t ad, bd;
    if (layout == 0) {
      ad = desc(a, R * 16, 128, 0);
      bd = desc(b, n * 16, 128, 0);
    } else {
      ad = desc(a, 16, 1024, 2);
      bd = desc(b, 16, 1024, 2);
    }
    uint32_t tap_a[9], tap_b[9];
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) {
      tap_a[tap] = (walk == 1 || walk == 3) ? (layout == 0 ? (tap / 3) * 15 + (tap % 3) : (tap / 3) * 64) : 0;
      tap_b[tap] = (walk == 2 || walk == 3) ? (tap % (n == 256 ? 2 : n == 128 ? 5 : 9)) * 8 * n : 0;
    }
    const uint32_t ka = (walk == 1 || walk == 3 || walk == 4) ? (layout == 0 ? 2 * R : 2) : 0;
    const uint32_t kb = (walk == 2 || walk == 3 || walk == 4) ? (layout == 0 ? 2 * n : 2) : 0;
    long long t0 = clock64();
    for (int rep = 0; rep < 16; ++rep) {
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        uint64_t a2 = ad + tap_a[tap], b2 = bd + tap_b[tap];
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
          asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                       "l"(a2), "l"(b2), "r"(idesc), "r"(rep | tap | kc));
          a2 += ka;
          b2 += kb;
        }
      }
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok)
                   : "r"(smem_u32(&bar)));
    if (threadIdx.x == 0) out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* walks[] = {"fixed", "A walks", "B walks", "A+B walk", "K-only walk"};
  for (int layout : {0, 2})
    for (int n : {64, 128, 256})
      for (int w = 0; w < 5; ++w) {
        long long h = 0;
        for (int rep = 0; rep < 3; ++rep) {
          bench<<<1, 128, 200 * 1024>>>(layout, n, w, d);
          cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        }
        cudaError_t e = cudaGetLastError();
        printf("%-6s N=%3d %-12s %7.1f cycles/MMA (math floor %d) %s\n", layout ? "sw128" : "noswz", n, walks[w],
               h / 576.0, n / 2, e == cudaSuccess ? "" : cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
      }
  return 0;
}
