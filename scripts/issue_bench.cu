// Microbenchmark: cycles per CTA-pair MMA (tcgen05.mma.cta_group::2.kind::f16,
// M=256, N=64, K=16) for different ways of issuing the fp32x3 conv tile's
// 216 MMAs (9 taps x 8 K steps x 3 products, three tap-row accumulators) from
// the leader CTA's MMA warp.  Operands are whatever sits in shared memory;
// only the issue / execution rate is measured (clock64 around 64 tiles,
// through the final commit).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/issue_bench scripts/issue_bench.cu
#include <cuda_runtime.h>

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
__device__ __forceinline__ void mma_w(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// single thread (caller elected), 32-bit low words + constant high words
__device__ __forceinline__ void mma_1(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi,
                                      uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 ad, bd;\n\tmov.b64 ad, {%1, %2};\n\tmov.b64 bd, {%3, %4};\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], ad, bd, %5, p;\n\t}" ::"r"(d),
      "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_w32(uint32_t d, uint32_t alo, uint32_t ahi, uint32_t blo, uint32_t bhi,
                                        uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 ad, bd;\n\tmov.b64 ad, {%1, %2};\n\tmov.b64 bd, {%3, %4};\n\t"
      "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %6, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], ad, bd, %5, p;\n\t}" ::"r"(d),
      "r"(alo), "r"(ahi), "r"(blo), "r"(bhi), "r"(idesc), "r"(acc)
      : "memory");
}

constexpr int TILES = 64;

__global__ void __cluster_dims__(2, 1, 1) bench(int variant, int Tp, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_ptr;
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_ptr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_ptr;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  constexpr int R = 160, NPH = 32;
  const uint32_t As = smem_u32(smem), Ws = smem_u32(smem + 40 * 1024);
  long long t0 = 0, t1 = 0;
  if (rank == 0 && warp == 1) {
    int shifts[9];
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) shifts[tap] = (tap / 3 - 1) * Tp + (tap % 3 - 1);
    const uint64_t a0 = desc(As, R * 16, 128) + 16, bh = desc(Ws, NPH * 16, 128), bl = bh + 2304;
    t0 = clock64();
    if (variant == 0) {  // warp-wide, elect per MMA, 64-bit descriptor adds (the kernel's form)
      for (int t = 0; t < TILES; ++t) {
        const uint32_t d0 = tmem + (t & 1) * 192;
#pragma unroll
        for (int pl = 0; pl < 2; ++pl)
#pragma unroll
          for (int src = 0; src < 2; ++src) {
            const uint64_t as = a0 + (uint32_t)((pl * 2 + src) * 1280);
#pragma unroll
            for (int pass = 0; pass < 2; ++pass) {
              if (pass == 1 && pl == 0) break;
#pragma unroll
              for (int tap = 0; tap < 9; ++tap)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  const uint64_t a = as + shifts[tap] + (uint32_t)(k * 2 * R);
                  const uint32_t bo = (uint32_t)((tap * 16 + src * 8 + 2 * k) * NPH);
                  if (pl == 0) mma_w(d0, a, bh + bo, idesc, (src | tap | k) != 0);
                  else if (pass == 0) mma_w(d0, a, bl + bo, idesc, 1);
                  else mma_w(d0 + (tap / 3) * 64, a, bh + bo, idesc, (tap / 3) == 0 || (src | (tap % 3) | k) != 0);
                }
            }
          }
      }
    } else {
      const uint32_t a_lo0 = (uint32_t)a0, a_hi = (uint32_t)(a0 >> 32);
      const uint32_t bh_lo = (uint32_t)bh, b_hi = (uint32_t)(bh >> 32), bl_lo = (uint32_t)bl;
      bool leader = true;
      if (variant == 2) {
        uint32_t e;
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(e));
        leader = e != 0;
      }
      if (leader) {
        for (int t = 0; t < TILES; ++t) {
          const uint32_t d0 = tmem + (t & 1) * 192;
#pragma unroll
          for (int pl = 0; pl < 2; ++pl)
#pragma unroll
            for (int src = 0; src < 2; ++src) {
              const uint32_t as = a_lo0 + (uint32_t)((pl * 2 + src) * 1280);
#pragma unroll
              for (int pass = 0; pass < 2; ++pass) {
                if (pass == 1 && pl == 0) break;
#pragma unroll
                for (int tap = 0; tap < 9; ++tap)
#pragma unroll
                  for (int k = 0; k < 4; ++k) {
                    const uint32_t a = as + shifts[tap] + (uint32_t)(k * 2 * R);
                    const uint32_t bo = (uint32_t)((tap * 16 + src * 8 + 2 * k) * NPH);
                    if (variant == 1) {
                      if (pl == 0) mma_w32(d0, a, a_hi, bh_lo + bo, b_hi, idesc, (src | tap | k) != 0);
                      else if (pass == 0) mma_w32(d0, a, a_hi, bl_lo + bo, b_hi, idesc, 1);
                      else mma_w32(d0 + (tap / 3) * 64, a, a_hi, bh_lo + bo, b_hi, idesc, (tap / 3) == 0 || (src | (tap % 3) | k) != 0);
                    } else {
                      if (pl == 0) mma_1(d0, a, a_hi, bh_lo + bo, b_hi, idesc, (src | tap | k) != 0);
                      else if (pass == 0) mma_1(d0, a, a_hi, bl_lo + bo, b_hi, idesc, 1);
                      else mma_1(d0 + (tap / 3) * 64, a, a_hi, bh_lo + bo, b_hi, idesc, (tap / 3) == 0 || (src | (tap % 3) | k) != 0);
                    }
                  }
              }
            }
        }
      }
      __syncwarp();
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)3)
        : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    t1 = clock64();
    if (threadIdx.x == 32) out[variant] = t1 - t0;
  } else if (rank == 1 && warp == 1) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[3] = {"warp-wide elect per MMA, 64-bit desc", "warp-wide elect per MMA, 32-bit lo",
                          "elected thread, 32-bit lo"};
  for (int v = 0; v < 3; ++v) {
    for (int rep = 0; rep < 2; ++rep) bench<<<2, 128, smem>>>(v, 15, d);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("fail %d\n", v); return 1; }
    long long c;
    cudaMemcpy(&c, d + v, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %6.1f cycles per pair MMA (M=256 N=64 K=16)\n", names[v], (double)c / (TILES * 216));
  }
  return 0;
}
