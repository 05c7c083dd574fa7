// Probe of the fp32 accumulation of tcgen05.mma.kind::f16 (fp16 in, fp32
// accumulate): NSTEP back-to-back K=16 MMAs into one TMEM accumulator,
// compared on the host with the exact (fp64) sum.  Reports the mean signed
// error (a round-toward-zero accumulator shows a bias towards zero) and the
// max error, both relative to |D|, next to fp32 round-to-nearest sequential
// accumulation of the same per-MMA partial sums.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/acc_probe scripts/acc_probe.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
constexpr int M = 128, N = 64, KS = 16;  // KS K=16 slices resident

// A [KS][2][M][8], B [KS][2][N][8] fp16 in global (already in core-matrix order)
__global__ void probe(const __half* A, const __half* B, int nstep, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_ptr;
  __shared__ __align__(8) uint64_t bar;
  __half* As = reinterpret_cast<__half*>(smem);
  __half* Bs = As + KS * 2 * M * 8;
  for (int i = threadIdx.x; i < KS * 2 * M * 8; i += blockDim.x) As[i] = A[i];
  for (int i = threadIdx.x; i < KS * 2 * N * 8; i += blockDim.x) Bs[i] = B[i];
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tmem_ptr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_ptr;
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int s = 0; s < nstep; ++s) {
      const int k = s % KS;
      const uint64_t ad = desc(smem_u32(As + k * 2 * M * 8), M * 16, 128);
      const uint64_t bd = desc(smem_u32(Bs + k * 2 * N * 8), N * 16, 128);
      asm volatile(
          "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(s));
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar)));
  }
  if (warp < 4) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;");
    const int row = 32 * warp + (threadIdx.x & 31);
    for (int c = 0; c < N; c += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(tmem + ((uint32_t)(32 * warp) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int e = 0; e < 8; ++e) out[row * N + c + e] = __uint_as_float(r[e]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
  }
}

int main() {
  srand(1);
  const size_t na = (size_t)KS * 2 * M * 8, nb = (size_t)KS * 2 * N * 8;
  std::vector<__half> A(na), B(nb);
  std::vector<double> Af(na), Bf(nb);
  // values with a spread of exponents (like activations / weights), mixed signs
  for (size_t i = 0; i < na; ++i) {
    const double v = ((rand() % 2) ? 1 : -1) * std::ldexp(1.0 + (rand() % 1024) / 1024.0, -(rand() % 6));
    A[i] = __float2half((float)v);
    Af[i] = __half2float(A[i]);
  }
  for (size_t i = 0; i < nb; ++i) {
    const double v = ((rand() % 3) ? 1 : -1) * std::ldexp(1.0 + (rand() % 1024) / 1024.0, 8 - (rand() % 6));
    B[i] = __float2half((float)v);
    Bf[i] = __half2float(B[i]);
  }
  __half *dA, *dB;
  float* dO;
  cudaMalloc(&dA, na * 2);
  cudaMalloc(&dB, nb * 2);
  cudaMalloc(&dO, M * N * 4);
  cudaMemcpy(dA, A.data(), na * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), nb * 2, cudaMemcpyHostToDevice);
  const size_t smem = (na + nb) * 2;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  auto elem = [&](const std::vector<double>& X, int rows, int k, int r, int kk) {  // [KS][2][rows][8]
    return X[(((size_t)k * 2 + kk / 8) * rows + r) * 8 + kk % 8];
  };
  for (int nstep : {1, 8, 72, 216}) {
    probe<<<1, 128, smem>>>(dA, dB, nstep, dO);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("launch failed\n"); return 1; }
    std::vector<float> O(M * N);
    cudaMemcpy(O.data(), dO, M * N * 4, cudaMemcpyDeviceToHost);
    double bias = 0, mx = 0, bias_rn = 0, mx_rn = 0;
    for (int r = 0; r < M; ++r)
      for (int n = 0; n < N; ++n) {
        double exact = 0;
        float rn = 0.f;
        for (int s = 0; s < nstep; ++s) {
          const int k = s % KS;
          double part = 0;
          for (int kk = 0; kk < 16; ++kk) part += elem(Af, M, k, r, kk) * elem(Bf, N, k, n, kk);
          exact += part;
          rn = (float)((double)rn + (double)(float)part);  // fp32 RN of each partial, RN accumulate
        }
        const double ulp = std::ldexp(1.0, std::ilogb(exact) - 23);
        const double e = (O[r * N + n] - exact) / ulp, erx = ((double)rn - exact) / ulp;
        // signed towards zero: negative = magnitude reduced
        bias += (exact >= 0 ? e : -e);
        bias_rn += (exact >= 0 ? erx : -erx);
        mx = std::fmax(mx, std::fabs(e));
        mx_rn = std::fmax(mx_rn, std::fabs(erx));
      }
    printf("nstep=%3d  tensor core: mean signed err %+.3f ulp(D), max %.2f ulp   |   fp32 RN: mean %+.3f, max %.2f\n",
           nstep, bias / (M * N), mx, bias_rn / (M * N), mx_rn);
  }
  return 0;
}
