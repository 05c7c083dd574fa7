// Shared tcgen05 / TMA / mbarrier building blocks of the tensor-core path
// (PTX wrappers, UMMA descriptors, persistent work iteration, tensor maps).
#pragma once
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "nrx_device.cuh"
#include "nrx_kernels.h"

namespace nrx {
namespace tc {

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------

// Optional per-role cycle accounting (build with -DNRX_TIMING; CTA 0 prints).
#ifdef NRX_TIMING
#define NRX_T(var) long long var = clock64()
#define NRX_TADD(acc, var) (acc) += clock64() - (var)
#else
#define NRX_T(var)
#define NRX_TADD(acc, var)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
// 8 consecutive fp32 values (e.g. a bias chunk) from a 16-B aligned shared address
__device__ __forceinline__ void ld_shared_f8(uint32_t addr, float* b) {
  const float4 lo = ld_shared_f4(addr), hi = ld_shared_f4(addr + 16);
  b[0] = lo.x; b[1] = lo.y; b[2] = lo.z; b[3] = lo.w;
  b[4] = hi.x; b[5] = hi.y; b[6] = hi.z; b[7] = hi.w;
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// uint32 shared-address overloads (no generic->shared conversion per call)
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// "TMEM drained" signals: the arriving thread's tcgen05.ld reads are complete
// (tcgen05.wait::ld); no memory ordering is needed, and the default
// release-semantics arrive compiles to a MEMBAR that also waits for the
// thread's outstanding global stores.
__device__ __forceinline__ void mbar_arrive_relaxed(uint32_t bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* bar) { mbar_arrive_relaxed(smem_u32(bar)); }
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_try_wait(a, parity)) {
  }
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  while (!mbar_try_wait(a, parity)) {
  }
}
// Long waits of roles that share SM sub-partitions with the MMA warp (the
// epilogue waiting a whole tile for its accumulator, the producer waiting for
// a free stage): back off between polls so the spin does not take issue slots
// from the MMA issuer.
__device__ __forceinline__ void mbar_wait_backoff(uint32_t a, uint32_t parity, uint32_t ns) {
  while (!mbar_try_wait(a, parity)) __nanosleep(ns);
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// weights: bulk copies of <= 32 KB chunks, all completing on one barrier
__device__ __forceinline__ void load_weights(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  mbar_expect_tx(bar, bytes);
  for (uint32_t off = 0; off < bytes; off += 32768u) {
    const uint32_t n = bytes - off < 32768u ? bytes - off : 32768u;
    bulk_load(static_cast<uint8_t*>(dst) + off, static_cast<const uint8_t*>(src) + off, n, bar);
  }
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, bf16 in, fp32 accumulate
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Warp-wide variants: every lane of the issuing warp executes them with the
// same operands and elect.sync picks one lane, so the compiler keeps the
// descriptor arithmetic on the uniform datapath without per-MMA divergence
// wrappers (issue cost ~49 cycles/MMA instead of ~150 measured from a
// single-lane branch, scripts/mma_bench.cu).
__device__ __forceinline__ void mma_bf16_warp(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// fp32x3: D = A B + D 2^-11 (scale-input-d) folds the lo*Whi partial sums,
// accumulated at scale 2^11, into the hi terms (accumulate always on)
__device__ __forceinline__ void mma_fold_warp(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1, 11;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc)
      : "memory");
}
// fp32x3 GEMM over nk K=16 steps: lo*Whi for every step, then hi*Wlo (the
// first one folding the lo sums in), then hi*Whi.  The tensor core's fp32
// accumulation truncates (~0.2 ulp of D per MMA towards zero,
// scripts/acc_probe.cu), so the small terms go first and only the last nk
// MMAs run at the full magnitude of D.  A: [2 planes][K/8 chunks][rows][8]
// (hi plane first, a_lo = plane distance in 16-B units), B: [hi | lo][K/8][N][8]
// (b_lo likewise).
template <int NK>
__device__ __forceinline__ void mma_x3_gemm_t(uint32_t d, uint64_t a_hi, uint32_t a_lo, uint32_t a_k, uint64_t b_hi,
                                              uint32_t b_lo, uint32_t b_k, uint32_t idesc) {
#pragma unroll
  for (int k = 0; k < NK; ++k) mma_bf16_warp(d, a_hi + a_lo + k * a_k, b_hi + k * b_k, idesc, k != 0);
  mma_fold_warp(d, a_hi, b_hi + b_lo, idesc);
#pragma unroll
  for (int k = 1; k < NK; ++k) mma_bf16_warp(d, a_hi + k * a_k, b_hi + b_lo + k * b_k, idesc, 1);
#pragma unroll
  for (int k = 0; k < NK; ++k) mma_bf16_warp(d, a_hi + k * a_k, b_hi + k * b_k, idesc, 1);
}
// Unrolled issue for the K sizes of the per-RE MLPs (a runtime loop of
// elect-per-MMA issues costs ~3x per MMA); other sizes fall back to the loop.
__device__ __forceinline__ void mma_x3_gemm(uint32_t d, uint64_t a_hi, uint32_t a_lo, uint32_t a_k, uint64_t b_hi,
                                            uint32_t b_lo, uint32_t b_k, int nk, uint32_t idesc) {
  switch (nk) {
    case 1: mma_x3_gemm_t<1>(d, a_hi, a_lo, a_k, b_hi, b_lo, b_k, idesc); return;
    case 2: mma_x3_gemm_t<2>(d, a_hi, a_lo, a_k, b_hi, b_lo, b_k, idesc); return;
    case 4: mma_x3_gemm_t<4>(d, a_hi, a_lo, a_k, b_hi, b_lo, b_k, idesc); return;
    case 8: mma_x3_gemm_t<8>(d, a_hi, a_lo, a_k, b_hi, b_lo, b_k, idesc); return;
    default: break;
  }
  for (int k = 0; k < nk; ++k) mma_bf16_warp(d, a_hi + a_lo + k * a_k, b_hi + k * b_k, idesc, k != 0);
  mma_fold_warp(d, a_hi, b_hi + b_lo, idesc);
  for (int k = 1; k < nk; ++k) mma_bf16_warp(d, a_hi + k * a_k, b_hi + b_lo + k * b_k, idesc, 1);
  for (int k = 0; k < nk; ++k) mma_bf16_warp(d, a_hi + k * a_k, b_hi + k * b_k, idesc, 1);
}
__device__ __forceinline__ void mma_commit_warp(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mma_commit_warp(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 16 consecutive fp32 columns; caller issues tmem_wait_ld() before use
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor, K-major, no swizzle (core matrix = 8 rows
// x 16 bytes, rows 16 bytes apart): LBO = byte distance between the two
// 8-element K halves of one K=16 step, SBO = distance between 8-row groups.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  return d;                             // base offset 0, layout SWIZZLE_NONE
}

// kind::f16 instruction descriptor: fp32 accumulate, bf16 A/B, K-major A/B.
// Same for fp16 or bf16 operands by element type (A/B format 0 = F16, 1 = BF16).
template <typename ET>
__host__ __device__ constexpr uint32_t idesc_f16kind(int M, int N) {
  constexpr uint32_t fmt = std::is_same<ET, __half>::value ? 0u : 1u;
  return (1u << 4) | (fmt << 7) | (fmt << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ uint32_t tmem_cols_pow2(uint32_t n) {
  uint32_t c = 32;
  while (c < n) c <<= 1;
  return c;
}

// ---------------------------------------------------------------------------
// work distribution shared by all roles of a persistent CTA
// ---------------------------------------------------------------------------

struct WorkIter {
  int u, tl, stride, units, tps, n_io, io;
  bool first;
  const int32_t* mod;
  const Geom* g;
  __device__ WorkIter(const Geom& geo, int n_units, int tiles_per_unit, int n_io_sets, const int32_t* mods)
      : u(0), tl(0), stride(gridDim.x), units(n_units), tps(tiles_per_unit), n_io(n_io_sets), io(blockIdx.y),
        first(true), mod(mods), g(&geo) {}
  // next (unit, tile) owned by this CTA (flat index blockIdx.x + k * gridDim.x);
  // units are slabs (or slots).  Incremental: one division on the first call.
  __device__ bool next(int& unit, int& tile) {
    while (true) {
      if (first) {
        first = false;
        u = blockIdx.x / tps;
        tl = blockIdx.x - u * tps;
      } else {
        tl += stride;
        while (tl >= tps) {
          tl -= tps;
          ++u;
        }
      }
      if (u >= units) return false;
      if (n_io > 1 && io_index(mod, u, *g) != io) continue;
      unit = u;
      tile = tl;
      return true;
    }
  }
};


// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 4-D map over a chunk-planar bf16 buffer [NU][C/8][rows_slab][8], viewed
// as [NU][C/8][rows_slab/16][16 rows x 8 channels]: one TMA element row is
// 16 consecutive grid rows (256 contiguous bytes), so a box moves 256-byte
// requests instead of 16-byte ones.  Box {128, rbox/16, C/8, 1} lands as the
// K-major no-swizzle [C/8][rbox][8] tile; the row coordinate is in units of
// 16 rows (tiles start on 16-row boundaries, zero fill outside the slab).
inline int make_map(CUtensorMap* m, const void* base, const Geom& g, int C, int rbox, int box_chunks = 0) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return NRX_ERR_NO_DEVICE;
  if (rbox % 16 || g.rows_slab % 16) return NRX_ERR_UNSUPPORTED;
  const cuuint64_t dims[4] = {128, (cuuint64_t)(g.rows_slab / 16), (cuuint64_t)(C / 8), (cuuint64_t)g.NU};
  const cuuint64_t strides[3] = {256, (cuuint64_t)g.rows_slab * 16, (cuuint64_t)(C / 8) * g.rows_slab * 16};
  const cuuint32_t box[4] = {128, (cuuint32_t)(rbox / 16), (cuuint32_t)(box_chunks ? box_chunks : C / 8), 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? NRX_OK : NRX_ERR_CUDA;
}

// Launch with programmatic stream serialization (see pdl_wait); NRX_PDL=0 in
// the environment turns it off (plain stream order).
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("NRX_PDL");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}
template <typename... Args, typename... Act>
inline cudaError_t launch_pdl(void (*fn)(Args...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Act&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fn, std::forward<Act>(args)...);
}

inline int num_sms() {
  static int n[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!n[dev & 63]) cudaDeviceGetAttribute(&n[dev & 63], cudaDevAttrMultiProcessorCount, dev);
  return n[dev & 63] > 0 ? n[dev & 63] : 148;
}

// opt every tensor-core kernel into the full 227 KB once per device
inline int set_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static const void* done[64][16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (int i = 0; i < 16; ++i) {
    if (done[dev & 63][i] == fn) return NRX_OK;
    if (done[dev & 63][i] == nullptr) {
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
        return NRX_ERR_CUDA;
      done[dev & 63][i] = fn;
      return NRX_OK;
    }
  }
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess
             ? NRX_OK
             : NRX_ERR_CUDA;
}


constexpr size_t SMEM_LIMIT = 232448;  // 227 KB per CTA on sm_100

}  // namespace tc
}  // namespace nrx
