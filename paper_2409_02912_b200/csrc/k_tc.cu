// bf16 tensor-core path (NRX_BF16): tcgen05.mma with TMEM accumulators, TMA
// tile loads, mbarrier pipelines, persistent CTAs.
//
//  k_conv_tc     k x k 'same' convolution as an implicit GEMM on the
//                row-linearised grid (nrx_internal.h).  Per 128-row M tile the
//                producer warp TMA-loads the tile plus +-H halo rows of every
//                input channel chunk ONCE (4-D box {8, 128+2H, C/8, 1}, zero
//                filled outside the slab); tap (a,b) is the same shared-memory
//                tile viewed at a row offset (a-r)*Tp + (b-r), which the
//                no-swizzle K-major UMMA descriptor addresses directly (16-byte
//                granular start address).  The whole layer's weights stay
//                resident in shared memory (bulk copy once per CTA).  One
//                thread issues taps * C/16 MMAs (M=128, N=rup(d,16), K=16) into
//                one of two TMEM accumulators; four epilogue warps drain the
//                other (tcgen05.ld) and apply bias / ReLU / positional channels /
//                fp32 residual while the next tile's MMAs run.
//  k_msg_tc      message MLP of every UE of a slot on a 128-RE tile (two
//                chained MMAs per UE, the ReLU'd hidden layer round-trips
//                TMEM -> registers -> shared memory as the next A operand),
//                messages kept in TMEM, then the float64 sum-of-others
//                (autodiff.py:276-294) in the epilogue.
//  k_readout_tc  LLR and channel-estimate MLPs fused into one N=2h GEMM plus a
//                block-diagonal N=32 GEMM; writes the (N,U,S,T,W) LLR and the
//                planar-decoded complex64 chest directly (nrx.py:266-289,382-384).
#include <cuda.h>

#include <mutex>

#include "nrx_device.cuh"
#include "nrx_kernels.h"
#include "nrx_profile.h"

namespace nrx {
namespace tc {

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
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
  int t, stride, total, tps, n_io, io;
  const int32_t* mod;
  const Geom* g;
  __device__ WorkIter(const Geom& geo, int units, int tiles_per_unit, int n_io_sets, const int32_t* mods)
      : t(blockIdx.x), stride(gridDim.x), total(units * tiles_per_unit), tps(tiles_per_unit), n_io(n_io_sets),
        io(blockIdx.y), mod(mods), g(&geo) {}
  // next (unit, tile) owned by this CTA; units are slabs (or slots)
  __device__ bool next(int& unit, int& tile) {
    while (t < total) {
      const int u = t / tps, tl = t - u * tps;
      t += stride;
      if (n_io > 1 && io_index(mod, u, *g) != io) continue;
      unit = u;
      tile = tl;
      return true;
    }
    return false;
  }
};

// ---------------------------------------------------------------------------
// K2/K3b/K3c: convolution
// ---------------------------------------------------------------------------

struct ConvTcParams {
  Geom g;
  int ktap, c0, c1;     // A channels per tap = c0 (source 0) + c1 (source 1)
  int np, cdst, mode, stages;
  int n_io, d4;
  uint32_t wbytes, abytes, tmem_cols, rbox;
  const uint8_t* wbase;
  uint64_t w_off[NRX_MAX_IO], b_off[NRX_MAX_IO];
  const int32_t* mod_order;
  __nv_bfloat16* dst;
  float* dst32;         // fp32 master state (STATE_INIT / RESIDUAL), or null
};

// warp 0 TMA producer, warp 1 MMA issuer, warps 2-9 epilogue (two warps per
// TMEM lane quarter, each draining half of the accumulator columns)
constexpr int CONV_THREADS = 320;
constexpr int CONV_EPI_THREADS = 256;

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

template <int NP, int MODE>
__global__ void __launch_bounds__(CONV_THREADS, 1)
    k_conv_tc(const __grid_constant__ ConvTcParams p, const __grid_constant__ CUtensorMap map0,
              const __grid_constant__ CUtensorMap map1) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const Geom& g = p.g;
  const int io = p.n_io > 1 ? blockIdx.y : 0;
  uint8_t* Ws = smem;
  uint8_t* As = smem + ((p.wbytes + 1023) & ~1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(As + (size_t)p.stages * p.abytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + 8;
  uint64_t* tfull = bars + 16;
  uint64_t* tempty = bars + 18;
  uint64_t* wbar = bars + 20;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(bars + 21);
  float* sbias = reinterpret_cast<float*>(bars + 22);  // NP floats

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(tmem_ptr, p.tmem_cols);
  if (threadIdx.x == 32) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], CONV_EPI_THREADS);
    }
    mbar_init(wbar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x >= 64 && threadIdx.x < 64 + NP)
    sbias[threadIdx.x - 64] = reinterpret_cast<const float*>(p.wbase + p.b_off[io])[threadIdx.x - 64];
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;
  const int R = p.rbox;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      load_weights(Ws, p.wbase + p.w_off[io], p.wbytes, wbar);
      WorkIter w(g, g.NU, g.tiles, p.n_io, p.mod_order);
      int slab, tile, st = 0;
      uint32_t ph = 0;
      while (w.next(slab, tile)) {
        mbar_wait(&empty[st], ph ^ 1);
        mbar_expect_tx(&full[st], p.abytes);
        uint8_t* a = As + (size_t)st * p.abytes;
        const int row0 = tile * NRX_TILE_M - g.H;
        tma_load_4d(a, &map0, &full[st], 0, row0, 0, slab);
        if (p.c1) tma_load_4d(a + (size_t)(p.c0 / 8) * R * 16, &map1, &full[st], 0, row0, 0, slab);
        if (++st == p.stages) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16(NRX_TILE_M, NP);
      const uint32_t wsm = smem_u32(Ws);
      const int kch = p.ktap / 8;  // 16-byte channel chunks per tap
      mbar_wait(wbar, 0);
      tc_fence_after();
      WorkIter w(g, g.NU, g.tiles, p.n_io, p.mod_order);
      int slab, tile, st = 0, it = 0;
      uint32_t ph = 0;
      while (w.next(slab, tile)) {
        const int acc = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        mbar_wait(&full[st], ph);
        tc_fence_after();
        const uint32_t asm_ = smem_u32(As + (size_t)st * p.abytes);
        const uint32_t d = tmem_base + acc * p.np;
        const int taps = g.ks * g.ks;
        for (int tap = 0; tap < taps; ++tap) {
          const int ta = tap / g.ks, tb = tap - ta * g.ks;
          const int shift = (ta - g.r) * g.Tp + (tb - g.r);
          for (int kc = 0; kc < kch; kc += 2) {
            const uint64_t ad = smem_desc(asm_ + (uint32_t)((kc * R + g.H + shift) * 16), (uint32_t)R * 16, 128);
            const uint64_t bd = smem_desc(wsm + (uint32_t)((tap * kch + kc) * p.np * 16), (uint32_t)p.np * 16, 128);
            mma_bf16(d, ad, bd, idesc, (tap | kc) != 0);
          }
        }
        mma_commit(&empty[st]);
        mma_commit(&tfull[acc]);
        if (++st == p.stages) { st = 0; ph ^= 1; }
        ++it;
      }
    }
  } else {  // ---------------- epilogue: warps 2..9
    constexpr int NC = NP / 2;  // accumulator columns per thread
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int r = 32 * q + lane;
    const int cbase = half * NC;
    const int nd = p.cdst / 8, n32 = p.d4 / 4;
    WorkIter w(g, g.NU, g.tiles, p.n_io, p.mod_order);
    int slab, tile, it = 0;
    while (w.next(slab, tile)) {
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      float v[NC];
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(32 * q) << 16) + acc * NP + cbase;
#pragma unroll
      for (int c = 0; c < NC / 8; ++c) tmem_ld8(taddr + 8 * c, v + 8 * c);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&tempty[acc]);

      const int row = tile * NRX_TILE_M + r;
      const int s = row / g.Tp, t = row - s * g.Tp;
      const bool valid = row < g.rows_data && t < g.T;
      float old[NC];
      if (MODE == EPI_RESIDUAL) {  // fp32 residual stream: issue every load before use
#pragma unroll
        for (int c4 = 0; c4 < NC / 4; ++c4) {
          const int cc = cbase / 4 + c4;
          float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
          if (valid && cc < n32) o = *reinterpret_cast<const float4*>(chunk_ptr(p.dst32, slab, n32, cc, row, g));
          old[4 * c4 + 0] = o.x;
          old[4 * c4 + 1] = o.y;
          old[4 * c4 + 2] = o.z;
          old[4 * c4 + 3] = o.w;
        }
      }
      float x[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const int c = cbase + j;
        float y = v[j] + sbias[c];  // conv + bias first, as the reference adds them
        if (MODE == EPI_RELU) y = fmaxf(y, 0.f);
        if (MODE == EPI_RESIDUAL) y = old[j] + y;
        x[j] = (valid && c < g.d) ? y : 0.f;
      }
      if (MODE != EPI_RELU) {
#pragma unroll
        for (int c4 = 0; c4 < NC / 4; ++c4) {
          const int cc = cbase / 4 + c4;
          if (cc < n32) store_chunk(chunk_ptr(p.dst32, slab, n32, cc, row, g), x + 4 * c4);
        }
        if (valid) {  // positional channels d, d+1 of the bf16 operand copy
          const float pdt = g.dt[t], pdf = pos_df(s, slab % g.U, g);
#pragma unroll
          for (int j = 0; j < NC; ++j) {
            const int c = cbase + j;
            if (c == g.d) x[j] = pdt;
            if (c == g.d + 1) x[j] = pdf;
          }
        }
      }
#pragma unroll
      for (int c8 = 0; c8 < NC / 8; ++c8) {
        const int cc = cbase / 8 + c8;
        if (cc < nd) store_chunk(chunk_ptr(p.dst, slab, nd, cc, row, g), x + 8 * c8);
      }
      if (half == 1) {  // buffer channels beyond the accumulator: positional / zero only
        for (int cc = NP / 8; cc < nd; ++cc) {
          float o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            o[e] = (valid && MODE != EPI_RELU) ? state_extra(8 * cc + e, s, t, slab % g.U, g) : 0.f;
          store_chunk(chunk_ptr(p.dst, slab, nd, cc, row, g), o);
        }
      }
      ++it;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// ---------------------------------------------------------------------------
// K3a: message MLP + float64 sum of the other UEs' messages
// ---------------------------------------------------------------------------

struct MsgTcParams {
  Geom g;
  int cs, hp, np;
  uint32_t w0bytes, w1bytes, abytes, hbytes, tmem_cols;
  const uint8_t* wbase;
  uint64_t w0, b0, w1, b1;
  __nv_bfloat16* agg;
};

constexpr int MLP_THREADS = 192;
constexpr int MSG_MAXU = 4;  // UEs per slot on the tensor-core path

__global__ void __launch_bounds__(MLP_THREADS, 1)
    k_msg_tc(const __grid_constant__ MsgTcParams p, const __grid_constant__ CUtensorMap smap) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const Geom& g = p.g;
  uint8_t* W0 = smem;
  uint8_t* W1 = W0 + p.w0bytes;
  uint8_t* As = W1 + p.w1bytes;  // 2 stages
  uint8_t* Hs = As + 2 * p.abytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(Hs + p.hbytes);
  uint64_t* afull = bars;        // [2]
  uint64_t* aempty = bars + 2;   // [2]
  uint64_t* hid_full = bars + 4;
  uint64_t* h_ready = bars + 5;
  uint64_t* h_used = bars + 6;
  uint64_t* msg_full = bars + 7;
  uint64_t* t_empty = bars + 8;
  uint64_t* wbar = bars + 9;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(bars + 10);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(tmem_ptr, p.tmem_cols);
  if (threadIdx.x == 32) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    mbar_init(hid_full, 1);
    mbar_init(h_ready, 128);
    mbar_init(h_used, 1);
    mbar_init(msg_full, 1);
    mbar_init(t_empty, 128);
    mbar_init(wbar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;
  const int U = g.U;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(wbar, p.w0bytes + p.w1bytes);
      bulk_load(W0, p.wbase + p.w0, p.w0bytes, wbar);
      bulk_load(W1, p.wbase + p.w1, p.w1bytes, wbar);
      WorkIter w(g, g.N, g.tiles, 1, nullptr);
      int n, tile, st = 0;
      uint32_t ph = 0;
      while (w.next(n, tile)) {
        for (int u = 0; u < U; ++u) {
          mbar_wait(&aempty[st], ph ^ 1);
          mbar_expect_tx(&afull[st], p.abytes);
          tma_load_4d(As + (size_t)st * p.abytes, &smap, &afull[st], 0, tile * NRX_TILE_M, 0, n * U + u);
          if (++st == 2) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id0 = idesc_bf16(NRX_TILE_M, p.hp), id1 = idesc_bf16(NRX_TILE_M, p.np);
      const uint32_t w0s = smem_u32(W0), w1s = smem_u32(W1), hs = smem_u32(Hs);
      mbar_wait(wbar, 0);
      tc_fence_after();
      WorkIter w(g, g.N, g.tiles, 1, nullptr);
      int n, tile, st = 0, item = 0, use = 0;
      uint32_t ph = 0;
      while (w.next(n, tile)) {
        mbar_wait(t_empty, (item & 1) ^ 1);  // epilogue finished the previous item
        tc_fence_after();
        for (int u = 0; u < U; ++u, ++use) {
          mbar_wait(&afull[st], ph);
          tc_fence_after();
          const uint32_t as = smem_u32(As + (size_t)st * p.abytes);
          for (int kc = 0; kc < p.cs / 8; kc += 2)
            mma_bf16(tmem_base, smem_desc(as + kc * NRX_TILE_M * 16, NRX_TILE_M * 16, 128),
                     smem_desc(w0s + kc * p.hp * 16, p.hp * 16, 128), id0, kc != 0);
          mma_commit(&aempty[st]);
          mma_commit(hid_full);
          if (++st == 2) { st = 0; ph ^= 1; }
          mbar_wait(h_ready, use & 1);
          tc_fence_after();
          const uint32_t dmsg = tmem_base + p.hp + u * p.np;
          for (int kc = 0; kc < p.hp / 8; kc += 2)
            mma_bf16(dmsg, smem_desc(hs + kc * NRX_TILE_M * 16, NRX_TILE_M * 16, 128),
                     smem_desc(w1s + kc * p.np * 16, p.np * 16, 128), id1, kc != 0);
          mma_commit(h_used);
        }
        mma_commit(msg_full);
        ++item;
      }
    }
  } else {
    const int q = warp & 3;
    const int r = 32 * q + lane;
    const uint32_t lane_off = static_cast<uint32_t>(32 * q) << 16;
    const float* b0 = reinterpret_cast<const float*>(p.wbase + p.b0);
    const float* b1 = reinterpret_cast<const float*>(p.wbase + p.b1);
    const int nca = g.Ca / 8;
    WorkIter w(g, g.N, g.tiles, 1, nullptr);
    int n, tile, item = 0, use = 0;
    while (w.next(n, tile)) {
      const int row = tile * NRX_TILE_M + r;
      const int s = row / g.Tp, t = row - s * g.Tp;
      const bool valid = row < g.rows_data && t < g.T;
      for (int u = 0; u < U; ++u, ++use) {
        mbar_wait(hid_full, use & 1);
        tc_fence_after();
        if (use > 0) mbar_wait(h_used, (use - 1) & 1);  // fc1 of the previous UE read Hs
        for (int c16 = 0; c16 < p.hp / 16; ++c16) {
          float v[16];
          tmem_ld16(tmem_base + lane_off + c16 * 16, v);
          tmem_wait_ld();
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            float o[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = fmaxf(v[8 * h2 + e] + b0[16 * c16 + 8 * h2 + e], 0.f);
            store_chunk(reinterpret_cast<__nv_bfloat16*>(Hs + ((size_t)(2 * c16 + h2) * NRX_TILE_M + r) * 16), o);
          }
        }
        fence_proxy_async();
        tc_fence_before();
        mbar_arrive(h_ready);
      }
      mbar_wait(msg_full, item & 1);
      tc_fence_after();
      for (int c16 = 0; c16 < p.np / 16; ++c16) {
        float m[MSG_MAXU][16];
#pragma unroll
        for (int u = 0; u < MSG_MAXU; ++u)
          if (u < U) tmem_ld16(tmem_base + lane_off + p.hp + u * p.np + c16 * 16, m[u]);
        tmem_wait_ld();
        double tot[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          tot[e] = 0.0;
          const float bb = b1[16 * c16 + e];
#pragma unroll
          for (int u = 0; u < MSG_MAXU; ++u)
            if (u < U) {
              m[u][e] += bb;
              tot[e] += (double)m[u][e];
            }
        }
#pragma unroll
        for (int u = 0; u < MSG_MAXU; ++u) {
          if (u >= U) break;
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int c8 = 2 * c16 + h2;
            if (c8 >= nca) break;
            float o[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int c = 8 * c8 + e;
              o[e] = (valid && c < g.d) ? (float)(tot[8 * h2 + e] - (double)m[u][8 * h2 + e]) : 0.f;
            }
            store_chunk(chunk_ptr(p.agg, n * U + u, nca, c8, row, g), o);
          }
        }
      }
      tc_fence_before();
      mbar_arrive(t_empty);
      ++item;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// ---------------------------------------------------------------------------
// K4: fused LLR + chest readout
// ---------------------------------------------------------------------------

struct ReadoutTcParams {
  Geom g;
  int cs, h2p, n_io;
  uint32_t w0bytes, w1bytes, abytes, hbytes, tmem_cols;
  const uint8_t* wbase;
  uint64_t w0[NRX_MAX_IO], b0[NRX_MAX_IO], w1[NRX_MAX_IO], b1[NRX_MAX_IO];
  const int32_t* mod_order;
  float* llr;
  float2* chest;
};

__global__ void __launch_bounds__(MLP_THREADS, 1)
    k_readout_tc(const __grid_constant__ ReadoutTcParams p, const __grid_constant__ CUtensorMap smap) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const Geom& g = p.g;
  const int io = p.n_io > 1 ? blockIdx.y : 0;
  uint8_t* W0 = smem;
  uint8_t* W1 = W0 + p.w0bytes;
  uint8_t* As = W1 + p.w1bytes;
  uint8_t* Hs = As + 2 * p.abytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(Hs + p.hbytes);
  uint64_t* afull = bars;
  uint64_t* aempty = bars + 2;
  uint64_t* hid_full = bars + 4;
  uint64_t* h_ready = bars + 5;
  uint64_t* out_full = bars + 6;
  uint64_t* t_empty = bars + 7;
  uint64_t* wbar = bars + 8;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(bars + 9);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc(tmem_ptr, p.tmem_cols);
  if (threadIdx.x == 32) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    mbar_init(hid_full, 1);
    mbar_init(h_ready, 128);
    mbar_init(out_full, 1);
    mbar_init(t_empty, 128);
    mbar_init(wbar, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(wbar, p.w0bytes + p.w1bytes);
      bulk_load(W0, p.wbase + p.w0[io], p.w0bytes, wbar);
      bulk_load(W1, p.wbase + p.w1[io], p.w1bytes, wbar);
      WorkIter w(g, g.NU, g.tiles, p.n_io, p.mod_order);
      int slab, tile, st = 0;
      uint32_t ph = 0;
      while (w.next(slab, tile)) {
        mbar_wait(&aempty[st], ph ^ 1);
        mbar_expect_tx(&afull[st], p.abytes);
        tma_load_4d(As + (size_t)st * p.abytes, &smap, &afull[st], 0, tile * NRX_TILE_M, 0, slab);
        if (++st == 2) { st = 0; ph ^= 1; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t id0 = idesc_bf16(NRX_TILE_M, p.h2p), id1 = idesc_bf16(NRX_TILE_M, 32);
      const uint32_t w0s = smem_u32(W0), w1s = smem_u32(W1), hs = smem_u32(Hs);
      mbar_wait(wbar, 0);
      tc_fence_after();
      WorkIter w(g, g.NU, g.tiles, p.n_io, p.mod_order);
      int slab, tile, st = 0, item = 0;
      uint32_t ph = 0;
      while (w.next(slab, tile)) {
        mbar_wait(t_empty, (item & 1) ^ 1);
        tc_fence_after();
        mbar_wait(&afull[st], ph);
        tc_fence_after();
        const uint32_t as = smem_u32(As + (size_t)st * p.abytes);
        for (int kc = 0; kc < p.cs / 8; kc += 2)
          mma_bf16(tmem_base, smem_desc(as + kc * NRX_TILE_M * 16, NRX_TILE_M * 16, 128),
                   smem_desc(w0s + kc * p.h2p * 16, p.h2p * 16, 128), id0, kc != 0);
        mma_commit(&aempty[st]);
        mma_commit(hid_full);
        if (++st == 2) { st = 0; ph ^= 1; }
        mbar_wait(h_ready, item & 1);
        tc_fence_after();
        for (int kc = 0; kc < p.h2p / 8; kc += 2)
          mma_bf16(tmem_base + p.h2p, smem_desc(hs + kc * NRX_TILE_M * 16, NRX_TILE_M * 16, 128),
                   smem_desc(w1s + kc * 32 * 16, 32 * 16, 128), id1, kc != 0);
        mma_commit(out_full);
        ++item;
      }
    }
  } else {
    const int q = warp & 3;
    const int r = 32 * q + lane;
    const uint32_t lane_off = static_cast<uint32_t>(32 * q) << 16;
    const float* b0 = reinterpret_cast<const float*>(p.wbase + p.b0[io]);
    const float* b1 = reinterpret_cast<const float*>(p.wbase + p.b1[io]);
    WorkIter w(g, g.NU, g.tiles, p.n_io, p.mod_order);
    int slab, tile, item = 0;
    while (w.next(slab, tile)) {
      mbar_wait(hid_full, item & 1);
      tc_fence_after();
      for (int c16 = 0; c16 < p.h2p / 16; ++c16) {
        float v[16];
        tmem_ld16(tmem_base + lane_off + c16 * 16, v);
        tmem_wait_ld();
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          float o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] = fmaxf(v[8 * h2 + e] + b0[16 * c16 + 8 * h2 + e], 0.f);
          store_chunk(reinterpret_cast<__nv_bfloat16*>(Hs + ((size_t)(2 * c16 + h2) * NRX_TILE_M + r) * 16), o);
        }
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(h_ready);
      mbar_wait(out_full, item & 1);
      tc_fence_after();
      float o[32];
      tmem_ld16(tmem_base + lane_off + p.h2p, o);
      tmem_ld16(tmem_base + lane_off + p.h2p + 16, o + 16);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(t_empty);
      const int row = tile * NRX_TILE_M + r;
      const int s = row / g.Tp, t = row - s * g.Tp;
      if (row < g.rows_data && t < g.T) {
        const int mio = io_index(p.mod_order, slab, g);
        const int width = mio < 0 ? 0 : g.io_width[mio];
        const size_t re = ((size_t)slab * g.S + s) * g.T + t;
        float* lp = p.llr + re * g.llr_width;
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (c < g.llr_width) lp[c] = mio < 0 ? __int_as_float(0x7fc00000) : (c < width ? o[c] + b1[c] : 0.f);
        float2* cp = p.chest + re * g.B;
#pragma unroll
        for (int b = 0; b < 8; ++b)
          if (b < g.B) cp[b] = make_float2(o[8 + b] + b1[8 + b], o[8 + g.B + b] + b1[8 + g.B + b]);
      }
      ++item;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
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

// 4-D map over a chunk-planar bf16 buffer [NU][C/8][rows_slab][8]; box
// {8, rbox, C/8, 1} lands as the K-major no-swizzle [C/8][rbox][8] tile.
static int make_map(CUtensorMap* m, const void* base, const Geom& g, int C, int rbox) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return NRX_ERR_NO_DEVICE;
  const cuuint64_t dims[4] = {8, (cuuint64_t)g.rows_slab, (cuuint64_t)(C / 8), (cuuint64_t)g.NU};
  const cuuint64_t strides[3] = {16, (cuuint64_t)g.rows_slab * 16, (cuuint64_t)(C / 8) * g.rows_slab * 16};
  const cuuint32_t box[4] = {8, (cuuint32_t)rbox, (cuuint32_t)(C / 8), 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? NRX_OK : NRX_ERR_CUDA;
}

static int num_sms() {
  static int n[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!n[dev & 63]) cudaDeviceGetAttribute(&n[dev & 63], cudaDevAttrMultiProcessorCount, dev);
  return n[dev & 63] > 0 ? n[dev & 63] : 148;
}

// opt every tensor-core kernel into the full 227 KB once per device
static int set_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static const void* done[64][4] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  for (int i = 0; i < 4; ++i) {
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

static int launch_conv(const Geom& g, const PackLayout& L, const ConvOff* offs, int n_off, const void* src0,
                       int c0, const void* src1, int c1, __nv_bfloat16* dst, int cdst, float* dst32, int mode,
                       const uint8_t* wb, const int32_t* mod_order, cudaStream_t st) {
  ConvTcParams p{};
  p.g = g;
  p.ktap = c0 + c1;
  p.c0 = c0;
  p.c1 = c1;
  p.np = rup(g.d, 16);
  p.cdst = cdst;
  p.mode = mode;
  p.n_io = n_off;
  p.d4 = rup(g.d, 4);
  // rows per channel chunk in shared memory; a multiple of 8 keeps every
  // chunk (and so the second source's TMA destination) 128-byte aligned
  p.rbox = rup(NRX_TILE_M + 2 * g.H, 8);
  p.wbytes = (uint32_t)(g.ks * g.ks * p.ktap * p.np * 2);
  p.abytes = (uint32_t)(p.ktap * p.rbox * 2);
  p.tmem_cols = p.np * 2 <= 32 ? 32 : p.np * 2 <= 64 ? 64 : p.np * 2 <= 128 ? 128 : 256;
  p.wbase = wb;
  for (int i = 0; i < n_off; ++i) {
    p.w_off[i] = offs[i].w;
    p.b_off[i] = offs[i].b;
  }
  p.mod_order = mod_order;
  p.dst = dst;
  p.dst32 = dst32;
  const size_t fixed = ((p.wbytes + 1023) & ~1023u) + 22 * 8 + 64 * 4 + 64;
  int stages = 4;
  while (stages > 1 && fixed + (size_t)stages * p.abytes > SMEM_LIMIT) --stages;
  if (fixed + (size_t)stages * p.abytes > SMEM_LIMIT || p.rbox > 256) return NRX_ERR_UNSUPPORTED;
  p.stages = stages;
  const size_t smem = fixed + (size_t)stages * p.abytes;
  CUtensorMap m0, m1;
  int rc = make_map(&m0, src0, g, c0, p.rbox);
  if (rc) return rc;
  rc = make_map(&m1, src1 ? src1 : src0, g, c1 ? c1 : c0, p.rbox);
  if (rc) return rc;
  using KFn = void (*)(const ConvTcParams, const CUtensorMap, const CUtensorMap);
  static const KFn table[4][3] = {
      {k_conv_tc<16, 0>, k_conv_tc<16, 1>, k_conv_tc<16, 2>},
      {k_conv_tc<32, 0>, k_conv_tc<32, 1>, k_conv_tc<32, 2>},
      {k_conv_tc<48, 0>, k_conv_tc<48, 1>, k_conv_tc<48, 2>},
      {k_conv_tc<64, 0>, k_conv_tc<64, 1>, k_conv_tc<64, 2>}};
  if (p.np % 16 || p.np < 16 || p.np > 64 || mode < 0 || mode > 2) return NRX_ERR_UNSUPPORTED;
  const KFn fn = table[p.np / 16 - 1][mode];
  if (set_smem((const void*)fn, SMEM_LIMIT)) return NRX_ERR_CUDA;
  const int total = g.NU * g.tiles;
  dim3 grid(total < num_sms() ? total : num_sms(), n_off);
  fn<<<grid, CONV_THREADS, smem, st>>>(p, m0, m1);
  return cudaPeekAtLastError() == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

static int launch_msg(const Geom& g, const PackLayout& L, const uint8_t* wb, const __nv_bfloat16* state,
                      __nv_bfloat16* agg, cudaStream_t st) {
  MsgTcParams p{};
  p.g = g;
  p.cs = g.Cs;
  p.hp = rup(g.h, 16);
  p.np = rup(g.d, 16);
  p.w0bytes = (uint32_t)(p.cs * p.hp * 2);
  p.w1bytes = (uint32_t)(p.hp * p.np * 2);
  p.abytes = (uint32_t)(p.cs * NRX_TILE_M * 2);
  p.hbytes = (uint32_t)(p.hp * NRX_TILE_M * 2);
  const uint32_t cols = p.hp + g.U * p.np;
  if (cols > 512 || g.U > MSG_MAXU) return NRX_ERR_UNSUPPORTED;
  p.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  p.wbase = wb;
  p.w0 = L.msg.w0;
  p.b0 = L.msg.b0;
  p.w1 = L.msg.w1;
  p.b1 = L.msg.b1;
  p.agg = agg;
  const size_t smem = (size_t)p.w0bytes + p.w1bytes + 2 * p.abytes + p.hbytes + 11 * 8 + 64;
  if (smem > SMEM_LIMIT) return NRX_ERR_UNSUPPORTED;
  CUtensorMap m;
  int rc = make_map(&m, state, g, g.Cs, NRX_TILE_M);
  if (rc) return rc;
  if (set_smem((const void*)k_msg_tc, SMEM_LIMIT)) return NRX_ERR_CUDA;
  const int total = g.N * g.tiles;
  const int per_sm = 512 / p.tmem_cols < 2 ? 1 : 2;
  const int cap = num_sms() * per_sm;
  k_msg_tc<<<total < cap ? total : cap, MLP_THREADS, smem, st>>>(p, m);
  return cudaPeekAtLastError() == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

static int launch_readout(const Geom& g, const PackLayout& L, const uint8_t* wb, const __nv_bfloat16* state,
                          const int32_t* mod_order, float* llr, float2* chest, cudaStream_t st) {
  ReadoutTcParams p{};
  p.g = g;
  p.cs = g.Cs;
  p.h2p = 2 * rup(g.h, 16);
  p.n_io = g.n_io;
  if (p.h2p > 256) return NRX_ERR_UNSUPPORTED;
  p.w0bytes = (uint32_t)(p.cs * p.h2p * 2);
  p.w1bytes = (uint32_t)(p.h2p * 32 * 2);
  p.abytes = (uint32_t)(p.cs * NRX_TILE_M * 2);
  p.hbytes = (uint32_t)(p.h2p * NRX_TILE_M * 2);
  const uint32_t cols = p.h2p + 32;
  p.tmem_cols = cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  p.wbase = wb;
  for (int i = 0; i < g.n_io; ++i) {
    p.w0[i] = L.llr[i].w0;
    p.b0[i] = L.llr[i].b0;
    p.w1[i] = L.llr[i].w1;
    p.b1[i] = L.llr[i].b1;
  }
  p.mod_order = mod_order;
  p.llr = llr;
  p.chest = chest;
  const size_t smem = (size_t)p.w0bytes + p.w1bytes + 2 * p.abytes + p.hbytes + 10 * 8 + 64;
  if (smem > SMEM_LIMIT) return NRX_ERR_UNSUPPORTED;
  CUtensorMap m;
  int rc = make_map(&m, state, g, g.Cs, NRX_TILE_M);
  if (rc) return rc;
  if (set_smem((const void*)k_readout_tc, SMEM_LIMIT)) return NRX_ERR_CUDA;
  const int total = g.NU * g.tiles;
  const int per_sm = 512 / p.tmem_cols < 2 ? 1 : 2;
  const int cap = num_sms() * per_sm;
  dim3 grid(total < cap ? total : cap, g.n_io);
  k_readout_tc<<<grid, MLP_THREADS, smem, st>>>(p, m);
  return cudaPeekAtLastError() == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

}  // namespace tc

#define NRX_TRY_TC(x)            \
  do {                           \
    int _s = (x);                \
    if (_s != NRX_OK) return _s; \
  } while (0)

int launch_forward_tc(const Geom& g, const PackLayout& L, const WsLayout& W, int n_it, const uint8_t* wb,
                      const int32_t* mod_order, uint8_t* ws, float* llr, float2* chest, cudaStream_t st) {
  using namespace tc;
  if (g.d > 64 || g.h > 128) return NRX_ERR_UNSUPPORTED;
  auto* feats = reinterpret_cast<__nv_bfloat16*>(ws + W.feats);
  auto* h = reinterpret_cast<__nv_bfloat16*>(ws + W.h);
  auto* state = reinterpret_cast<__nv_bfloat16*>(ws + W.state);
  auto* agg = reinterpret_cast<__nv_bfloat16*>(ws + W.agg);
  auto* state32 = reinterpret_cast<float*>(ws + W.state32);
  {
    ProfScope ps(KID_INIT0, st);
    NRX_TRY_TC(launch_conv(g, L, L.init0, g.n_io, feats, g.Cf, nullptr, 0, h, g.Ch, nullptr, EPI_RELU, wb,
                           mod_order, st));
  }
  {
    ProfScope ps(KID_INIT1, st);
    NRX_TRY_TC(launch_conv(g, L, L.init1, g.n_io, h, g.Ch, nullptr, 0, state, g.Cs, state32, EPI_STATE_INIT, wb,
                           mod_order, st));
  }
  for (int it = 0; it < n_it; ++it) {
    {
      ProfScope ps(KID_MSG, st);
      NRX_TRY_TC(launch_msg(g, L, wb, state, agg, st));
    }
    {
      ProfScope ps(KID_UPD0, st);
      NRX_TRY_TC(launch_conv(g, L, &L.upd0, 1, state, g.Cs, agg, g.Ca, h, g.Ch, nullptr, EPI_RELU, wb, mod_order,
                             st));
    }
    {
      ProfScope ps(KID_UPD1, st);
      NRX_TRY_TC(launch_conv(g, L, &L.upd1, 1, h, g.Ch, nullptr, 0, state, g.Cs, state32, EPI_RESIDUAL, wb,
                             mod_order, st));
    }
  }
  ProfScope ps(KID_READOUT, st);
  return launch_readout(g, L, wb, state, mod_order, llr, chest, st);
}

int tc_launch_count(int n_it) { return 2 + 3 * n_it + 1; }

}  // namespace nrx
