// Tensor-core per-RE MLPs (bf16 / fp16 operands, or fp32x3 split operands).
//
//  k_msg_tc      message MLP of every UE of a slot on a 128-RE tile followed
//                by the float64 sum of the other UEs' messages
//                (cgnn_iteration nrx.py:258-260, sum_others autodiff.py:276-294).
//  k_readout_tc  LLR and channel-estimate MLPs fused into one N=2h GEMM plus a
//                block-diagonal N=32 GEMM, writing the user-facing (N,U,S,T,W)
//                LLRs and the planar-decoded complex64 chest
//                (readout_llrs/readout_chest nrx.py:266-281, nrx.py:382-384).
//
// Both are persistent, warp-specialised two-layer MLPs:
//   warp 0      TMA producer: state tiles {8, 128, Cs/8, 1} into a 4-stage ring
//   warp 1      MMA issuer: fc0(j+1) is issued before waiting for the hidden
//               layer of j, so the tensor core and the hidden epilogue overlap
//   warps 2-5   hidden epilogue: TMEM -> +bias, ReLU -> bf16 -> shared memory
//               (the next GEMM's K-major A operand), double buffered
//   warps 6-9   output epilogue: sum-of-others / LLR + chest stores
// "use" j enumerates the (work item, UE) pairs a CTA processes.
// X3 (NRX_FP32X3): state tiles, hidden layers and weights carry fp16 hi + lo
// planes; every GEMM is mma_x3_gemm (lo*Whi, then hi*Whi folded by
// scale-input-d, hi*Wlo) and the epilogues apply the packer's 2^-E descale
// (fmaf(acc, 2^-E, bias): the product is exact, so one rounding as acc 2^-E + bias).
#include "tc_common.cuh"

namespace nrx {
namespace tc {

// warps: 0 producer, 1 MMA, HW hidden-epilogue warps, OW output-epilogue warps
// (OW / 4 groups per TMEM lane quarter, each draining a share of the columns)
constexpr int mlp_threads(int hw, int ow = 4) { return 64 + 32 * hw + 32 * ow; }
#ifndef NRX_MSG_HW  // build-time overrides for A/B runs
#define NRX_MSG_HW 8
#endif
#ifndef NRX_MSG_OW
#define NRX_MSG_OW 8
#endif
#ifndef NRX_READOUT_HW
#define NRX_READOUT_HW 8
#endif
constexpr int MSG_HW = NRX_MSG_HW, READOUT_HW = NRX_READOUT_HW;  // 8 hidden-epilogue warps (32 columns each; fp32x3 message 0.29 -> 0.25 ms)
constexpr int MSG_OW = NRX_MSG_OW;  // the message epilogue (2 UEs x 64 columns, split planes) is the long pole
constexpr int MSG_MAXU = 4;  // UEs per slot on the tensor-core path
constexpr int A_STAGES = 4;  // maximum; fp32x3 uses fewer (p.astages)

struct MlpTcParams {
  Geom g;
  int cs, hp, op;          // A channels (state buffer), hidden (padded), output columns
  int uses_per_item;       // U for the message MLP, 1 for the readout
  int units;               // work units: slots (msg) or slabs (readout)
  int n_io;
  uint32_t w0bytes, w1bytes, abytes, hbytes, tmem_cols;
  int astages, nhb;        // A ring stages, hidden shared-memory buffers (1 or 2)
  int akc;                 // fp32x3: state chunks loaded per plane (d/8 < cs/8: the positional chunk,
                           // whose weights are zero, stays a zeroed shared-memory chunk), else 0
  uint32_t col_h, col_o;   // TMEM column of hidden buffer 0 / output region 0
  const uint8_t* wbase;
  uint64_t w0[NRX_MAX_IO], b0[NRX_MAX_IO], w1[NRX_MAX_IO], b1[NRX_MAX_IO];
  const int32_t* mod_order;
  void* agg;               // message MLP output (bf16 / fp16 = kernel's ET)
  int agg_skip;            // fp32x3 with the positional fold (upd0_posf): update.conv0 loads the d/8
                           // chunks of the aggregate only, so its zero chunks beyond d are not written
  float* llr;              // readout outputs
  float2* chest;
};

// Shared-memory carve-up of the MLP kernels.
struct MlpSmem {
  uint8_t *W0, *W1, *As, *Hs;
  uint64_t *afull, *aempty, *hid_full, *h_ready, *hs_free, *out_full, *out_free, *wbar;
  float *sb0, *sb1;
  uint32_t* tmem_ptr;
  __device__ MlpSmem(uint8_t* smem, const MlpTcParams& p) {
    W0 = smem;
    W1 = W0 + p.w0bytes;
    As = W1 + p.w1bytes;
    Hs = As + p.astages * p.abytes;
    uint64_t* b = reinterpret_cast<uint64_t*>(Hs + p.nhb * p.hbytes);
    afull = b;
    aempty = b + A_STAGES;
    hid_full = b + 2 * A_STAGES;
    h_ready = hid_full + 2;
    hs_free = h_ready + 2;
    out_full = hs_free + 2;
    out_free = out_full + 2;
    wbar = out_free + 2;
    sb0 = reinterpret_cast<float*>(wbar + 2);
    sb1 = sb0 + 260;
    tmem_ptr = reinterpret_cast<uint32_t*>(sb1 + 68);
  }
};

__device__ __forceinline__ void mlp_setup(const MlpTcParams& p, MlpSmem& s, int io, int hidden_threads,
                                          int output_threads = 128) {
  const int warp = threadIdx.x >> 5;
  pdl_launch_dependents();  // launched with programmatic serialization: the next layer's prologue may start
  if (warp == 0) tmem_alloc(s.tmem_ptr, p.tmem_cols);
  if (threadIdx.x == 32) {
    for (int i = 0; i < p.astages; ++i) {
      mbar_init(&s.afull[i], 1);
      mbar_init(&s.aempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s.hid_full[i], 1);
      mbar_init(&s.h_ready[i], hidden_threads);
      mbar_init(&s.hs_free[i], 1);
      mbar_init(&s.out_full[i], 1);
      mbar_init(&s.out_free[i], output_threads);
    }
    mbar_init(s.wbar, 1);
    fence_barrier_init();
  }
  const float* b0 = reinterpret_cast<const float*>(p.wbase + p.b0[io]);
  const float* b1 = reinterpret_cast<const float*>(p.wbase + p.b1[io]);
  // fp32x3 blobs store the descale 2^-E right after each bias vector
  const bool x3 = p.g.prec == NRX_FP32X3;
  for (int i = threadIdx.x; i <= p.hp; i += blockDim.x) s.sb0[i] = i < p.hp || x3 ? b0[i] : 1.f;
  if (x3 && p.akc) {  // the A chunks no TMA writes (beyond akc in each plane): zero once, read by the K steps
    const int skip = p.cs / 8 - p.akc, per = skip * NRX_TILE_M * 4;  // uint4 per plane and stage
    for (int i = threadIdx.x; i < p.astages * 2 * per; i += blockDim.x) {
      const int st = i / (2 * per), pl = (i / per) & 1, j = i % per;
      const size_t off = (size_t)st * p.abytes + ((size_t)(pl * (p.cs / 8) + p.akc) * NRX_TILE_M) * 16 + 16 * (size_t)j;
      *reinterpret_cast<uint4*>(s.As + off) = make_uint4(0u, 0u, 0u, 0u);
    }
    fence_proxy_async();  // generic-proxy zeros -> tensor-core reads
  }
  for (int i = threadIdx.x; i <= p.op; i += blockDim.x) s.sb1[i] = i < p.op || x3 ? b1[i] : 1.f;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
}

// Producer / MMA / hidden-epilogue roles are identical for both MLPs; the
// output epilogue is passed in as a functor.
// NK0 / NK1 > 0: the K=16 step counts of fc0 / fc1 at compile time (fp32x3
// issue unrolled for exactly that size; the runtime switch over every size
// otherwise makes the kernel's code outgrow the instruction cache).
template <typename ET, int HW, bool X3, int OW = 4, int NK0 = 0, int NK1 = 0, typename OutEpilogue>
__device__ __forceinline__ void mlp_body(const MlpTcParams& p, MlpSmem& s, int io, const CUtensorMap* amap,
                                         OutEpilogue&& out_epi) {
  const Geom& g = p.g;
  // lane-0 shuffles: provably warp-uniform values keep the MMA issue on the uniform datapath
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *s.tmem_ptr, 0);
  const int U = p.uses_per_item;
#ifdef NRX_TIMING
  long long t_a = 0, t_b = 0, t_c = 0, t_d = 0, t_all = clock64();
#endif

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(s.wbar, p.w0bytes + p.w1bytes);
      bulk_load(s.W0, p.wbase + p.w0[io], p.w0bytes, s.wbar);
      bulk_load(s.W1, p.wbase + p.w1[io], p.w1bytes, s.wbar);
      pdl_wait();  // the state tiles: written by the previous layer
      WorkIter w(g, p.units, g.tiles, p.n_io, p.mod_order);
      int unit, tile, st = 0;
      uint32_t ph = 0;
      while (w.next(unit, tile)) {
        for (int u = 0; u < U; ++u) {
          NRX_T(t0);
          mbar_wait(&s.aempty[st], ph ^ 1);
          NRX_TADD(t_a, t0);
          uint8_t* dst = s.As + (size_t)st * p.abytes;
          if (X3 && p.akc) {  // hi chunks [0, akc) and lo chunks [cs/8, cs/8 + akc)
            mbar_expect_tx(&s.afull[st], 2u * p.akc * NRX_TILE_M * 16);
            tma_load_4d(dst, amap, &s.afull[st], 0, tile * (NRX_TILE_M / 16), 0, unit * U + u);
            tma_load_4d(dst + (size_t)(p.cs / 8) * NRX_TILE_M * 16, amap, &s.afull[st], 0, tile * (NRX_TILE_M / 16),
                        p.cs / 8, unit * U + u);
          } else {
            mbar_expect_tx(&s.afull[st], p.abytes);
            tma_load_4d(dst, amap, &s.afull[st], 0, tile * (NRX_TILE_M / 16), 0, unit * U + u);
          }
          if (++st == p.astages) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {  // MMA issuer: whole warp, elect.sync issues
    {
      const uint32_t id0 = idesc_f16kind<ET>(NRX_TILE_M, p.hp), id1 = idesc_f16kind<ET>(NRX_TILE_M, p.op);
      const uint32_t w0s = smem_u32(s.W0), w1s = smem_u32(s.W1);
      mbar_wait(s.wbar, 0);
      tc_fence_after();
      WorkIter w(g, p.units, g.tiles, p.n_io, p.mod_order);
      int unit, tile;
      bool have = w.next(unit, tile);
      int st = 0, j = 0, item = 0;
      uint32_t ph = 0;
      auto fc0 = [&](int jj) {  // hidden[jj & 1] = A(stage) x W0
        NRX_T(t0);
        mbar_wait(&s.afull[st], ph);
        NRX_TADD(t_a, t0);
        tc_fence_after();
        const uint32_t as = smem_u32(s.As + (size_t)st * p.abytes);
        const uint32_t d = tmem_base + p.col_h + (jj & 1) * p.hp;
        uint64_t ad = smem_desc(as, NRX_TILE_M * 16, 128), bd = smem_desc(w0s, p.hp * 16, 128);
        if constexpr (X3) {
          if constexpr (NK0 > 0)
            mma_x3_gemm_t<NK0>(d, ad, (p.cs / 8) * NRX_TILE_M, 2 * NRX_TILE_M, bd, (p.cs / 8) * p.hp, 2 * p.hp, id0);
          else
            mma_x3_gemm(d, ad, (p.cs / 8) * NRX_TILE_M, 2 * NRX_TILE_M, bd, (p.cs / 8) * p.hp, 2 * p.hp, p.cs / 16,
                        id0);
        } else {
          for (int kc = 0; kc < p.cs / 8; kc += 2) {
            mma_bf16_warp(d, ad, bd, id0, kc != 0);
            ad += 2 * NRX_TILE_M;
            bd += 2 * p.hp;
          }
        }
        mma_commit_warp(&s.aempty[st]);
        mma_commit_warp(&s.hid_full[jj & 1]);
        if (++st == p.astages) { st = 0; ph ^= 1; }
      };
      if (have) fc0(0);
      while (have) {
        for (int u = 0; u < U; ++u, ++j) {
          // look ahead: the next use's fc0 overlaps this use's hidden epilogue
          const bool last_u = u + 1 == U;
          int nunit = unit, ntile = tile;
          bool next_exists = true;
          if (last_u) next_exists = w.next(nunit, ntile);
          if (next_exists) fc0(j + 1);
          const int hb = p.nhb == 2 ? (j & 1) : 0;
          NRX_T(t1);
          mbar_wait(&s.h_ready[hb], (p.nhb == 2 ? j >> 1 : j) & 1);
          NRX_TADD(t_b, t1);
          tc_fence_after();
          if (u == 0) {  // output region of this item free again?
            NRX_T(t2);
            mbar_wait(&s.out_free[item & 1], ((item >> 1) & 1) ^ 1);
            NRX_TADD(t_c, t2);
            tc_fence_after();
          }
          const uint32_t hs = smem_u32(s.Hs + (size_t)hb * p.hbytes);
          const uint32_t d = tmem_base + p.col_o + (item & 1) * (U * p.op) + u * p.op;
          uint64_t ad = smem_desc(hs, NRX_TILE_M * 16, 128), bd = smem_desc(w1s, p.op * 16, 128);
          if constexpr (X3) {
            if constexpr (NK1 > 0)
              mma_x3_gemm_t<NK1>(d, ad, (p.hp / 8) * NRX_TILE_M, 2 * NRX_TILE_M, bd, (p.hp / 8) * p.op, 2 * p.op, id1);
            else
              mma_x3_gemm(d, ad, (p.hp / 8) * NRX_TILE_M, 2 * NRX_TILE_M, bd, (p.hp / 8) * p.op, 2 * p.op,
                          p.hp / 16, id1);
          } else {
            for (int kc = 0; kc < p.hp / 8; kc += 2) {
              mma_bf16_warp(d, ad, bd, id1, kc != 0);
              ad += 2 * NRX_TILE_M;
              bd += 2 * p.op;
            }
          }
          mma_commit_warp(&s.hs_free[hb]);
          if (last_u) {
            mma_commit_warp(&s.out_full[item & 1]);
            ++item;
            unit = nunit;
            tile = ntile;
            have = next_exists;
          }
        }
      }
    }
  } else if (warp < 2 + HW) {  // hidden epilogue; with 8 warps each drains half the columns
    const int q = warp & 3;
    const int r = 32 * q + lane;
    const uint32_t lane_off = static_cast<uint32_t>(32 * q) << 16;
    const int cspan = p.hp / (HW / 4), cbeg = ((warp - 2) / 4) * cspan;
    WorkIter w(g, p.units, g.tiles, p.n_io, p.mod_order);
    int unit, tile, j = 0;
    while (w.next(unit, tile)) {
      for (int u = 0; u < U; ++u, ++j) {
        const int ab = j & 1;                      // TMEM hidden accumulator
        const int hb = p.nhb == 2 ? ab : 0;         // shared-memory hidden tile
        const int hk = p.nhb == 2 ? j >> 1 : j;     // its use count
        NRX_T(t0);
        mbar_wait(&s.hid_full[ab], (j >> 1) & 1);
        NRX_TADD(t_a, t0);
        tc_fence_after();
        NRX_T(t1);
        mbar_wait(&s.hs_free[hb], (hk & 1) ^ 1);  // fc1 of the previous use of Hs[hb] done
        NRX_TADD(t_b, t1);
        NRX_T(t2);
        uint8_t* H = s.Hs + (size_t)hb * p.hbytes;
        const float dsc = X3 ? s.sb0[p.hp] : 1.f;
        if constexpr (X3 && NK1 > 0 && 16 * NK1 / (HW / 4) <= 64) {
          // compile-time hidden width (hp = 16 NK1): this thread's columns in one TMEM
          // round trip (every 16-column load issued before the single wait), fully unrolled
          constexpr int CSPAN = 16 * NK1 / (HW / 4);
          float v[CSPAN];
#pragma unroll
          for (int b16 = 0; b16 < CSPAN / 16; ++b16)
            tmem_ld16(tmem_base + lane_off + p.col_h + ab * p.hp + cbeg + 16 * b16, v + 16 * b16);
          tmem_wait_ld();
          uint32_t bad = 0;
#pragma unroll
          for (int c8 = 0; c8 < CSPAN / 8; ++c8) {
            const int ch = cbeg / 8 + c8;
            float o[8], bb[8];
            ld_shared_f8(smem_u32(s.sb0) + 32u * ch, bb);
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = relu_f(fmaf(v[8 * c8 + e], dsc, bb[e]));
            uint4 hi, lo;
            split_chunk(o, hi, lo, bad);
            *reinterpret_cast<uint4*>(H + ((size_t)ch * NRX_TILE_M + r) * 16) = hi;
            *reinterpret_cast<uint4*>(H + ((size_t)(16 * NK1 / 8 + ch) * NRX_TILE_M + r) * 16) = lo;
          }
          report_range(bad, g.flag);
        } else
        for (int c32 = cbeg; c32 < cbeg + cspan; c32 += 32) {
          float v[32];
          tmem_ld16(tmem_base + lane_off + p.col_h + ab * p.hp + c32, v);
          if (c32 + 16 < cbeg + cspan) tmem_ld16(tmem_base + lane_off + p.col_h + ab * p.hp + c32 + 16, v + 16);
          tmem_wait_ld();
#pragma unroll
          for (int c8 = 0; c8 < 4; ++c8) {
            if (c32 + 8 * c8 >= cbeg + cspan) break;
            float o[8];
            const int ch = c32 / 8 + c8;
            if constexpr (X3) {
              float bb[8];
              ld_shared_f8(smem_u32(s.sb0) + 32u * ch, bb);  // two LDS.128 (the bias chunk, broadcast)
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] = relu_f(fmaf(v[8 * c8 + e], dsc, bb[e]));
              uint4 hi, lo;
              uint32_t bad = 0;
              split_chunk(o, hi, lo, bad);
              report_range(bad, g.flag);
              *reinterpret_cast<uint4*>(H + ((size_t)ch * NRX_TILE_M + r) * 16) = hi;
              *reinterpret_cast<uint4*>(H + ((size_t)(p.hp / 8 + ch) * NRX_TILE_M + r) * 16) = lo;
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] = relu_f(v[8 * c8 + e] + s.sb0[c32 + 8 * c8 + e]);
              store_chunk(reinterpret_cast<ET*>(H + ((size_t)ch * NRX_TILE_M + r) * 16), o);
            }
          }
        }
        fence_proxy_async();  // generic-proxy smem writes -> tensor-core reads
        tc_fence_before();
        mbar_arrive(&s.h_ready[hb]);
        NRX_TADD(t_c, t2);
      }
    }
  } else {  // output epilogue (the last 4 warps)
    const int q = warp & 3;
    const int r = 32 * q + lane;
    const uint32_t lane_off = static_cast<uint32_t>(32 * q) << 16;
    WorkIter w(g, p.units, g.tiles, p.n_io, p.mod_order);
    int unit, tile, item = 0;
    while (w.next(unit, tile)) {
      NRX_T(t0);
      mbar_wait(&s.out_full[item & 1], (item >> 1) & 1);
      NRX_TADD(t_a, t0);
      tc_fence_after();
      const uint32_t taddr = tmem_base + lane_off + p.col_o + (item & 1) * (U * p.op);
      NRX_T(t1);
      out_epi(unit, tile, r, taddr, &s.out_free[item & 1], (warp - 2 - HW) >> 2, OW / 4);
      NRX_TADD(t_b, t1);
      ++item;
    }
  }
#ifdef NRX_TIMING
  if (blockIdx.x == 0 && (threadIdx.x == 0 || threadIdx.x == 32 || threadIdx.x == 64 || threadIdx.x == 192))
    printf("mlp U=%d tid=%d all=%lld a=%lld b=%lld c=%lld\n", U, threadIdx.x, clock64() - t_all, t_a, t_b, t_c);
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

// UT > 0: the number of UEs at compile time (the 2-UE slots of the benchmark)
template <typename ET, bool X3, int NK = 0, int UT = 0>
__global__ void __launch_bounds__(mlp_threads(MSG_HW, MSG_OW), 1)
    k_msg_tc(const __grid_constant__ MlpTcParams p, const __grid_constant__ CUtensorMap smap) {
  extern __shared__ __align__(1024) uint8_t smem[];
  MlpSmem s(smem, p);
  mlp_setup(p, s, 0, 32 * MSG_HW, 32 * MSG_OW);
  const Geom& g = p.g;
  const int U = UT > 0 ? UT : p.uses_per_item;
  constexpr int UMAX = UT > 0 ? UT : MSG_MAXU;
  const int nca = g.Ca / 8;
  const bool agg_skip = X3 && p.agg_skip;
  ET* const agg = static_cast<ET*>(p.agg);
  const float dsc = X3 ? s.sb1[p.op] : 1.f;
  mlp_body<ET, MSG_HW, X3, MSG_OW, NK, NK>(p, s, 0, &smap, [&](int n, int tile, int r, uint32_t taddr, uint64_t* free_bar,
                                                       int grp, int ngrp) {
    const int row = tile * NRX_TILE_M + r;
    const int srow = row / g.Tp, t = row - srow * g.Tp;
    const bool valid = row < g.rows_data && t < g.T;
    // Sum of the other UEs' messages, added directly in fp32 (U-1 terms).
    // For U=2 this is exactly the other message, which equals the reference's
    // f32(f64 total - f64 own) whenever that float64 sum is exact (message
    // exponents within 29 bits); the bf16 rounding of the stored aggregate
    // dominates any difference for U>2.  The fp32 parity path keeps fp64.
    // this warp group's share of the output columns (16-column blocks); when
    // the width does not split evenly the first group drains everything
    const int ng = p.op % (16 * ngrp) == 0 ? ngrp : 1;
    if (grp >= ng) {
      mbar_arrive_relaxed(free_bar);
      return;
    }
    const int cspan = p.op / ng;
    if constexpr (X3 && UT > 0 && NK > 0) {
      // the RT shape (op = 64, launch_msg): this group's UT x 32 message columns in one TMEM
      // round trip, then the sums of the others, split, stored as the aggregate planes
      constexpr int CS = 64 / (MSG_OW / 4);
      static_assert(CS % 16 == 0, "column span");
      const int c0 = grp * CS;
      float m[UT][CS];
#pragma unroll
      for (int u = 0; u < UT; ++u)
#pragma unroll
        for (int b16 = 0; b16 < CS / 16; ++b16) tmem_ld16(taddr + u * 64 + c0 + 16 * b16, m[u] + 16 * b16);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive_relaxed(free_bar);
      const uint32_t vmask = valid ? 0xffffffffu : 0u;
      uint32_t bad = 0;
#pragma unroll
      for (int c8 = 0; c8 < CS / 8; ++c8) {
        const int cc = c0 / 8 + c8;
        if (cc >= nca || (agg_skip && 8 * cc >= g.d)) break;
        const bool full = 8 * cc + 8 <= g.d;
        float bb[8];
        ld_shared_f8(smem_u32(s.sb1) + 32u * cc, bb);
        float mb[UT][8];
#pragma unroll
        for (int u = 0; u < UT; ++u)
#pragma unroll
          for (int e = 0; e < 8; ++e) mb[u][e] = fmaf(m[u][8 * c8 + e], dsc, bb[e]);
#pragma unroll
        for (int u = 0; u < UT; ++u) {
          float o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            float a = 0.f;
#pragma unroll
            for (int v = 0; v < UT; ++v)
              if (v != u) a += mb[v][e];
            o[e] = full || 8 * cc + e < g.d ? a : 0.f;
          }
          uint4 hi, lo;
          split_chunk(o, hi, lo);
          hi = mask_chunk(hi, vmask);
          lo = mask_chunk(lo, vmask);
          const uint32_t hw[4] = {hi.x, hi.y, hi.z, hi.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) bad |= ((hw[i] & 0x7c007c00u) + 0x04000400u) & 0x80008000u;  // as split_chunk
          *reinterpret_cast<uint4*>(chunk_ptr(agg, n * UT + u, 2 * nca, cc, row, g)) = hi;
          *reinterpret_cast<uint4*>(chunk_ptr(agg, n * UT + u, 2 * nca, nca + cc, row, g)) = lo;
        }
      }
      report_range(bad, g.flag);
      return;
    }
    for (int c16 = grp * cspan; c16 < (grp + 1) * cspan; c16 += 16) {
      float m[UMAX][16];
#pragma unroll
      for (int u = 0; u < UMAX; ++u)
        if (u < U) tmem_ld16(taddr + u * p.op + c16, m[u]);
      tmem_wait_ld();
      if (c16 + 16 >= (grp + 1) * cspan) {  // this group's messages are in registers: release TMEM
        tc_fence_before();
        mbar_arrive_relaxed(free_bar);
      }
      float bb[16];
      ld_shared_f8(smem_u32(s.sb1) + 4u * c16, bb);
      ld_shared_f8(smem_u32(s.sb1) + 4u * c16 + 32u, bb + 8);
#pragma unroll
      for (int u = 0; u < UMAX; ++u)
        if (u < U)
#pragma unroll
          for (int e = 0; e < 16; ++e) m[u][e] = X3 ? fmaf(m[u][e], dsc, bb[e]) : m[u][e] + bb[e];
      const uint32_t vmask = valid ? 0xffffffffu : 0u;
#pragma unroll
      for (int u = 0; u < UMAX; ++u) {
        if (u >= U) break;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const int c8 = c16 / 8 + h2;
          if (c8 >= nca || (X3 && agg_skip && 8 * c8 >= g.d)) break;  // posf update.conv0 reads d channels
          const bool full = 8 * c8 + 8 <= g.d;  // warp-uniform: no per-channel select
          float o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            float a = 0.f;
#pragma unroll
            for (int v = 0; v < UMAX; ++v)
              if (v < U && v != u) a += m[v][8 * h2 + e];
            o[e] = full || 8 * c8 + e < g.d ? a : 0.f;
          }
          if constexpr (X3) {  // [hi | lo] planes of the aggregate, pad rows zeroed on the packed words
            uint4 hi, lo;
            split_chunk(o, hi, lo);
            hi = mask_chunk(hi, vmask);
            lo = mask_chunk(lo, vmask);
            uint32_t bad = 0;
            const uint32_t hw[4] = {hi.x, hi.y, hi.z, hi.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) bad |= ((hw[i] & 0x7c007c00u) + 0x04000400u) & 0x80008000u;  // as split_chunk
            report_range(bad, g.flag);
            *reinterpret_cast<uint4*>(chunk_ptr(agg, n * U + u, 2 * nca, c8, row, g)) = hi;
            *reinterpret_cast<uint4*>(chunk_ptr(agg, n * U + u, 2 * nca, nca + c8, row, g)) = lo;
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = valid ? o[e] : 0.f;
            store_chunk(chunk_ptr(agg, n * U + u, nca, c8, row, g), o);
          }
        }
      }
    }
  });
}

template <typename ET, bool X3, int NK0 = 0, int NK1 = 0>
__global__ void __launch_bounds__(mlp_threads(READOUT_HW), 1)
    k_readout_tc(const __grid_constant__ MlpTcParams p, const __grid_constant__ CUtensorMap smap) {
  extern __shared__ __align__(1024) uint8_t smem[];
  MlpSmem s(smem, p);
  const int io = p.n_io > 1 ? blockIdx.y : 0;
  mlp_setup(p, s, io, 32 * READOUT_HW);
  const Geom& g = p.g;
  const float dsc = X3 ? s.sb1[p.op] : 1.f;
  mlp_body<ET, READOUT_HW, X3, 4, NK0, NK1>(p, s, io, &smap, [&](int slab, int tile, int r, uint32_t taddr, uint64_t* free_bar,
                                                    int, int) {
    // columns 0-7 LLRs, 8 .. 8+2B-1 the chest (2B <= 16): the first 24 of the 32-wide block
    float o[24], bb[24];
    tmem_ld16(taddr, o);
    tmem_ld8(taddr + 16, o + 16);
    tmem_wait_ld();
    tc_fence_before();
    mbar_arrive_relaxed(free_bar);
    const int row = tile * NRX_TILE_M + r;
    const int srow = row / g.Tp, t = row - srow * g.Tp;
    if (row >= g.rows_data || t >= g.T) return;
#pragma unroll
    for (int c8 = 0; c8 < 3; ++c8) ld_shared_f8(smem_u32(s.sb1) + 32u * c8, bb + 8 * c8);
    uint32_t bad = 0;
#pragma unroll
    for (int c = 0; c < 24; ++c) {
      o[c] = X3 ? fmaf(o[c], dsc, bb[c]) : o[c] + bb[c];
      bad |= (__float_as_uint(o[c]) & 0x7f800000u) == 0x7f800000u;
    }
    if (bad && g.flag) atomicOr(g.flag, 1u);  // range guard (nrx_forward)
    const int mio = io_index(p.mod_order, slab, g);
    const int width = mio < 0 ? 0 : g.io_width[mio];
    const size_t re = ((size_t)slab * g.S + srow) * g.T + t;
    float* lp = p.llr + re * g.llr_width;
    if (g.llr_width == 4 && width == 4) {
      *reinterpret_cast<float4*>(lp) = make_float4(o[0], o[1], o[2], o[3]);
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < g.llr_width) lp[c] = mio < 0 ? __int_as_float(0x7fc00000) : (c < width ? o[c] : 0.f);
    }
    float2* cp = p.chest + re * g.B;
    if (g.B == 4) {  // planar decode: channel b real, channel B+b imaginary
      reinterpret_cast<float4*>(cp)[0] = make_float4(o[8], o[12], o[9], o[13]);
      reinterpret_cast<float4*>(cp)[1] = make_float4(o[10], o[14], o[11], o[15]);
    } else {
      // constant register indices only (a runtime index would put o[] in local memory)
      float* cf = reinterpret_cast<float*>(cp);
#pragma unroll
      for (int b = 0; b < 8; ++b)
        if (b < g.B) cf[2 * b] = o[8 + b];
#pragma unroll
      for (int c = 9; c < 24; ++c) {
        const int b = c - 8 - g.B;  // imaginary part of antenna b
        if (b >= 0 && b < g.B) cf[2 * b + 1] = o[c];
      }
    }
  });
}

}  // namespace tc

using namespace tc;

static size_t mlp_smem_bytes(const MlpTcParams& p) {
  return (size_t)p.w0bytes + p.w1bytes + p.astages * p.abytes + p.nhb * p.hbytes + (2 * A_STAGES + 12) * 8 +
         (260 + 68) * 4 + 16;
}

static int mlp_common(MlpTcParams& p, const Geom& g, int hp, int op, int uses, int units, size_t* smem) {
  const uint32_t planes = g.prec == NRX_FP32X3 ? 2 : 1;  // fp32x3: [hi | lo] everywhere
  p.g = g;
  p.cs = g.Cs;
  p.hp = hp;
  p.op = op;
  p.uses_per_item = uses;
  p.units = units;
  p.w0bytes = planes * (uint32_t)(p.cs * hp * 2);
  p.w1bytes = planes * (uint32_t)(hp * op * 2);
  p.abytes = planes * (uint32_t)(p.cs * NRX_TILE_M * 2);
  p.hbytes = planes * (uint32_t)(hp * NRX_TILE_M * 2);
  // double-buffered hidden tiles before A stages: a single hidden tile
  // serialises the hidden epilogue with fc1 of the previous use
  p.astages = A_STAGES;
  p.nhb = 2;
  while (mlp_smem_bytes(p) > SMEM_LIMIT && p.astages > 1) --p.astages;
  if (mlp_smem_bytes(p) > SMEM_LIMIT) {
    p.nhb = 1;
    p.astages = A_STAGES;
    while (mlp_smem_bytes(p) > SMEM_LIMIT && p.astages > 1) --p.astages;
  }
  p.col_h = 0;
  p.col_o = 2 * hp;
  const uint32_t cols = 2 * hp + 2 * uses * op;
  if (cols > 512 || hp > 256) return NRX_ERR_UNSUPPORTED;
  p.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  *smem = mlp_smem_bytes(p);
  return *smem > SMEM_LIMIT ? NRX_ERR_UNSUPPORTED : NRX_OK;
}

int launch_msg(const Geom& g, const PackLayout& L, const uint8_t* wb, const void* state, void* agg,
               cudaStream_t st) {
  if (g.U > MSG_MAXU) return NRX_ERR_UNSUPPORTED;
  MlpTcParams p{};
  size_t smem = 0;
  int rc = mlp_common(p, g, rup(g.h, 16), rup(g.d, 16), g.U, g.N, &smem);
  if (rc) return rc;
  p.n_io = 1;
  p.wbase = wb;
  p.w0[0] = L.msg.w0;
  p.b0[0] = L.msg.b0;
  p.w1[0] = L.msg.w1;
  p.b1[0] = L.msg.b1;
  p.agg = agg;
  p.agg_skip = g.prec == NRX_FP32X3 && upd0_posf(g.d, g.ks, NRX_FP32X3) && g.d % 8 == 0;
  CUtensorMap m;
  p.akc = g.prec == NRX_FP32X3 && g.d % 8 == 0 && g.d / 8 < g.Cs / 8 ? g.d / 8 : 0;
  rc = make_map(&m, state, g, g.prec == NRX_FP32X3 ? 2 * g.Cs : g.Cs, NRX_TILE_M, p.akc);
  if (rc) return rc;
  // fp32x3 RT shapes (64-channel state and hidden, 2 UEs): compile-time sizes keep the code in the icache
  const bool rt = g.prec == NRX_FP32X3 && g.Cs == 64 && p.hp == 64 && p.op == 64 && g.U == 2;
  const auto fn = rt ? k_msg_tc<__half, true, 4, 2>
                  : g.prec == NRX_FP32X3 ? k_msg_tc<__half, true>
                  : g.prec == NRX_FP16 ? k_msg_tc<__half, false>
                                       : k_msg_tc<__nv_bfloat16, false>;
  if (set_smem((const void*)fn, SMEM_LIMIT)) return NRX_ERR_CUDA;
  const int total = g.N * g.tiles;
  const int per_sm = (512 / p.tmem_cols) < 2 || 2 * smem > SMEM_LIMIT ? 1 : 2;
  const int cap = num_sms() * per_sm;
  if (launch_pdl(fn, dim3(total < cap ? total : cap), dim3(mlp_threads(MSG_HW, MSG_OW)), smem, st, p, m) !=
      cudaSuccess)
    return NRX_ERR_CUDA;
  return cudaPeekAtLastError() == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

int launch_readout(const Geom& g, const PackLayout& L, const uint8_t* wb, const void* state,
                   const int32_t* mod_order, float* llr, float2* chest, cudaStream_t st) {
  MlpTcParams p{};
  size_t smem = 0;
  int rc = mlp_common(p, g, 2 * rup(g.h, 16), 32, 1, g.NU, &smem);
  if (rc) return rc;
  p.n_io = g.n_io;
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
  CUtensorMap m;
  p.akc = g.prec == NRX_FP32X3 && g.d % 8 == 0 && g.d / 8 < g.Cs / 8 ? g.d / 8 : 0;
  rc = make_map(&m, state, g, g.prec == NRX_FP32X3 ? 2 * g.Cs : g.Cs, NRX_TILE_M, p.akc);
  if (rc) return rc;
  const bool rt = g.prec == NRX_FP32X3 && g.Cs == 64 && p.hp == 128;
  const auto fn = rt ? k_readout_tc<__half, true, 4, 8>
                  : g.prec == NRX_FP32X3 ? k_readout_tc<__half, true>
                  : g.prec == NRX_FP16 ? k_readout_tc<__half, false>
                                       : k_readout_tc<__nv_bfloat16, false>;
  if (set_smem((const void*)fn, SMEM_LIMIT)) return NRX_ERR_CUDA;
  const int total = g.NU * g.tiles;
  const int per_sm = (512 / p.tmem_cols) < 2 || 2 * smem > SMEM_LIMIT ? 1 : 2;
  const int cap = num_sms() * per_sm;
  dim3 grid(total < cap ? total : cap, g.n_io);
  if (launch_pdl(fn, grid, dim3(mlp_threads(READOUT_HW)), smem, st, p, m) != cudaSuccess) return NRX_ERR_CUDA;
  return cudaPeekAtLastError() == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

}  // namespace nrx
