// fp32-grade tensor-core convolution (NRX_FP32X3) on CTA pairs.
//
// The reference computes every convolution as an fp32 sgemm over im2col
// (autodiff.py:315-350).  This path keeps that accuracy on the fp16 tensor
// cores by splitting both operands:
//   activation  a = hi + lo' 2^-11  (fp16 planes, split_chunk)
//   weight      W 2^E = Whi + Wlo   (fp16 halves, host packer)
//   a W 2^E = hi Whi + hi Wlo + (lo' Whi + lo' Wlo) 2^-11      (all four terms)
// Each MMA multiplies one activation plane by the concatenated B operand
// [Whi | Wlo] (N = 2 np): one MMA yields [a Whi | a Wlo] in two adjacent
// TMEM column blocks.  Per tile the MMA warp first issues the lo' MMAs (sums
// at scale 2^11), then the hi MMAs; the first hi MMA into a block uses
// scale-input-d = 11 (D = A B + D 2^-11), which folds the lo' sums in with
// the exact power-of-two weight.  The epilogue adds the blocks in fp32,
// multiplies by 2^-E (exact) and adds the bias as the reference does.  The
// operand representation error is <= 2^-23 relative (fp32: 2^-24).
//
// Accumulation: the tensor core's fp32 accumulate truncates, ~0.2 ulp of D
// towards zero per MMA (scripts/acc_probe.cu: -14.7 ulp mean after 72 MMAs,
// where round-to-nearest stays at ~0).  Only MMAs at the full magnitude of D
// matter (the lo' sums are scaled by 2^-11 afterwards, the Wlo block is 2^-11
// smaller), so the hi MMAs are spread over P = 2 partial accumulators by tap
// row (rows 0, 2 / row 1 for 3x3 kernels), added by the epilogue in fp32
// round-to-nearest.  C2 LLRs stay within 2.1e-6 of the float64 oracle
// (SIMT fp32: 6.5e-7; gate 1e-5).
//
// Weights of one plane for every output channel (147 KB for
// iteration.update.conv0) use most of an SM's shared memory, so every layer
// runs on a CTA pair (cluster of 2, tcgen05.mma.cta_group::2, M = 256): the
// pair MMA reads B as rank 0's rows followed by rank 1's, so rank 0 keeps Whi
// and rank 1 Wlo resident; each CTA loads its own 128-row tile + halo of the
// activations and receives the accumulator of its own rows in its own TMEM.
// Per SM an MMA (128 x 128 x 16) reads 4 KB of A and 2 KB of B and is
// math-bound at 64 cycles: 2 MMAs = 128 cycles per tap and K=16 step.
//
// Roles (both CTAs): warp 0 lane 0 TMA producer (its tile, signalling the
// leader's full barrier through the .cta_group::2 TMA form), warp 1 the MMA
// issuer in the leader / the weights-resident relay in the peer, 4 np/NC
// epilogue warps per CTA draining their own TMEM.  Pipeline stages are
// (tile, plane, source): lo planes of every source first, then hi planes.
// Layout of the activations: chunk-planar as everywhere (nrx_internal.h),
// buffers with 2C channels = [C hi | C lo].
#include "nrx_profile.h"
#include "tc_common.cuh"

namespace nrx {
namespace tc {

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_rank(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Arrive without release semantics: the epilogue's "accumulator drained"
// signal orders only its completed tcgen05.ld reads (tcgen05.wait::ld), not
// its global stores; a .release.cluster arrive compiles to MEMBAR.ALL.GPU and
// would wait for every store of the previous tile still in flight.
__device__ __forceinline__ void arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// pair MMA D[tmem] (+)= A[smem, both CTAs] * B[smem, both CTAs]^T (fp16, fp32 accumulate)
__device__ __forceinline__ void mma2_warp(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// D = A B + D 2^-11: folds the lo*Whi partial sums (scale 2^11) into the hi terms
__device__ __forceinline__ void mma2_warp_fold(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 1, 11;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc)
      : "memory");
}
// commit to the barrier at the same offset in both CTAs of the pair
__device__ __forceinline__ void commit2_warp(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          bar),
      "h"((uint16_t)3)
      : "memory");
}
// TMA into this CTA's shared memory, completing on the leader CTA's barrier
__device__ __forceinline__ void tma_load_4d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                 int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// Work of a CTA pair: flat tiles f over the units (slabs) whose IO set is this
// grid row's (all slabs unless var_io); pair p takes f = 2k, 2k+1 for
// k = p, p + npairs, ...; rank 0 the even tile, rank 1 the odd one.  When the
// tile count is odd the last pair's rank 1 recomputes rank 0's tile with its
// stores suppressed (real = false), so both CTAs always step together.
struct PairIter {
  int u, tl, units, tps, n_io, io, rank, pair, npairs;
  bool first;
  const int32_t* mod;
  const Geom* g;
  __device__ PairIter(const Geom& geo, int n_units, int tiles_per_unit, int n_io_sets, const int32_t* mods,
                      int r)
      : u(0), tl(0), units(n_units), tps(tiles_per_unit), n_io(n_io_sets), io(blockIdx.y), rank(r),
        pair(blockIdx.x >> 1), npairs(gridDim.x >> 1), first(true), mod(mods), g(&geo) {}
  __device__ bool match(int v) const { return n_io <= 1 || io_index(mod, v, *g) == io; }
  __device__ int next_match(int v) const {
    while (v < units && !match(v)) ++v;
    return v;
  }
  __device__ void advance(int n) {
    tl += n;
    while (tl >= tps && u < units) {
      tl -= tps;
      u = next_match(u + 1);
    }
  }
  __device__ bool next(int& slab, int& tile, bool& real) {
    if (first) {
      first = false;
      u = next_match(0);
      tl = 0;
      advance(2 * pair);
    } else {
      advance(2 * npairs);
    }
    if (u >= units) return false;
    slab = u;
    tile = tl;
    real = true;
    if (rank == 1) {
      int u2 = u, t2 = tl + 1;
      if (t2 >= tps) {
        t2 = 0;
        u2 = next_match(u + 1);
      }
      if (u2 >= units) {
        real = false;
      } else {
        slab = u2;
        tile = t2;
      }
    }
    return true;
  }
};

struct ConvX3Params {
  Geom g;
  int c0, c1;        // channels per plane of source 0 / 1 (buffers hold 2x: [hi | lo])
  int np;            // pair MMA N = rup(d, 32); each CTA holds np/2 B rows
  int nacc;          // partial accumulators per tile (hi*Whi MMAs by tap row)
  int cdst, stages, n_io, src1_xor, hup;
  int posf, kc;      // positional channels folded out (upd0_posf): both sources' kc chunks share one stage
  int ptab;          // posf: per-(comb residue, symbol) table of the positional contribution in shared memory
  int hskip;         // RELU layer writing h for a tap-pair conv1: its zero chunks beyond d are never read
  uint32_t wbytes;   // one rank's weight block: [hi | lo][taps*ktap/8][np/2][8] fp16
  uint32_t abytes, tmem_cols, rbox;
  const uint8_t* wbase;
  uint64_t w_off[NRX_MAX_IO], b_off[NRX_MAX_IO];
  const int32_t* mod_order;
  __half* dst;
};

struct ConvX3Smem {
  uint32_t w, a, bars, tmem_ptr, sbias, dt, posw, ptab, total;
};
__host__ __device__ inline ConvX3Smem conv_x3_smem(const ConvX3Params& p) {
  ConvX3Smem s;
  uint32_t off = 0;
  s.w = off;
  off = (p.wbytes + 1023u) & ~1023u;
  s.a = off;
  off += p.stages * p.abytes;
  s.bars = off;
  off += 32 * 8;
  s.tmem_ptr = off;
  off += 16;
  s.sbias = off;
  off += 80 * 4;
  s.dt = off;
  off += 32 * 4;
  s.posw = off;
  off += p.posf ? 18 * p.np * 4 : 0;
  s.ptab = off;
  off += p.posf && p.ptab ? p.g.comb * p.g.T * (p.np + 4) * 4 : 0;  // rows padded: conflict-free by symbol
  s.total = off;
  return s;
}

// Epilogue columns per thread: 32 (2 + 4 np/32 warps, so each SM sub-partition
// holds <= 3 warps and the fully unrolled MMA issue gets up to 168 registers)
// for update.conv0; the layers whose epilogue is the bottleneck run twice the
// warps (16 columns each).
// Layers with at most two K=16 steps per tap (state_init.conv0: 19 -> 32
// feature channels) issue few MMAs per tile, so their epilogue is the long
// pole: 16 columns per thread (twice the warps) there too.
__host__ __device__ constexpr int x3_epi_cols(int mode, bool small_k = false) {
  // the state-writing layers (state init, residual update) drain with twice the
  // warps: state_init.conv1 0.50 -> 0.44 ms once the epilogue's full-chunk fast
  // path made the 18-warp (96-register) configuration cheap enough
  return small_k || mode != EPI_RELU ? 16 : 32;
}
// NC accumulator columns of this thread's lane (x16 loads, x8 for a remainder)
template <int NC>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float* v) {
#pragma unroll
  for (int c = 0; c + 16 <= NC; c += 16) tmem_ld16(taddr + c, v + c);
  if constexpr (NC % 16 != 0) tmem_ld8(taddr + NC / 16 * 16, v + NC / 16 * 16);
}
__host__ __device__ constexpr bool x3_small_k(int ks, int nk0, int nk1) { return ks > 0 && nk0 + nk1 <= 2; }

// PREC = NRX_FP32X3: the split-operand kernel described above.  PREC =
// NRX_FP16 / NRX_BF16: the same CTA-pair pipeline for one half-precision plane
// (the bf16 / fp16 modes' ReLU convolutions without a tail: state_init.conv0
// and iteration.update.conv0): each CTA holds the weights of np/2 output
// channels, an N = np pair MMA reads 4 KB of A and 1 KB of B per SM (5 KB
// instead of 6 KB single-CTA: 40 instead of 48 cycles per K=16 step).
//
// POSF (iteration.update.conv0, upd0_posf): the A operand is [state (d) |
// agg (d)] without the two positional channels -- both sources land in one
// stage (kc chunks each, contiguous, so a K=16 step may straddle them) and
// the K loop runs NK0 = d/8 steps; the epilogue adds the positional
// contribution sum_{tap, ch} W_pos[ch][tap][c] pos_ch(s + a - 1, t + b - 1)
// (zero outside the grid, as the reference's zero padding) in fp32.  pos_dt
// depends on t only and pos_df on the distance to the UE's comb, so away from
// the band edges (o < s < S - comb - 1, o the UE's comb offset) the sum is a
// function of ((s - o) mod comb, t): each CTA tabulates it once (comb x T x np
// fp32, before griddepcontrol.wait) and the epilogue adds one table row; edge
// rows evaluate the 18 terms.
//
// TPC (fp32x3 3x3 layers over C = TPC data chunks, tp2_chunks): the tap-pair
// K order of nrx_internal.h -- 4 C + (C+1)/2 instead of 9 (C+1)/2 MMA steps per
// plane (C = 7: 32 instead of 36; C = 3: 14 instead of 18), C loaded chunks.
template <int NP, int MODE, int KS = 0, int NK0 = 0, int NK1 = 0, int PREC = NRX_FP32X3, bool POSF = false,
          int TPC = 0>
__global__ void __launch_bounds__(64 + 128 * ((NP + x3_epi_cols(MODE, x3_small_k(KS, NK0, NK1)) - 1) /
                                              x3_epi_cols(MODE, x3_small_k(KS, NK0, NK1))),
                                  1)
    k_conv_x3(const __grid_constant__ ConvX3Params p, const __grid_constant__ CUtensorMap map0,
              const __grid_constant__ CUtensorMap map1) {
  constexpr bool SPLIT = PREC == NRX_FP32X3;
  using ET = typename std::conditional<PREC == NRX_BF16, __nv_bfloat16, __half>::type;
  constexpr int NPL = SPLIT ? 2 : 1;         // activation planes
  constexpr int NB = SPLIT ? 2 * NP : NP;     // pair MMA N (accumulator block)
  constexpr int BROWS = SPLIT ? NP : NP / 2;  // B rows held by each CTA
  constexpr int DST = SPLIT ? (NB + 31) / 32 * 32 : NB;  // TMEM columns per partial accumulator
  static_assert(SPLIT || MODE == EPI_RELU, "half-precision pair kernels: ReLU layers only");
  static_assert(!POSF || (KS == 3 && NK1 == 0 && MODE == EPI_RELU), "positional fold: 3x3 update.conv0 only");
  static_assert(TPC == 0 || (KS == 3 && 2 * NK0 == TPC + 1 && NK1 == 0 && PREC == NRX_FP32X3 && !POSF),
                "tap pairs: 3x3 layers over TPC data chunks of 2 NK0");
  // 32 accumulator columns per epilogue thread: 2 + 4 * NP/32 warps (10 for
  // NP = 64) leave each SM sub-partition <= 3 warps, i.e. up to 168 registers
  // for the fully unrolled MMA issue (18 warps would cap it at 96 and spill)
  constexpr int NC = x3_epi_cols(MODE, x3_small_k(KS, NK0, NK1));  // accumulator columns per epilogue thread
  constexpr int PARTS = (NP + NC - 1) / NC;  // NP = 56: the last part's columns past NP are ignored
  constexpr int EPI_WARPS = 4 * PARTS;
  extern __shared__ __align__(1024) uint8_t smem[];
  const Geom& g = p.g;
  const uint32_t rank = cta_rank();
  const int io = p.n_io > 1 ? blockIdx.y : 0;
  const ConvX3Smem L = conv_x3_smem(p);
  uint8_t* Ws = smem + L.w;
  const uint32_t As_s = smem_u32(smem + L.a);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* full = bars;         // [8] leader: both CTAs' stage landed
  uint64_t* empty = bars + 8;    // [8] both: stage consumed
  uint64_t* tfull = bars + 16;   // [2] both: accumulator ready
  uint64_t* tempty = bars + 18;  // [2] leader: both CTAs drained the accumulator
  uint64_t* wbar = bars + 20;    // own weights resident
  uint64_t* wpeer = bars + 21;   // leader: the peer's weights resident
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L.tmem_ptr);
  float* sbias = reinterpret_cast<float*>(smem + L.sbias);
  float* sdt = reinterpret_cast<float*>(smem + L.dt);
  float* sposw = reinterpret_cast<float*>(smem + L.posw);
  float* sptab = reinterpret_cast<float*>(smem + L.ptab);
  const uint32_t B_full = smem_u32(full), B_empty = smem_u32(empty), B_tfull = smem_u32(tfull),
                 B_tempty = smem_u32(tempty), B_wbar = smem_u32(wbar), B_wpeer = smem_u32(wpeer);

  // warp index and TMEM base through a lane-0 shuffle: provably warp-uniform, so the
  // MMA issue keeps its descriptors on the uniform datapath (no R2UR per MMA)
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
  pdl_launch_dependents();
  if (warp == 0) tmem_alloc2(tmem_ptr, p.tmem_cols);
  if (threadIdx.x == 32) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EPI_WARPS);
    }
    mbar_init(wbar, 1);
    mbar_init(wpeer, 1);
    fence_barrier_init();
  }
  if (threadIdx.x >= 64 && threadIdx.x <= 64 + NP)  // bias[0..NP) and the descale 2^-E at [NP]
    sbias[threadIdx.x - 64] = reinterpret_cast<const float*>(p.wbase + p.b_off[io])[threadIdx.x - 64];
  if (threadIdx.x < 32) sdt[threadIdx.x] = g.dt[threadIdx.x];
  if constexpr (POSF) {
    const float* pw = reinterpret_cast<const float*>(p.wbase + p.b_off[0]) + (NP + 4);  // posw_off(NP)
    for (int i = threadIdx.x; i < 18 * NP; i += blockDim.x) sposw[i] = pw[i];
  }
  if constexpr (POSF) {
    if (p.ptab) {  // interior positional contribution per (comb residue, symbol): weights and geometry only
      __syncthreads();
      const int cb = g.comb, n = cb * g.T * NP;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int c = i % NP, t = (i / NP) % g.T, r = i / (NP * g.T);
        float acc = 0.f;
        for (int a = 0; a < 3; ++a) {
          int q = (r + a - 1 + cb) % cb;
          q = q < cb - q ? q : cb - q;  // comb distance of the neighbour row
          const float f = g.freq_enc ? (cb <= 16 ? g.df_tab[q] : __fdiv_rn((float)q, (float)g.S)) : 0.f;
          for (int b = 0; b < 3; ++b) {
            const int t2 = t + b - 1;
            if (t2 < 0 || t2 >= g.T) continue;
            acc = fmaf(sdt[t2], sposw[(3 * a + b) * NP + c], acc);
            acc = fmaf(f, sposw[(9 + 3 * a + b) * NP + c], acc);
          }
        }
        sptab[(r * g.T + t) * (NP + 4) + c] = acc;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_ptr, 0);
  const int R = p.rbox;
#ifdef NRX_TIMING
  long long t_a = 0, t_b = 0, t_c = 0, t_all = clock64();
#endif
  const int nsrc = p.c1 ? 2 : 1;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      mbar_expect_tx(wbar, p.wbytes);
      const uint8_t* wsrc = p.wbase + p.w_off[io] + (size_t)rank * p.wbytes;
      for (uint32_t off = 0; off < p.wbytes; off += 32768u) {
        const uint32_t n = p.wbytes - off < 32768u ? p.wbytes - off : 32768u;
        bulk_load(Ws + off, wsrc + off, n, wbar);
      }
      const uint32_t full_leader = map_rank(B_full, 0);
      pdl_wait();
      PairIter w(g, g.NU, g.tiles, p.n_io, p.mod_order, (int)rank);
      int slab, tile, st = 0;
      bool real;
      uint32_t ph = 0;
      while (w.next(slab, tile, real)) {
        const int grp0 = (tile * NRX_TILE_M - p.hup) / 16;
        if constexpr (POSF) {  // one stage per plane: [src0 kc chunks | src1 kc chunks]
          for (int pl = 0; pl < NPL; ++pl) {
            mbar_wait_backoff(B_empty + 8u * st, ph ^ 1, 64);
            if (rank == 0) mbar_expect_tx(B_full + 8u * st, 2u * 2u * (uint32_t)p.kc * R * 16);
            const uint32_t dst = As_s + st * p.abytes;
            tma_load_4d_pair(dst, &map0, full_leader + 8u * st, 0, grp0, SPLIT && pl == 0 ? p.c0 / 8 : 0, slab);
            tma_load_4d_pair(dst + (uint32_t)p.kc * R * 16, &map1, full_leader + 8u * st, 0, grp0,
                             SPLIT && pl == 0 ? p.c1 / 8 : 0, slab ^ p.src1_xor);
            if (++st == p.stages) { st = 0; ph ^= 1; }
          }
          continue;
        }
        for (int pl = 0; pl < NPL; ++pl) {  // lo planes first (their MMAs run first), then hi
          for (int src = 0; src < nsrc; ++src) {
            const int cs = src ? p.c1 : p.c0;
            NRX_T(t0);
            mbar_wait_backoff(B_empty + 8u * st, ph ^ 1, 64);
            NRX_TADD(t_a, t0);
            if (rank == 0) mbar_expect_tx(B_full + 8u * st, 2u * (uint32_t)(TPC ? 8 * TPC : cs) * R * 2);
            tma_load_4d_pair(As_s + st * p.abytes, src ? &map1 : &map0, full_leader + 8u * st, 0, grp0,
                             SPLIT && pl == 0 ? cs / 8 : 0, src ? (slab ^ p.src1_xor) : slab);
            if (++st == p.stages) { st = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank != 0) {  // ---------------- peer: tell the leader this CTA's weights are resident
      if (lane == 0) {
        mbar_wait(B_wbar, 0);
        arrive_cluster(map_rank(B_wpeer, 0));
      }
    } else {  // ---------------- MMA issuer (leader, whole warp, elect.sync issues)
      // pair MMA M = 256, N = 2 NP: B = [W_hi (rank 0) | W_lo (rank 1)], so every
      // MMA writes [a W_hi | a W_lo] into a partial's two adjacent NP-column blocks
      constexpr uint32_t idesc = idesc_f16kind<ET>(2 * NRX_TILE_M, NB);
      const uint64_t a_desc0 = smem_desc(0, (uint32_t)R * 16, 128);
      const uint64_t b_desc0 = smem_desc(smem_u32(Ws), BROWS * 16, 128);
      const uint32_t a_kstep = 2 * R;
      const int ktap = p.c0 + p.c1, kch = ktap / 8;
      mbar_wait(B_wbar, 0);
      mbar_wait(B_wpeer, 0);
      tc_fence_after();
      PairIter w(g, g.NU, g.tiles, p.n_io, p.mod_order, 0);
      int slab, tile, st = 0, it = 0;
      bool real;
      uint32_t ph = 0;
      const int P = !SPLIT ? 1 : KS > 0 ? (KS > 1 ? 2 : 1) : p.nacc;  // partial accumulators (tap row % P)
      int shifts[KS > 0 ? KS * KS : 1];                               // tap row offsets (16-B units)
      if constexpr (KS > 0) {
#pragma unroll
        for (int tap = 0; tap < KS * KS; ++tap) shifts[tap] = (tap / KS - KS / 2) * g.Tp + (tap % KS - KS / 2);
      }
      while (w.next(slab, tile, real)) {
        const int acc = it & 1;
        NRX_T(t0);
        mbar_wait(B_tempty + 8u * acc, ((it >> 1) & 1) ^ 1);
        NRX_TADD(t_a, t0);
        tc_fence_after();
        const uint32_t d0 = tmem_base + acc * P * DST;
        // Plane lo: D_ra = lo' [W_hi | W_lo] (scale 2^11, first MMA of each partial
        // overwrites); plane hi: the first MMA of each partial folds (D 2^-11 +),
        // the rest accumulate hi [W_hi | W_lo].
        if constexpr (TPC > 0) {
          // tap-pair K order (tp2_slot): per plane pairs (0,1) (2,3) (4,5) (6,7) into
          // partials 0 1 0 1, then tap 8 into partial 0; step q reads B slots 2q, 2q+1
#pragma unroll
          for (int pl = 0; pl < NPL; ++pl) {
            mbar_wait(B_full + 8u * st, ph);
            tc_fence_after();
            const uint64_t a_stage = a_desc0 + (((As_s + st * p.abytes) >> 4) + p.hup);
            int q = 0;
            auto step = [&](uint64_t a, int part, bool first) {
              const uint64_t b = b_desc0 + (uint32_t)(2 * q * BROWS);
              const uint32_t d = d0 + part * DST;
              if (pl == 1 && first)
                mma2_warp_fold(d, a, b, idesc);
              else
                mma2_warp(d, a, b, idesc, !(pl == 0 && first));
              ++q;
            };
            constexpr int HALF = (TPC - 1) / 2;
#pragma unroll
            for (int pr = 0; pr < 4; ++pr) {
              const int t = 2 * pr, u = t + 1, part = pr & 1;
              const uint64_t at = a_stage + shifts[t], au = a_stage + shifts[u];
              // the straddling step: half 0 = (u, chunk 0), half 1 = (t, chunk C-1)
              const uint64_t lbo = (uint64_t)(uint32_t)(shifts[t] + (TPC - 1) * R - shifts[u] - R) << 16;
#pragma unroll
              for (int k = 0; k < HALF; ++k) step(at + (uint32_t)(2 * k * R), part, pr < 2 && k == 0);
              step(au + lbo, part, false);
#pragma unroll
              for (int k = 1; k <= HALF; ++k) step(au + (uint32_t)((2 * k - 1) * R), part, false);
            }
            const uint64_t a8 = a_stage + shifts[8];
#pragma unroll
            for (int k = 0; k < HALF; ++k) step(a8 + (uint32_t)(2 * k * R), 0, false);
            step(a8 + (uint32_t)((TPC - 2) * R), 0, false);  // zero-weight slot over chunk C-2, then chunk C-1
            commit2_warp(B_empty + 8u * st);
            if (++st == p.stages) { st = 0; ph ^= 1; }
          }
        } else if constexpr (KS > 0) {
          constexpr int KCH = 2 * (NK0 + NK1);
          constexpr int NSRC = NK1 > 0 ? 2 : 1;
          constexpr int PK = SPLIT && KS > 1 ? 2 : 1;
#pragma unroll
          for (int pl = 0; pl < NPL; ++pl) {
#pragma unroll
            for (int src = 0; src < NSRC; ++src) {
              NRX_T(t1);
              mbar_wait(B_full + 8u * st, ph);
              NRX_TADD(t_b, t1);
              tc_fence_after();
              const uint64_t a_stage = a_desc0 + (((As_s + st * p.abytes) >> 4) + p.hup);
              const int nk = src ? NK1 : NK0, kc0 = src ? 2 * NK0 : 0;
#pragma unroll
              for (int tap = 0; tap < KS * KS; ++tap) {
                const int ra = (tap / KS) % PK;
                const bool first = src == 0 && tap == ra * KS;  // first tap of the partial (k = 0)
#pragma unroll
                for (int k = 0; k < (NK0 > NK1 ? NK0 : NK1); ++k) {
                  if (k >= nk) break;
                  const uint64_t a = a_stage + shifts[tap] + (uint32_t)(k * a_kstep);
                  const uint64_t b = b_desc0 + (uint32_t)((tap * KCH + kc0 + 2 * k) * BROWS);
                  const uint32_t d = d0 + ra * DST;
                  if (SPLIT && pl == 1 && first && k == 0)
                    mma2_warp_fold(d, a, b, idesc);
                  else
                    mma2_warp(d, a, b, idesc, !(pl == 0 && first && k == 0));
                }
              }
              commit2_warp(B_empty + 8u * st);
              if (++st == p.stages) { st = 0; ph ^= 1; }
            }
          }
        } else {
          for (int pl = 0; pl < NPL; ++pl) {
            for (int src = 0; src < nsrc; ++src) {
              NRX_T(t1);
              mbar_wait(B_full + 8u * st, ph);
              NRX_TADD(t_b, t1);
              tc_fence_after();
              const uint64_t a_stage = a_desc0 + (((As_s + st * p.abytes) >> 4) + p.hup);
              const int nk = (src ? p.c1 : p.c0) / 16, kc0 = src ? p.c0 / 8 : 0;
              for (int tap = 0; tap < g.ks * g.ks; ++tap) {
                const int row = tap / g.ks, col = tap % g.ks;
                const int shift = (row - g.r) * g.Tp + (col - g.r);
                const int ra = row % P;
                const bool first = src == 0 && row == ra && col == 0;
                for (int k = 0; k < nk; ++k) {
                  const uint64_t a = a_stage + shift + (uint32_t)(k * a_kstep);
                  const uint64_t b = b_desc0 + (uint32_t)((tap * kch + kc0 + 2 * k) * BROWS);
                  const uint32_t d = d0 + ra * DST;
                  if (SPLIT && pl == 1 && first && k == 0)
                    mma2_warp_fold(d, a, b, idesc);
                  else
                    mma2_warp(d, a, b, idesc, !(pl == 0 && first && k == 0));
                }
              }
              commit2_warp(B_empty + 8u * st);
              if (++st == p.stages) { st = 0; ph ^= 1; }
            }
          }
        }
        commit2_warp(B_tfull + 8u * acc);
        ++it;
      }
    }
  } else {  // ---------------- epilogue (both CTAs): warps 2 .. 2 + EPI_WARPS - 1
    pdl_wait();
    const int q = warp & 3, part = (warp - 2) >> 2;
    const int r = 32 * q + lane;
    const int cbase = part * NC;
    const int nd = p.cdst / 8;              // chunks per plane of the output buffer
    const int dch = (g.d + 7) / 8;          // chunks holding state channels
    const uint32_t lane_off = static_cast<uint32_t>(32 * q) << 16;
    const uint32_t tempty_leader = map_rank(B_tempty, 0);
    const uint32_t sbias_s = smem_u32(sbias);
    const float descale = SPLIT ? sbias[NP] : 1.f;
    const int ndb = SPLIT ? 2 * nd : nd;  // chunks of the output buffer (both planes)
    const size_t dcs = (size_t)g.rows_slab * 8;  // chunk stride
    PairIter w(g, g.NU, g.tiles, p.n_io, p.mod_order, (int)rank);
    int slab, tile, it = 0;
    bool real;
    // residual update: the previous state of the NEXT tile is loaded while this
    // tile is processed (latency-bound loads: one tile in flight ahead)
    uint4 rhi[NC / 8], rlo[NC / 8];
    auto load_residual = [&](int sl, int tl, bool re) {
      const int rw = tl * NRX_TILE_M + r;
      int s2, t2;
      row_to_st(rw, g, s2, t2);
      const bool ok = re && rw < g.rows_data && t2 < g.T;
      const __half* src = chunk_ptr(p.dst, sl, ndb, 0, rw, g);
#pragma unroll
      for (int c8 = 0; c8 < NC / 8; ++c8) {
        const int cc = cbase / 8 + c8;
        rhi[c8] = rlo[c8] = make_uint4(0u, 0u, 0u, 0u);
        if (ok && cc < dch) {
          rhi[c8] = *reinterpret_cast<const uint4*>(src + cc * dcs);
          rlo[c8] = *reinterpret_cast<const uint4*>(src + (nd + cc) * dcs);
        }
      }
    };
    bool have = w.next(slab, tile, real);
    if (MODE == EPI_RESIDUAL && have) load_residual(slab, tile, real);
    while (have) {
      const int acc = it & 1;
      const int row = tile * NRX_TILE_M + r;
      int s, t;
      row_to_st(row, g, s, t);
      const bool valid = real && row < g.rows_data && t < g.T;
      __half* const drow = chunk_ptr(p.dst, slab, ndb, 0, row, g);
      const int cslab = slab;
      float old[NC];
      int nslab = 0, ntile = 0;
      bool nreal = false;
      const bool nhave = w.next(nslab, ntile, nreal);
      if (MODE == EPI_RESIDUAL) {
#pragma unroll
        for (int c8 = 0; c8 < NC / 8; ++c8) unsplit_chunk(rhi[c8], rlo[c8], old + 8 * c8);
        if (nhave) load_residual(nslab, ntile, nreal);
      }
      NRX_T(t0);
      mbar_wait_backoff(B_tfull + 8u * acc, (it >> 1) & 1, 128);
      NRX_TADD(t_a, t0);
      tc_fence_after();
      float v[NC];
      const int P = !SPLIT ? 1 : KS > 0 ? (KS > 1 ? 2 : 1) : p.nacc;
      const uint32_t taddr = tmem_base + lane_off + acc * P * DST + cbase;
      // sum of the partials' a*W_hi and a*W_lo blocks (fp32 round-to-nearest);
      // two blocks per TMEM round trip
      tmem_ld_cols<NC>(taddr, v);
      if (!SPLIT) tmem_wait_ld();
      if (SPLIT && NC <= 16 && KS > 1) {  // narrow threads: all four blocks in one TMEM round trip
        float w2[NC], w3[NC], w4[NC];
        tmem_ld_cols<NC>(taddr + NP, w2);
        tmem_ld_cols<NC>(taddr + DST, w3);
        tmem_ld_cols<NC>(taddr + DST + NP, w4);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < NC; ++c) v[c] = __fadd_rn(__fadd_rn(v[c], w2[c]), __fadd_rn(w3[c], w4[c]));
      } else if (SPLIT) {
        float w2[NC];
        tmem_ld_cols<NC>(taddr + NP, w2);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < NC; ++c) v[c] = __fadd_rn(v[c], w2[c]);
      }
      if (SPLIT && P > 1 && !(NC <= 16 && KS > 1)) {
        float w3[NC], w4[NC];
        tmem_ld_cols<NC>(taddr + DST, w3);
        tmem_ld_cols<NC>(taddr + DST + NP, w4);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < NC; ++c) v[c] = __fadd_rn(v[c], __fadd_rn(w3[c], w4[c]));
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_cluster_relaxed(tempty_leader + 8u * acc);
      ++it;
      const bool cur_real = real;
      have = nhave;
      slab = nslab;
      tile = ntile;
      real = nreal;
      if (!cur_real) continue;

      uint32_t bad = 0;  // range guard (fp16 planes)
      float pc[POSF ? 18 : 1];  // coefficients of W_pos[ch][tap]: pos_ch(s + a - 1, t + b - 1), 0 outside
      int prow = -1;            // row of the interior table, or -1: evaluate the 18 terms
      if constexpr (POSF) {
        const int u = cslab % g.U;
        const int o = u < g.comb ? u : u % g.comb;
        if (p.ptab && !valid) {
          prow = 0;  // pad row: stored as zero whatever the sum (keeps the warp on the table path)
        } else if (p.ptab && s > o && s < g.S - g.comb - 1) {
          const unsigned x = (unsigned)(s - o);
          const int q = g.comb == 1 ? 0 : (int)(x - (unsigned)g.comb * __umulhi(x, g.comb_magic));
          prow = q * g.T + t;
        }
        if (prow < 0) {
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const int s2 = s + a - 1;
            const bool ins = valid && s2 >= 0 && s2 < g.S;
            const float f = ins ? pos_df(s2, u, g) : 0.f;
#pragma unroll
            for (int b = 0; b < 3; ++b) {
              const int t2 = t + b - 1;
              const bool in = ins && t2 >= 0 && t2 < g.T;
              pc[3 * a + b] = in ? sdt[t2] : 0.f;
              pc[9 + 3 * a + b] = in ? f : 0.f;
            }
          }
        }
      }
      const uint32_t vmask = valid ? 0xffffffffu : 0u;
#pragma unroll
      for (int c8 = 0; c8 < NC / 8; ++c8) {
        const int cc = cbase / 8 + c8;
        if (MODE == EPI_RESIDUAL && cc >= dch) continue;  // constant positional / zero chunk
        if (cc >= nd || 8 * cc >= NP) continue;         // past the buffer / the accumulator
        float bb[8], x[8], pz[8];
        ld_shared_f8(sbias_s + 32u * cc, bb);
        const bool full = 8 * cc + 8 <= g.d;  // warp-uniform
#pragma unroll
        for (int e = 0; e < 8; ++e) pz[e] = 0.f;
        if constexpr (POSF) {
          if (prow >= 0) {
            ld_shared_f8(smem_u32(sptab) + 4u * (uint32_t)(prow * (NP + 4) + 8 * cc), pz);
          } else {
#pragma unroll
            for (int k = 0; k < 18; ++k) {
              float wp[8];
              ld_shared_f8(smem_u32(sposw) + 4u * (uint32_t)(k * NP + 8 * cc), wp);
#pragma unroll
              for (int e = 0; e < 8; ++e) pz[e] = fmaf(pc[k], wp[e], pz[e]);
            }
          }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          // conv (exact 2^-E; + the folded positional terms) + bias, as the reference
          // (v 2^-E is exact, so the fma rounds once exactly like the separate multiply and add)
          float y = POSF ? __fadd_rn(fmaf(v[8 * c8 + e], descale, pz[e]), bb[e]) : fmaf(v[8 * c8 + e], descale, bb[e]);
          if (MODE == EPI_RELU) y = relu_f(y);
          if (MODE == EPI_RESIDUAL) y = old[8 * c8 + e] + y;
          x[e] = y;
        }
        if (full) {  // every channel of the chunk is a state channel: pad rows zeroed on the packed words
          if constexpr (SPLIT) {
            uint4 hi, lo;
            split_chunk(x, hi, lo);
            hi = mask_chunk(hi, vmask);
            lo = mask_chunk(lo, vmask);
            const uint32_t h[4] = {hi.x, hi.y, hi.z, hi.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) bad |= ((h[i] & 0x7c007c00u) + 0x04000400u) & 0x80008000u;  // as split_chunk
            *reinterpret_cast<uint4*>(drow + cc * dcs) = hi;
            *reinterpret_cast<uint4*>(drow + (nd + cc) * dcs) = lo;
          } else {
            *reinterpret_cast<uint4*>(drow + cc * dcs) = mask_chunk(pack_chunk(x, static_cast<const ET*>(nullptr)), vmask);
          }
          continue;
        }
        // the chunk holding channel d (and the positional channels d, d+1 of the state)
        const float pdt = (MODE != EPI_RELU && valid) ? sdt[t] : 0.f;
        const float pdf = (MODE != EPI_RELU && valid) ? pos_df(s, cslab % g.U, g) : 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int c = 8 * cc + e;
          x[e] = (valid && c < g.d) ? x[e] : 0.f;
          if (MODE != EPI_RELU && valid && c == g.d) x[e] = pdt;
          if (MODE != EPI_RELU && valid && c == g.d + 1) x[e] = pdf;
        }
        if constexpr (SPLIT) {
          uint4 hi, lo;
          split_chunk(x, hi, lo, bad);
          *reinterpret_cast<uint4*>(drow + cc * dcs) = hi;
          *reinterpret_cast<uint4*>(drow + (nd + cc) * dcs) = lo;
        } else {
          *reinterpret_cast<uint4*>(drow + cc * dcs) = pack_chunk(x, static_cast<const ET*>(nullptr));
        }
      }
      report_range(bad, g.flag);
      if (part == PARTS - 1) {  // buffer channels beyond the accumulator: positional / zero only
        const float qdt = (valid && MODE != EPI_RELU) ? sdt[t] : 0.f;
        const float qdf = (valid && MODE != EPI_RELU && MODE != EPI_RESIDUAL) ? pos_df(s, cslab % g.U, g) : 0.f;
        for (int cc = NP / 8; cc < nd; ++cc) {
          if (MODE == EPI_RESIDUAL) break;  // written once by the state init
          if (MODE == EPI_RELU && p.hskip) break;  // h for a tap-pair conv1, which reads 7 chunks only
          float o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int c = 8 * cc + e;
            o[e] = c == g.d ? qdt : c == g.d + 1 ? qdf : 0.f;
          }
          if constexpr (SPLIT) {
            uint4 hi, lo;
            split_chunk(o, hi, lo);
            *reinterpret_cast<uint4*>(drow + cc * dcs) = hi;
            *reinterpret_cast<uint4*>(drow + (nd + cc) * dcs) = lo;
          } else {
            *reinterpret_cast<uint4*>(drow + cc * dcs) = pack_chunk(o, static_cast<const ET*>(nullptr));
          }
        }
      }
    }
  }
#ifdef NRX_TIMING
  if (blockIdx.x < 2 && blockIdx.y == 0 && (threadIdx.x == 0 || threadIdx.x == 32 || threadIdx.x == 64))
    printf("x3 NP=%d mode=%d KS=%d c0=%d c1=%d cta=%d tid=%d all=%lld waitA=%lld waitB=%lld\n", NP, MODE, KS, p.c0,
           p.c1, blockIdx.x, threadIdx.x, clock64() - t_all, t_a, t_b);
#endif
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the leader's last MMAs read the peer's shared memory / write its TMEM
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, p.tmem_cols);
  }
}

using X3Fn = void (*)(const ConvX3Params, const CUtensorMap, const CUtensorMap);

template <int NP>
static X3Fn select_conv_x3(const Geom& g, int mode, int c0, int c1, int prec, bool posf, bool* small) {
  *small = false;
  if (posf) {  // update.conv0 without the positional channels in K (upd0_posf)
    if constexpr (NP == 56) return g.d == 56 ? k_conv_x3<56, EPI_RELU, 3, 7, 0, NRX_FP32X3, true> : nullptr;
    if constexpr (NP == 16) {
      *small = true;
      return g.d == 16 ? k_conv_x3<16, EPI_RELU, 3, 2, 0, NRX_FP32X3, true> : nullptr;
    }
    return nullptr;
  }
  if (prec != NRX_FP32X3) {  // half-precision pair kernels: ReLU layers only, np 32 / 64
    if constexpr (NP == 32 || NP == 64) {
      const bool f16 = prec == NRX_FP16;
      if (mode != EPI_RELU) return nullptr;
      if (NP == 64 && g.ks == 3 && c0 == 32 && c1 == 0) {
        *small = true;
        return f16 ? k_conv_x3<64, EPI_RELU, 3, 2, 0, NRX_FP16> : k_conv_x3<64, EPI_RELU, 3, 2, 0, NRX_BF16>;
      }
      if (NP == 64 && g.ks == 3 && c0 == 64 && c1 == 64)
        return f16 ? k_conv_x3<64, EPI_RELU, 3, 4, 4, NRX_FP16> : k_conv_x3<64, EPI_RELU, 3, 4, 4, NRX_BF16>;
      return f16 ? k_conv_x3<NP, EPI_RELU, 0, 0, 0, NRX_FP16> : k_conv_x3<NP, EPI_RELU, 0, 0, 0, NRX_BF16>;
    }
    return nullptr;
  }
  static const X3Fn generic[3] = {k_conv_x3<NP, 0>, k_conv_x3<NP, 1>, k_conv_x3<NP, 2>};
  X3Fn fn = generic[mode];
  if (NP == 16 && g.ks == 3) {  // the desk models (d_s = 16): features 32, state 32, h / messages 16 channels
    const int nk0 = c0 / 16, nk1 = c1 / 16;
    if (mode == EPI_RELU && nk0 == 2 && nk1 == 0) fn = k_conv_x3<16, EPI_RELU, 3, 2, 0>, *small = true;
    if (mode == EPI_RELU && nk0 == 2 && nk1 == 1) fn = k_conv_x3<16, EPI_RELU, 3, 2, 1>;
    if (mode == EPI_STATE_INIT && nk0 == 1 && nk1 == 0) fn = k_conv_x3<16, EPI_STATE_INIT, 3, 1, 0>, *small = true;
    if (mode == EPI_RESIDUAL && nk0 == 1 && nk1 == 0) fn = k_conv_x3<16, EPI_RESIDUAL, 3, 1, 0>, *small = true;
  }
  if (NP == 56 && g.ks == 3) {  // fully unrolled issue for the RT / large models' 3x3 layers
    const int nk0 = c0 / 16, nk1 = c1 / 16;
    if (mode == EPI_RELU && nk0 == 2 && nk1 == 0) fn = k_conv_x3<56, EPI_RELU, 3, 2, 0>, *small = true;
    if (mode == EPI_RELU && nk0 == 4 && nk1 == 4) fn = k_conv_x3<56, EPI_RELU, 3, 4, 4>;
    const bool tp2 = tp2_layer(g.d, g.ks, prec);
    if (mode == EPI_STATE_INIT && nk0 == 4 && nk1 == 0)
      fn = tp2 ? k_conv_x3<56, EPI_STATE_INIT, 3, 4, 0, NRX_FP32X3, false, 7> : k_conv_x3<56, EPI_STATE_INIT, 3, 4, 0>;
    if (mode == EPI_RESIDUAL && nk0 == 4 && nk1 == 0)
      fn = tp2 ? k_conv_x3<56, EPI_RESIDUAL, 3, 4, 0, NRX_FP32X3, false, 7> : k_conv_x3<56, EPI_RESIDUAL, 3, 4, 0>;
    if (mode == EPI_RELU && nk0 == 2 && nk1 == 0 && tp2_chunks(g.d, g.ks, prec, c0, g.Cin) == 3)
      fn = k_conv_x3<56, EPI_RELU, 3, 2, 0, NRX_FP32X3, false, 3>, *small = true;
  }
  return fn;
}

// 4-D map over a split buffer [NU][2C/8][rows][8] fp16 whose box covers the
// C/8 chunks of one plane (the plane is picked by the chunk coordinate).
static int make_map_plane(CUtensorMap* m, const void* base, const Geom& g, int C, int rbox, int box_chunks) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return NRX_ERR_NO_DEVICE;
  if (rbox % 16 || g.rows_slab % 16) return NRX_ERR_UNSUPPORTED;
  const cuuint64_t dims[4] = {128, (cuuint64_t)(g.rows_slab / 16), (cuuint64_t)(2 * C / 8), (cuuint64_t)g.NU};
  const cuuint64_t strides[3] = {256, (cuuint64_t)g.rows_slab * 16, (cuuint64_t)(2 * C / 8) * g.rows_slab * 16};
  const cuuint32_t box[4] = {128, (cuuint32_t)(rbox / 16), (cuuint32_t)box_chunks, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? NRX_OK : NRX_ERR_CUDA;
}

}  // namespace tc

int launch_conv_x3(const Geom& g, const ConvX3Launch& c, const uint8_t* wb, const int32_t* mod_order,
                   cudaStream_t st) {
  using namespace tc;
  const bool split = c.prec == NRX_FP32X3;
  ConvX3Params p{};
  p.g = g;
  p.c0 = c.c0;
  p.c1 = c.c1;
  p.src1_xor = c.src1_xor;
  p.np = split ? x3_np(g.d) : rup(g.d, 16);
  if (!split && p.np != 32 && p.np != 64) return NRX_ERR_UNSUPPORTED;
  p.cdst = c.cdst;
  p.n_io = c.n_off;
  p.hup = rup(g.H, 16);
  p.rbox = NRX_TILE_M + 2 * p.hup;
  p.posf = c.posf ? 1 : 0;
  p.hskip = split && c.mode == EPI_RELU && tp2_layer(g.d, g.ks, c.prec) && c.cdst == g.Ch ? 1 : 0;
  p.kc = g.d / 8;
  if (c.posf && (g.d % 8 || !c.c1)) return NRX_ERR_UNSUPPORTED;
  const int ktap = c.posf ? 2 * g.d : c.c0 + c.c1;
  // split: W_hi (rank 0) or W_lo (rank 1) for every output channel; else np/2 output channels
  p.wbytes = (uint32_t)(g.ks * g.ks * ktap * (split ? p.np : p.np / 2) * 2);
  p.abytes = c.posf ? (uint32_t)(2 * p.kc * p.rbox * 16) : (uint32_t)((c.c0 > c.c1 ? c.c0 : c.c1) * p.rbox * 2);
  p.wbase = wb;
  for (int i = 0; i < p.n_io; ++i) {
    p.w_off[i] = c.offs[i].w;
    p.b_off[i] = c.offs[i].b;
  }
  p.mod_order = mod_order;
  p.dst = static_cast<__half*>(c.dst);
  // partial accumulators (tap row % P), each [a W_hi | a W_lo]: 2 P np columns per tile, double buffered
  p.nacc = split && g.ks > 1 ? 2 : 1;
  const uint32_t cols = split ? 2 * p.nacc * ((2 * p.np + 31) / 32 * 32) : 2 * p.np;
  p.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  p.ptab = p.posf;
  p.stages = 8;
  while (p.stages > 2 && conv_x3_smem(p).total > SMEM_LIMIT) --p.stages;
  if (p.ptab && conv_x3_smem(p).total > SMEM_LIMIT) {  // no room for the table: edge path for every row
    p.ptab = 0;
    p.stages = 8;
    while (p.stages > 2 && conv_x3_smem(p).total > SMEM_LIMIT) --p.stages;
  }
  if (conv_x3_smem(p).total > SMEM_LIMIT || p.rbox > 256 || p.np > 64 || c.mode < 0 || c.mode > 2)
    return NRX_ERR_UNSUPPORTED;
  const size_t smem = conv_x3_smem(p).total;
  CUtensorMap m0, m1;
  const void* s1 = c.src1 ? c.src1 : c.src0;
  const int cc1 = c.c1 ? c.c1 : c.c0;
  // tap-pair layers load only their C data chunks (the kernel's TPC instance): the conv1 layers of
  // d_s = 56 (C = 7) and state_init.conv0 over the 19 feature channels (C = 3)
  int tpc = 0;
  if (split && !c.posf && c.c1 == 0) {
    if ((c.mode == EPI_STATE_INIT || c.mode == EPI_RESIDUAL) && c.c0 == 64 && tp2_layer(g.d, g.ks, c.prec)) tpc = 7;
    if (c.mode == EPI_RELU && tp2_chunks(g.d, g.ks, c.prec, c.c0, g.Cin) == 3 && c.c0 == g.Cf) tpc = 3;
  }
  const int box0 = c.posf ? p.kc : tpc ? tpc : c.c0 / 8, box1 = c.posf ? p.kc : cc1 / 8;
  int rc = split ? make_map_plane(&m0, c.src0, g, c.c0, p.rbox, box0) : make_map(&m0, c.src0, g, c.c0, p.rbox, box0);
  if (rc) return rc;
  rc = split ? make_map_plane(&m1, s1, g, cc1, p.rbox, box1) : make_map(&m1, s1, g, cc1, p.rbox, box1);
  if (rc) return rc;
  X3Fn fn = nullptr;
  bool small = false;  // the selected instance drains 16 columns per epilogue thread (x3_small_k)
  switch (p.np) {
    case 16: fn = select_conv_x3<16>(g, c.mode, c.c0, c.c1, c.prec, c.posf, &small); break;
    case 32: fn = select_conv_x3<32>(g, c.mode, c.c0, c.c1, c.prec, c.posf, &small); break;
    case 48: fn = select_conv_x3<48>(g, c.mode, c.c0, c.c1, c.prec, c.posf, &small); break;
    case 56: fn = select_conv_x3<56>(g, c.mode, c.c0, c.c1, c.prec, c.posf, &small); break;
    case 64: fn = select_conv_x3<64>(g, c.mode, c.c0, c.c1, c.prec, c.posf, &small); break;
    default: return NRX_ERR_UNSUPPORTED;
  }
  if (!fn) return NRX_ERR_UNSUPPORTED;
  if (set_smem((const void*)fn, SMEM_LIMIT)) return NRX_ERR_CUDA;
  const int total = g.NU * g.tiles;
  const int pairs_max = num_sms() / 2;
  const int pairs = (total + 1) / 2 < pairs_max ? (total + 1) / 2 : pairs_max;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs, p.n_io);
  const int nc = x3_epi_cols(c.mode, small);
  cfg.blockDim = dim3(64 + 128 * ((p.np + nc - 1) / nc));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  if (cudaLaunchKernelEx(&cfg, fn, p, m0, m1) != cudaSuccess) return NRX_ERR_CUDA;
  return cudaPeekAtLastError() == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

#define NRX_TRY_X3(x)            \
  do {                           \
    int _s = (x);                \
    if (_s != NRX_OK) return _s; \
  } while (0)

int launch_msg(const Geom& g, const PackLayout& L, const uint8_t* wb, const void* state, void* agg,
               cudaStream_t st);
int launch_readout(const Geom& g, const PackLayout& L, const uint8_t* wb, const void* state,
                   const int32_t* mod_order, float* llr, float2* chest, cudaStream_t st);

// fp32x3 forward (after K1): state init, per iteration message MLP + sum of
// the others, update conv0 on [state | agg], update conv1 + residual; readout.
int launch_forward_x3(const Geom& g, const PackLayout& L, const WsLayout& W, int n_it, const uint8_t* wb,
                      const int32_t* mod_order, uint8_t* ws, float* llr, float2* chest, cudaStream_t st) {
  if (g.d > 64 || g.h > 128) return NRX_ERR_UNSUPPORTED;
  void* feats = ws + W.feats;
  void* h = ws + W.h;
  void* state = ws + W.state;
  void* agg = ws + W.agg;
  ConvX3Launch c{};
  c.offs = L.init0;
  c.n_off = g.n_io;
  c.src0 = feats;
  c.c0 = g.Cf;
  c.dst = h;
  c.cdst = g.Ch;
  c.mode = EPI_RELU;
  {
    ProfScope ps(KID_INIT0, st);
    NRX_TRY_X3(launch_conv_x3(g, c, wb, mod_order, st));
  }
  c = ConvX3Launch{};
  c.offs = L.init1;
  c.n_off = g.n_io;
  c.src0 = h;
  c.c0 = g.Ch;
  c.dst = state;
  c.cdst = g.Cs;
  c.mode = EPI_STATE_INIT;
  {
    ProfScope ps(KID_INIT1, st);
    NRX_TRY_X3(launch_conv_x3(g, c, wb, mod_order, st));
  }
  for (int it = 0; it < n_it; ++it) {
    {
      ProfScope ps(KID_MSG, st);
      NRX_TRY_X3(launch_msg(g, L, wb, state, agg, st));
    }
    c = ConvX3Launch{};
    c.offs = &L.upd0;
    c.n_off = 1;
    c.src0 = state;
    c.c0 = g.Cs;
    c.src1 = agg;
    c.c1 = g.Ca;
    c.dst = h;
    c.cdst = g.Ch;
    c.mode = EPI_RELU;
    c.posf = upd0_posf(g.d, g.ks, NRX_FP32X3);
    {
      ProfScope ps(KID_UPD0, st);
      NRX_TRY_X3(launch_conv_x3(g, c, wb, mod_order, st));
    }
    c = ConvX3Launch{};
    c.offs = &L.upd1;
    c.n_off = 1;
    c.src0 = h;
    c.c0 = g.Ch;
    c.dst = state;
    c.cdst = g.Cs;
    c.mode = EPI_RESIDUAL;
    ProfScope ps(KID_UPD1, st);
    NRX_TRY_X3(launch_conv_x3(g, c, wb, mod_order, st));
  }
  ProfScope ps(KID_READOUT, st);
  return launch_readout(g, L, wb, state, mod_order, llr, chest, st);
}

}  // namespace nrx
