// Tensor-core (bf16 / fp16) convolution with an optional fused per-RE MLP
// tail, and the launch sequence of the tensor-core forward pass.
//
//  k_conv_tc     k x k 'same' convolution as an implicit GEMM on the
//                row-linearised grid (nrx_internal.h).  Per 128-row M tile the
//                producer warp TMA-loads the tile plus +-H halo rows of every
//                input channel chunk ONCE per input source (4-D box
//                {128, rows/16, C/8, 1}, zero filled outside the slab); tap (a,b)
//                is the same shared-memory tile viewed at a row offset
//                (a-r)*Tp + (b-r), which the no-swizzle K-major UMMA descriptor
//                addresses directly (16-byte granular start address).  The whole
//                layer's weights stay resident in shared memory (bulk copy once
//                per CTA).  The MMA warp issues taps * C/16 MMAs (M=128,
//                N=rup(d,16), K=16) into one of two TMEM accumulators; eight
//                epilogue warps drain the other (tcgen05.ld) and apply bias /
//                ReLU / positional channels / residual while the next tile's
//                MMAs run.
//
//  Fused MLP tail (conv1 of the state init and of the iteration block):
//  the epilogue also writes the fresh state tile into shared memory as the A
//  operand of a two-layer per-RE MLP that runs on the same tensor core
//  between the next tile's conv MMAs:
//    TAIL_MSG      the message MLP of the next iteration (nrx.py:258); for
//                  U = 2 the sum of the other UE's messages is exactly that
//                  UE's message, so the next update conv reads the partner
//                  slab's messages directly (source-1 slab ^ 1) and the
//                  separate message kernel disappears;
//    TAIL_READOUT  the fused LLR + chest readout after the last iteration
//                  (nrx.py:338-340), writing the user-facing outputs.
#include "nrx_profile.h"
#include "tc_common.cuh"

namespace nrx {
namespace tc {

enum ConvTail { TAIL_NONE = 0, TAIL_MSG = 1, TAIL_READOUT = 2 };

struct ConvTcParams {
  Geom g;
  int ktap, c0, c1;     // A channels per tap = c0 (source 0) + c1 (source 1)
  int np, cdst, mode, stages;
  int n_io, d4;
  uint32_t wbytes, abytes, tmem_cols, rbox;
  int hup;              // halo rows loaded on each side (H rounded up to 16)
  int src1_xor;         // source-1 slab = slab ^ src1_xor (1: partner UE's messages)
  const uint8_t* wbase;
  uint64_t w_off[NRX_MAX_IO], b_off[NRX_MAX_IO];
  const int32_t* mod_order;
  void* dst;            // bf16 / fp16 output buffer (element type = kernel's ET)
  float* dst32;         // fp32 master state (bf16 STATE_INIT / RESIDUAL), or null
  // fused MLP tail
  int thp, top;         // tail hidden (padded) / output columns
  uint32_t tw0bytes, tw1bytes;
  uint64_t tw0[NRX_MAX_IO], tb0[NRX_MAX_IO], tw1[NRX_MAX_IO], tb1[NRX_MAX_IO];
  void* msg;            // TAIL_MSG output: [slab][Ca/8][rows][8] ET
  float* llr;           // TAIL_READOUT outputs
  float2* chest;
  int racc;             // residual through the accumulator (conv_racc): three state tiles + identity B
};

// fp16 update.conv1 with the RT message / readout tail: the previous state
// enters the accumulator as a fifth K block (the state tile by TMA into the
// tail's A buffer, times a 64 x 64 identity B; fp16 -> fp32 is exact) instead
// of a global load + convert + add per element in the epilogue.
template <typename ET, int MODE, int TPC, int TH>
__host__ __device__ constexpr bool conv_racc() {
  return std::is_same<ET, __half>::value && MODE == 2 && TPC == 7 && TH > 0;
}

// warp 0 TMA producer, warp 1 MMA issuer, then NP/16 groups of four epilogue
// warps (one per TMEM lane quarter); every epilogue thread drains 16
// accumulator columns of one row (NP=64: 16 epilogue warps, 576 threads).
__host__ __device__ constexpr int conv_parts(int np) { return np / 16; }
__host__ __device__ constexpr int conv_epi_threads(int np) { return 128 * conv_parts(np); }
__host__ __device__ constexpr int conv_threads(int np) { return 64 + conv_epi_threads(np); }

// Shared-memory carve-up (identical on host and device).
struct ConvSmem {
  uint32_t w, a, tw0, tw1, ta, th, ident, bars, tmem_ptr, sbias, tb0, tb1, dt, total;
};
__host__ __device__ inline ConvSmem conv_smem_layout(const ConvTcParams& p, int tail) {
  ConvSmem s;
  uint32_t off = 0;
  s.w = off;
  off = (p.wbytes + 1023u) & ~1023u;
  s.a = off;
  off += p.stages * p.abytes;
  s.tw0 = s.tw1 = s.ta = s.th = off;
  if (tail) {  // tail weights, double-buffered state tile (A), hidden tile(s) (H: two for TAIL_MSG)
    s.tw0 = off;
    off += p.tw0bytes;
    s.tw1 = off;
    off += p.tw1bytes;
    s.ta = off;
    off += (p.racc ? 3u : 2u) * p.g.Cs * NRX_TILE_M * 2;
    s.th = off;
    off += (tail == TAIL_MSG ? 2u : 1u) * p.thp * NRX_TILE_M * 2;
  }
  s.ident = off;  // racc: identity B operand (64 x 64 fp16, K-major core matrices)
  if (p.racc) off += 64 * 64 * 2;
  s.bars = off;
  off += 40 * 8;
  s.tmem_ptr = off;
  off += 16;
  s.sbias = off;
  off += 64 * 4;
  s.tb0 = off;
  off += 256 * 4;
  s.tb1 = off;
  off += 64 * 4;
  s.dt = off;  // symbol-axis positional encoding (per-lane indexed: shared, not the constant bank)
  off += 32 * 4;
  s.total = off;
  return s;
}

// KS > 0 selects the fully unrolled MMA issue for kernel size KS with NK0 /
// NK1 K=16 steps per tap from source 0 / 1 (host picks it when the layer
// matches); KS = 0 is the generic runtime-loop version.
// ET = __nv_bfloat16 or __half: operand/activation element type.
// TPC > 0: the tap-pair K order over TPC data chunks (tp2_chunks, nrx_internal.h).
// TH > 0: compile-time tail shape of the RT models (Cs = Ca = 64, hidden TH: 64
// for the message tail, 128 for the readout), fully unrolled tail stages.
template <typename ET, int NP, int MODE, int TAIL, int KS = 0, int NK0 = 0, int NK1 = 0, int TPC = 0, int TH = 0>
__global__ void __launch_bounds__(conv_threads(NP), 1)
    k_conv_tc(const __grid_constant__ ConvTcParams p, const __grid_constant__ CUtensorMap map0,
              const __grid_constant__ CUtensorMap map1) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const Geom& g = p.g;
  ET* const dst = static_cast<ET*>(p.dst);
  const int io = p.n_io > 1 ? blockIdx.y : 0;
  const ConvSmem L = conv_smem_layout(p, TAIL);
  uint8_t* Ws = smem + L.w;
  uint8_t* As = smem + L.a;
  const uint32_t As_s = smem_u32(As);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* full = bars;
  uint64_t* empty = bars + 8;
  uint64_t* tfull = bars + 16;
  uint64_t* tempty = bars + 18;
  uint64_t* wbar = bars + 20;
  uint64_t* ta_ready = bars + 29;   // [NTA] tail: state tile in shared memory
  uint64_t* hid_full = bars + 23;   // [2] tail: fc0 done
  uint64_t* h_ready = bars + 25;    // [2] tail: hidden layer in shared memory
  uint64_t* tout_full = bars + 27;  // [2] tail: fc1 done
  uint64_t* ta_free = bars + 32;    // [3] racc: fc0 read the state tile
  uint64_t* res_full = bars + 35;   // [3] racc: previous state tile loaded
  constexpr bool RACC = conv_racc<ET, MODE, TPC, TH>();
  constexpr int NTA = RACC ? 3 : 2;  // state tiles (fc0's A operand)
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L.tmem_ptr);
  // shared-space addresses of the barriers (8 B each)
  const uint32_t B_full = smem_u32(full), B_empty = smem_u32(empty), B_tfull = smem_u32(tfull),
                 B_tempty = smem_u32(tempty), B_wbar = smem_u32(wbar), B_ta_ready = smem_u32(ta_ready),
                 B_hid_full = smem_u32(hid_full), B_h_ready = smem_u32(h_ready), B_tout_full = smem_u32(tout_full),
                 B_ta_free = smem_u32(ta_free), B_res_full = smem_u32(res_full);
  float* sbias = reinterpret_cast<float*>(smem + L.sbias);
  float* stb0 = reinterpret_cast<float*>(smem + L.tb0);
  float* stb1 = reinterpret_cast<float*>(smem + L.tb1);
  float* sdt = reinterpret_cast<float*>(smem + L.dt);

  // lane-0 shuffles: provably warp-uniform values keep the MMA issue on the uniform datapath
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
  pdl_launch_dependents();  // the next layer's prologue may run on SMs this grid frees
  if (warp == 0) tmem_alloc(tmem_ptr, p.tmem_cols);
  if (threadIdx.x == 32) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], conv_epi_threads(NP));
    }
    mbar_init(wbar, 1);
    for (int b = 0; b < NTA; ++b) mbar_init(&ta_ready[b], conv_epi_threads(NP));
    if (RACC)
      for (int b = 0; b < 3; ++b) {
        mbar_init(&ta_free[b], 1);
        mbar_init(&res_full[b], 1);
      }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&hid_full[b], 1);
      mbar_init(&h_ready[b], conv_epi_threads(NP));
      mbar_init(&tout_full[b], 1);
    }
    fence_barrier_init();
  }
  if (threadIdx.x >= 64 && threadIdx.x < 64 + NP)
    sbias[threadIdx.x - 64] = reinterpret_cast<const float*>(p.wbase + p.b_off[io])[threadIdx.x - 64];
  if (threadIdx.x < 32) sdt[threadIdx.x] = g.dt[threadIdx.x];
  if (RACC) {
    // B of the fifth K block: chunk kc, row n < d holds e_n over K = 8 kc .. 8 kc + 7 (identity:
    // + previous state), and in chunk 7 (K = 56..63, the state tile's pad channels) the conv
    // bias split into fp16 hi / lo at K = 62 / 63, which the state tiles hold as constant ones
    const float* cb = reinterpret_cast<const float*>(p.wbase + p.b_off[io]);
    for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) {
      const int kc = i >> 6, n = i & 63, e = n - 8 * kc;
      const uint32_t one = (e & 1) ? 0x3c000000u : 0x3c00u;  // 1.0 in fp16, low / high half
      const int wd = n < g.d && e >= 0 && e < 8 ? e >> 1 : -1;
      uint4 v = make_uint4(wd == 0 ? one : 0u, wd == 1 ? one : 0u, wd == 2 ? one : 0u, wd == 3 ? one : 0u);
      if (kc == 7 && n < g.d) {
        const __half bh = __float2half_rn(cb[n]);
        const __half bl = __float2half_rn(cb[n] - __half2float(bh));
        v.w = (uint32_t)__half_as_ushort(bh) | ((uint32_t)__half_as_ushort(bl) << 16);
      }
      *reinterpret_cast<uint4*>(smem + L.ident + 16u * i) = v;
    }
    // the state tiles' pad chunks (never loaded or written per tile): zero, ones at K = 62, 63
    for (int i = threadIdx.x; i < 3 * NRX_TILE_M; i += blockDim.x)
      *reinterpret_cast<uint4*>(smem + L.ta + (i / NRX_TILE_M) * (uint32_t)g.Cs * NRX_TILE_M * 2 +
                                ((uint32_t)7 * NRX_TILE_M + i % NRX_TILE_M) * 16u) = make_uint4(0u, 0u, 0u, 0x3c003c00u);
    fence_proxy_async();  // generic-proxy stores -> tensor-core reads
  }
  if (TAIL) {
    const float* b0 = reinterpret_cast<const float*>(p.wbase + p.tb0[io]);
    const float* b1 = reinterpret_cast<const float*>(p.wbase + p.tb1[io]);
    for (int i = threadIdx.x; i < p.thp; i += blockDim.x) stb0[i] = b0[i];
    for (int i = threadIdx.x; i < p.top; i += blockDim.x) stb1[i] = b1[i];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_ptr, 0);
  // tail shape: compile-time for TH > 0
  const int thp = TH ? TH : p.thp, top = TH ? (TAIL == TAIL_MSG ? 64 : 32) : p.top, tcs = TH ? 64 : g.Cs;
  // tail TMEM regions (double buffered): hidden at col_h + b*thp, outputs at col_o + b*top
  const uint32_t col_h = 2 * NP, col_o = 2 * NP + 2 * thp;
  const uint32_t ta_bytes = (uint32_t)tcs * NRX_TILE_M * 2, th_bytes = (uint32_t)thp * NRX_TILE_M * 2;
  const int R = p.rbox;
  // fc1 of tile j is issued LAG tiles after conv(j).  TAIL_MSG: LAG = 3 with two
  // hidden tiles, so the MMA warp's wait for a hidden layer never holds back the
  // next conv by less than two epilogue iterations; TAIL_READOUT (wider hidden
  // layer, one tile fits): LAG = 2.
  constexpr int LAG = TAIL == TAIL_MSG ? 3 : 2;
  constexpr uint32_t NTH = TAIL == TAIL_MSG ? 2 : 1;
#ifdef NRX_TIMING
  long long t_a = 0, t_b = 0, t_c = 0, t_d = 0, t_all = clock64();
#endif

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      const uint32_t tbytes = TAIL ? p.tw0bytes + p.tw1bytes : 0;
      mbar_expect_tx(wbar, p.wbytes + tbytes);
      for (uint32_t off = 0; off < p.wbytes; off += 32768u) {
        const uint32_t n = p.wbytes - off < 32768u ? p.wbytes - off : 32768u;
        bulk_load(Ws + off, p.wbase + p.w_off[io] + off, n, wbar);
      }
      if (TAIL) {
        bulk_load(smem + L.tw0, p.wbase + p.tw0[io], p.tw0bytes, wbar);
        bulk_load(smem + L.tw1, p.wbase + p.tw1[io], p.tw1bytes, wbar);
      }
      pdl_wait();  // activations: written by the previous layer
      // one pipeline stage per (tile, input source): finer-grained stages keep
      // more loads in flight next to the resident weights
      WorkIter w(g, g.NU, g.tiles, p.n_io, p.mod_order);
      int slab, tile, st = 0, it = 0;
      uint32_t ph = 0;
      while (w.next(slab, tile)) {
        const int grp0 = (tile * NRX_TILE_M - p.hup) / 16;  // 16-row groups
        for (int src = 0; src < (p.c1 ? 2 : 1); ++src) {
          NRX_T(t0);
          mbar_wait(B_empty + 8u * (st), ph ^ 1);
          NRX_TADD(t_a, t0);
          mbar_expect_tx(B_full + 8u * (st), (uint32_t)(TPC ? 8 * TPC : src ? p.c1 : p.c0) * R * 2);
          tma_load_4d(As_s + st * p.abytes, src ? &map1 : &map0, B_full + 8u * (st), 0, grp0, 0,
                      src ? (slab ^ p.src1_xor) : slab);
          if (++st == p.stages) { st = 0; ph ^= 1; }
        }
        if constexpr (RACC) {  // previous state of this tile -> state tile it % 3 once fc0(it - 3) read it
          const int b = it % 3;
          mbar_wait(B_ta_free + 8u * b, ((it / 3) & 1) ^ 1);
          mbar_expect_tx(B_res_full + 8u * b, 7u * NRX_TILE_M * 16);
          tma_load_4d(smem_u32(smem + L.ta) + b * ta_bytes, &map1, B_res_full + 8u * b, 0, tile * (NRX_TILE_M / 16),
                      0, slab);
        }
        ++it;
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer (whole warp, elect.sync issues)
    constexpr uint32_t idesc = idesc_f16kind<ET>(NRX_TILE_M, NP);
    const int kch = p.ktap / 8;  // 16-byte channel chunks per tap
    // descriptors with a zero start address; start fields are added in 16-B units
    const uint64_t a_desc0 = smem_desc(0, (uint32_t)R * 16, 128);
    const uint64_t b_desc0 = smem_desc(smem_u32(Ws), NP * 16, 128);
    const uint32_t a_kstep = 2 * R, b_kstep = 2 * NP;  // one K=16 step
    int shifts[KS > 0 ? KS * KS : 1];                   // tap row offsets (16-B units)
    if constexpr (KS > 0) {
#pragma unroll
      for (int ta = 0; ta < KS; ++ta)
#pragma unroll
        for (int tb = 0; tb < KS; ++tb) shifts[ta * KS + tb] = (ta - KS / 2) * g.Tp + (tb - KS / 2);
    }
    // tail MLP, software-pipelined against the epilogue: in loop step i the MMA
    // warp issues conv(i), fc0(i-1) (hidden = state_tile x W0, N = thp) and
    // fc1(i-LAG) (out = relu-hidden x W1, N = top); buffers alternate by tile parity
    auto issue_fc0 = [&](int j) {
      const int b = j & 1, ta_b = j % NTA;
      const uint32_t id0 = idesc_f16kind<ET>(NRX_TILE_M, thp);
      NRX_T(tw);
      mbar_wait(B_ta_ready + 8u * ta_b, (j / NTA) & 1);
      NRX_TADD(t_c, tw);
      tc_fence_after();
      uint64_t ad = smem_desc(smem_u32(smem + L.ta + ta_b * ta_bytes), NRX_TILE_M * 16, 128);
      uint64_t bd = smem_desc(smem_u32(smem + L.tw0), thp * 16, 128);
#pragma unroll 4
      for (int kc = 0; kc < tcs / 8; kc += 2) {
        mma_bf16_warp(tmem_base + col_h + b * thp, ad, bd, id0, kc != 0);
        ad += 2 * NRX_TILE_M;
        bd += 2 * thp;
      }
      mma_commit_warp(B_hid_full + 8u * (b));
      if (RACC) mma_commit_warp(B_ta_free + 8u * ta_b);
    };
    auto issue_fc1 = [&](int j) {
      const int b = j & 1;
      const uint32_t id1 = idesc_f16kind<ET>(NRX_TILE_M, top);
      NRX_T(tw);
      mbar_wait(B_h_ready + 8u * (b), (j >> 1) & 1);
      NRX_TADD(t_d, tw);
      tc_fence_after();
      uint64_t ad = smem_desc(smem_u32(smem + L.th + (NTH == 2 ? b : 0) * th_bytes), NRX_TILE_M * 16, 128);
      uint64_t bd = smem_desc(smem_u32(smem + L.tw1), top * 16, 128);
#pragma unroll 8
      for (int kc = 0; kc < thp / 8; kc += 2) {
        mma_bf16_warp(tmem_base + col_o + b * top, ad, bd, id1, kc != 0);
        ad += 2 * NRX_TILE_M;
        bd += 2 * top;
      }
      mma_commit_warp(B_tout_full + 8u * (b));
    };
    mbar_wait(B_wbar, 0);
    tc_fence_after();
    if constexpr (RACC) {
      // the hidden bias into fc0 as well: W0's rows K = 62 / 63 (zero: pad channels of the state)
      // take b0 split into fp16 hi / lo, against the state tiles' constant ones
      for (int n = lane; n < thp; n += 32) {
        const __half bh = __float2half_rn(stb0[n]);
        const __half bl = __float2half_rn(stb0[n] - __half2float(bh));
        *reinterpret_cast<uint32_t*>(smem + L.tw0 + ((uint32_t)(7 * thp + n) * 16u + 12u)) =
            (uint32_t)__half_as_ushort(bh) | ((uint32_t)__half_as_ushort(bl) << 16);
      }
      fence_proxy_async();
      __syncwarp();
    }
    WorkIter w(g, g.NU, g.tiles, p.n_io, p.mod_order);
    int slab, tile, st = 0, it = 0;
    uint32_t ph = 0;
    while (w.next(slab, tile)) {
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      NRX_T(t0);
      mbar_wait(B_tempty + 8u * (acc), aph ^ 1);
      NRX_TADD(t_a, t0);
      tc_fence_after();
      const uint32_t d = tmem_base + acc * NP;
      if constexpr (TPC > 0) {
        // tap-pair K order: pairs (0,1) (2,3) (4,5) (6,7), then tap 8; the straddling
        // step's second half through its descriptor's leading-byte offset
        static_assert(KS == 3 && NK1 == 0 && 2 * NK0 == TPC + 1, "tap pairs: one source of TPC data chunks");
        NRX_T(t1);
        mbar_wait(B_full + 8u * (st), ph);
        NRX_TADD(t_b, t1);
        tc_fence_after();
        const uint64_t a_stage = a_desc0 + (((As_s + st * p.abytes) >> 4) + p.hup);
        int q = 0;
        auto step = [&](uint64_t a) {
          mma_bf16_warp(d, a, b_desc0 + (uint32_t)(2 * q * NP), idesc, q != 0);
          ++q;
        };
        constexpr int HALF = (TPC - 1) / 2;
#pragma unroll
        for (int pr = 0; pr < 4; ++pr) {
          const int t = 2 * pr, u = t + 1;
          const uint64_t at = a_stage + shifts[t], au = a_stage + shifts[u];
          const uint64_t lbo = (uint64_t)(uint32_t)(shifts[t] + (TPC - 1) * R - shifts[u] - R) << 16;
#pragma unroll
          for (int k = 0; k < HALF; ++k) step(at + (uint32_t)(2 * k * R));
          step(au + lbo);
#pragma unroll
          for (int k = 1; k <= HALF; ++k) step(au + (uint32_t)((2 * k - 1) * R));
        }
        const uint64_t a8 = a_stage + shifts[8];
#pragma unroll
        for (int k = 0; k < HALF; ++k) step(a8 + (uint32_t)(2 * k * R));
        step(a8 + (uint32_t)((TPC - 2) * R));  // zero-weight slot over chunk C-2, then chunk C-1
        if constexpr (RACC) {  // + previous state: its tile (chunk 7 zero) x identity, K = 64
          const int b = it % 3;
          mbar_wait(B_res_full + 8u * b, (it / 3) & 1);
          tc_fence_after();
          uint64_t ad = smem_desc(smem_u32(smem + L.ta) + b * ta_bytes, NRX_TILE_M * 16, 128);
          uint64_t bd = smem_desc(smem_u32(smem + L.ident), NP * 16, 128);
#pragma unroll
          for (int kc = 0; kc < 8; kc += 2) {
            mma_bf16_warp(d, ad, bd, idesc, 1);
            ad += 2 * NRX_TILE_M;
            bd += 2 * NP;
          }
        }
        mma_commit_warp(B_empty + 8u * (st));
        if (++st == p.stages) { st = 0; ph ^= 1; }
      } else if constexpr (KS > 0) {
        // Specialised issue: taps and K steps fully unrolled with constant
        // descriptor offsets (48 cycles per N=64 MMA, the shared-memory
        // operand floor, vs 74 for the runtime loop; scripts/mma_bench_conv_loop.cu).
#pragma unroll
        for (int src = 0; src < (NK1 > 0 ? 2 : 1); ++src) {
          NRX_T(t1);
          mbar_wait(B_full + 8u * (st), ph);
          NRX_TADD(t_b, t1);
          tc_fence_after();
          const uint64_t a_stage = a_desc0 + (((As_s + st * p.abytes) >> 4) + p.hup);
          constexpr int KCH = 2 * (NK0 + NK1);
          const int nk = src ? NK1 : NK0, kc0 = src ? 2 * NK0 : 0;
#pragma unroll
          for (int tap = 0; tap < KS * KS; ++tap) {
#pragma unroll
            for (int k = 0; k < (NK0 > NK1 ? NK0 : NK1); ++k) {
              if (k < nk)
                mma_bf16_warp(d, a_stage + shifts[tap] + (uint32_t)(k * a_kstep),
                              b_desc0 + (uint32_t)((tap * KCH + kc0 + 2 * k) * NP), idesc, (src | tap | k) != 0);
            }
          }
          mma_commit_warp(B_empty + 8u * (st));
          if (++st == p.stages) { st = 0; ph ^= 1; }
        }
      } else {
        for (int src = 0; src < (p.c1 ? 2 : 1); ++src) {
          NRX_T(t1);
          mbar_wait(B_full + 8u * (st), ph);
          NRX_TADD(t_b, t1);
          tc_fence_after();
          const uint32_t a_stage = ((As_s + st * p.abytes) >> 4) + p.hup;
          const int kc0 = src ? p.c0 / 8 : 0, nks = (src ? p.c1 : p.c0) / 16;
          uint32_t b_tap = (uint32_t)kc0 * NP;
          for (int ta = 0; ta < g.ks; ++ta) {
            for (int tb = 0; tb < g.ks; ++tb) {
              uint64_t ad = a_desc0 + (a_stage + (ta - g.r) * g.Tp + (tb - g.r));  // row-shifted view
              uint64_t bd = b_desc0 + b_tap;
              const uint32_t first = (src | ta | tb) == 0;
#pragma unroll 4
              for (int ks = 0; ks < nks; ++ks) {
                mma_bf16_warp(d, ad, bd, idesc, !(first && ks == 0));
                ad += a_kstep;
                bd += b_kstep;
              }
              b_tap += (uint32_t)kch * NP;
            }
          }
          mma_commit_warp(B_empty + 8u * (st));
          if (++st == p.stages) { st = 0; ph ^= 1; }
        }
      }
      mma_commit_warp(B_tfull + 8u * (acc));
      // earlier tiles' MLP tails run while this tile's conv MMAs execute
      if (TAIL && it >= 1) issue_fc0(it - 1);
      if (TAIL && it >= LAG) issue_fc1(it - LAG);
      ++it;
    }
    if (TAIL) {  // drain: fc0(n-1), fc1(n-LAG) .. fc1(n-1)
      if (it >= 1) issue_fc0(it - 1);
      for (int j = it - LAG > 0 ? it - LAG : 0; j < it; ++j) issue_fc1(j);
    }
  } else {  // ---------------- epilogue: warps 2 .. 2 + 4*PARTS - 1
    pdl_wait();  // reads (residual) and writes activation buffers of the previous layers
    // bf16 keeps an fp32 master of the state (dst32, STATE_INIT / RESIDUAL); fp16 has none
    constexpr bool MASTER = std::is_same<ET, __nv_bfloat16>::value;
    constexpr int PARTS = conv_parts(NP);
    constexpr int NC = NP / PARTS;  // = 16 accumulator columns per thread
    const int q = warp & 3, part = (warp - 2) >> 2;
    const int r = 32 * q + lane;
    const int cbase = part * NC;
    const int nd = p.cdst / 8, n32 = p.d4 / 4;
    const uint32_t lane_off = static_cast<uint32_t>(32 * q) << 16;
    // tiles whose tail outputs are pending: hs[k] / ht[k] = tile it-1-k (a register shift chain)
    int hs[3] = {0, 0, 0}, ht[3] = {0, 0, 0};
    const uint32_t ta_s = smem_u32(smem + L.ta), th_s = smem_u32(smem + L.th);
    const uint32_t sbias_s = smem_u32(sbias), stb0_s = smem_u32(stb0), stb1_s = smem_u32(stb1);
    // chunks holding no state channel (8 cc >= d) are the positional / zero
    // channels: constant over the iterations, written once by the state init;
    // the residual update skips them (and their zero rows in the tail's A tile)
    const int dch = (g.d + 7) / 8;
    if (TAIL && MODE == EPI_RESIDUAL && !RACC && part == PARTS - 1) {
      for (int b = 0; b < NTA; ++b)
        for (int cc = dch; cc < nd; ++cc)
          st_shared_u4(ta_s + b * ta_bytes + (uint32_t)(cc * NRX_TILE_M + r) * 16u, make_uint4(0u, 0u, 0u, 0u));
    }

    // ---- tail stage 2: hidden layer relu(state x W0 + b0) -> smem (fc1's A operand)
    auto tail_hidden = [&](int j) {
      const int b = j & 1;
      NRX_T(tw);
      mbar_wait(B_hid_full + 8u * (b), (j >> 1) & 1);
      NRX_TADD(t_d, tw);
      tc_fence_after();
      // TH[j] is free: fc1 of its previous tile (j - NTH) completed (tail_out(j + 1 - LAG) ran first)
      const uint32_t thb = th_s + (NTH == 2 ? b : 0) * th_bytes;
      auto hchunk = [&](int c8) {
        float hv[8], bb[8];
        tmem_ld8(tmem_base + lane_off + col_h + b * thp + 8 * c8, hv);
        if (!RACC) ld_shared_f8(stb0_s + 32u * c8, bb);  // RACC: b0 is in the accumulator
        tmem_wait_ld();
        if (!RACC)
#pragma unroll
          for (int e = 0; e < 8; ++e) hv[e] += bb[e];
        st_shared_u4(thb + (uint32_t)(c8 * NRX_TILE_M + r) * 16u,
                     relu_chunk(pack_chunk(hv, static_cast<const ET*>(nullptr)), static_cast<const ET*>(nullptr)));
      };
      if constexpr (TH > 0) {
        constexpr int HPP = TH / 8 / PARTS;
#pragma unroll
        for (int k = 0; k < HPP; ++k) hchunk(part * HPP + k);
      } else {
        const int hch = thp / 8, hbeg = part * hch / PARTS, hend = (part + 1) * hch / PARTS;
        for (int c8 = hbeg; c8 < hend; ++c8) hchunk(c8);
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(B_h_ready + 8u * (b));
    };
    // ---- tail stage 3: outputs of tile j (+b1): messages, or LLRs + chest
    auto tail_out = [&](int j, int jslab, int jtile) {
      const int b = j & 1;
      NRX_T(tw);
      mbar_wait(B_tout_full + 8u * (b), (j >> 1) & 1);
      NRX_TADD(t_c, tw);
      tc_fence_after();
      const int row = jtile * NRX_TILE_M + r;
      int s, t;
      row_to_st(row, g, s, t);
      const bool valid = row < g.rows_data && t < g.T;
      const uint32_t tcol = tmem_base + lane_off + col_o + b * top;
      const uint32_t vmask = valid ? 0xffffffffu : 0u;
      if (TAIL == TAIL_MSG) {  // messages of this slab, zero on pad rows/channels
        constexpr int OPP = 8 / PARTS;  // TH > 0: Ca = 64
        const int och = TH ? 8 : g.Ca / 8, obeg = TH ? part * OPP : part * och / PARTS,
                  oend = TH ? obeg + OPP : (part + 1) * och / PARTS;
        ET* const mrow = chunk_ptr(static_cast<ET*>(p.msg), jslab, och, 0, row, g);
#pragma unroll 2
        for (int cc = obeg; cc < oend; ++cc) {
          float mv[8], bb[8];
          tmem_ld8(tcol + 8 * cc, mv);
          ld_shared_f8(stb1_s + 32u * cc, bb);
          tmem_wait_ld();
          // channels >= d come out as exact zeros: zero fc1 columns and zero bias padding
#pragma unroll
          for (int e = 0; e < 8; ++e) mv[e] += bb[e];
          *reinterpret_cast<uint4*>(mrow + (size_t)cc * g.rows_slab * 8) =
              mask_chunk(pack_chunk(mv, static_cast<const ET*>(nullptr)), vmask);
        }
      } else if (part == 0) {  // LLRs (masked width) + planar-decoded chest
        float o[32];
        tmem_ld16(tcol, o);
        tmem_ld16(tcol + 16, o + 16);
        tmem_wait_ld();
        if (valid) {
          uint32_t bad = 0;
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            o[c] += stb1[c];
            bad |= (__float_as_uint(o[c]) & 0x7f800000u) == 0x7f800000u;
          }
          if (bad && g.flag) atomicOr(g.flag, 1u);
          const int mio = io_index(p.mod_order, jslab, g);
          const int width = mio < 0 ? 0 : g.io_width[mio];
          const size_t re = ((size_t)jslab * g.S + s) * g.T + t;
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
            for (int bb = 0; bb < 8; ++bb)
              if (bb < g.B) cf[2 * bb] = o[8 + bb];
#pragma unroll
            for (int c = 9; c < 24; ++c) {
              const int bb = c - 8 - g.B;  // imaginary part of antenna bb
              if (bb >= 0 && bb < g.B) cf[2 * bb + 1] = o[c];
            }
          }
        }
      }
      tc_fence_before();
    };

    WorkIter w(g, g.NU, g.tiles, p.n_io, p.mod_order);
    int slab, tile, it = 0;
    // residual: the previous state of the next tile (fp16: the state buffer
    // itself; bf16: the fp32 master) is loaded while this tile is processed
    // (each row is read and rewritten only by its own thread)
    constexpr bool PREF = MODE == EPI_RESIDUAL && !RACC;  // RACC: the residual is in the accumulator
    WorkIter wp = w;
    uint4 nraw[PREF && !MASTER ? NC / 8 : 1];
    float4 nold[PREF && MASTER ? NC / 4 : 1];
    auto load_res = [&](int sl, int tl) {
      const int prow = tl * NRX_TILE_M + r;
      int ps, pt;
      row_to_st(prow, g, ps, pt);
      const bool pv = prow < g.rows_data && pt < g.T;
      if constexpr (MASTER) {
        const float4* src = reinterpret_cast<const float4*>(chunk_ptr(p.dst32, sl, n32, cbase / 4, prow, g));
#pragma unroll
        for (int c4 = 0; c4 < NC / 4; ++c4)
          nold[c4] = (pv && cbase / 4 + c4 < n32) ? src[(size_t)c4 * g.rows_slab] : make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        const uint4* src = reinterpret_cast<const uint4*>(chunk_ptr(dst, sl, nd, cbase / 8, prow, g));
#pragma unroll
        for (int c8 = 0; c8 < NC / 8; ++c8)
          nraw[c8] = (pv && cbase / 8 + c8 < dch) ? src[(size_t)c8 * g.rows_slab] : make_uint4(0u, 0u, 0u, 0u);
      }
    };
    if (PREF) {
      int sl, tl;
      if (wp.next(sl, tl)) load_res(sl, tl);
    }
    while (w.next(slab, tile)) {
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      const int row = tile * NRX_TILE_M + r;
      int s, t;
      row_to_st(row, g, s, t);
      const bool valid = row < g.rows_data && t < g.T;
      float old[MASTER ? NC : 1];
      uint4 raw[MASTER ? 1 : NC / 8];
      if (PREF) {
        if constexpr (MASTER) {
#pragma unroll
          for (int c4 = 0; c4 < NC / 4; ++c4) {
            old[4 * c4 + 0] = nold[c4].x;
            old[4 * c4 + 1] = nold[c4].y;
            old[4 * c4 + 2] = nold[c4].z;
            old[4 * c4 + 3] = nold[c4].w;
          }
        } else {
#pragma unroll
          for (int c8 = 0; c8 < NC / 8; ++c8) raw[c8] = nraw[c8];
        }
        int sl, tl;
        if (wp.next(sl, tl)) load_res(sl, tl);
      }
      NRX_T(t0);
      mbar_wait(B_tfull + 8u * (acc), aph);
      NRX_TADD(t_a, t0);
      NRX_T(t1);
      tc_fence_after();
      float v[NC];
      const uint32_t taddr = tmem_base + lane_off + acc * NP + cbase;
#pragma unroll
      for (int c = 0; c < NC / 8; ++c) tmem_ld8(taddr + 8 * c, v + 8 * c);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive_relaxed(B_tempty + 8u * (acc));

      // positional channels only where a written chunk holds them
      const int clo = cbase / 8, chi = cbase / 8 + NC / 8;
      const bool need_pos = MODE != EPI_RELU && valid && (MODE != EPI_RESIDUAL || g.d % 8 != 0) &&
                            ((g.d / 8 >= clo && g.d / 8 < chi) || ((g.d + 1) / 8 >= clo && (g.d + 1) / 8 < chi));
      const float pdt = need_pos ? sdt[t] : 0.f;
      const float pdf = need_pos ? pos_df(s, slab % g.U, g) : 0.f;
      ET* const drow = chunk_ptr(dst, slab, nd, 0, row, g);
      const uint32_t vmask = valid ? 0xffffffffu : 0u;
      const size_t dcs = (size_t)g.rows_slab * 8;  // chunk stride of a half-precision buffer
#pragma unroll
      for (int c8 = 0; c8 < NC / 8; ++c8) {  // one 8-channel chunk at a time (few live registers)
        const int cc = cbase / 8 + c8;
        if (MODE == EPI_RESIDUAL && cc >= dch) continue;   // constant positional / zero chunk
        float o8[8], bb[8];
        if (PREF && !MASTER) unpack_chunk(raw[c8], static_cast<const ET*>(nullptr), o8);
        if (!RACC) ld_shared_f8(sbias_s + 32u * cc, bb);
        float* x = v + 8 * c8;
        const bool full = 8 * cc + 8 <= g.d;  // warp-uniform
        if (!MASTER && full) {  // fast path: pack, then ReLU / pad-row mask on the packed words
#pragma unroll
          for (int e = 0; e < 8; ++e) x[e] = PREF ? o8[e] + (x[e] + bb[e]) : RACC ? x[e] : x[e] + bb[e];
          uint4 qx = pack_chunk(x, static_cast<const ET*>(nullptr));
          if (MODE == EPI_RELU) qx = relu_chunk(qx, static_cast<const ET*>(nullptr));
          qx = mask_chunk(qx, vmask);
          *reinterpret_cast<uint4*>(drow + cc * dcs) = qx;
          if (TAIL) st_shared_u4(ta_s + (it % NTA) * ta_bytes + (uint32_t)(cc * NRX_TILE_M + r) * 16u, qx);
          continue;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          float y = RACC ? x[e] : x[e] + bb[e];  // conv + bias first, as the reference adds them (RACC: in the accumulator)
          if (MODE == EPI_RELU) y = relu_f(y);
          if (PREF) y = (MASTER ? old[8 * c8 + e] : o8[e]) + y;
          x[e] = (valid && (full || 8 * cc + e < g.d)) ? y : 0.f;
        }
        if (MODE != EPI_RELU) {
          if (MASTER) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (2 * cc + h < n32) store_chunk(chunk_ptr(p.dst32, slab, n32, 2 * cc + h, row, g), x + 4 * h);
          }
          if (!full) {  // positional channels d, d+1 of the half-precision operand copy
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int c = 8 * cc + e;
              if (valid && c == g.d) x[e] = pdt;
              if (valid && c == g.d + 1) x[e] = pdf;
            }
          }
        }
        if (cc < nd) {
          const uint4 qx = pack_chunk(x, static_cast<const ET*>(nullptr));
          *reinterpret_cast<uint4*>(drow + cc * dcs) = qx;
          if (TAIL) st_shared_u4(ta_s + (it % NTA) * ta_bytes + (uint32_t)(cc * NRX_TILE_M + r) * 16u, qx);
        }
      }
      if (part == PARTS - 1) {  // buffer channels beyond the accumulator: positional / zero only
        for (int cc = NP / 8; cc < nd; ++cc) {
          float o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            o[e] = (valid && MODE != EPI_RELU) ? state_extra(8 * cc + e, s, t, slab % g.U, g) : 0.f;
          store_chunk(chunk_ptr(dst, slab, nd, cc, row, g), o);
          if (TAIL) st_shared_u4(ta_s + (it % NTA) * ta_bytes + (uint32_t)(cc * NRX_TILE_M + r) * 16u,
                                 pack_chunk(o, static_cast<const ET*>(nullptr)));
        }
      }
      if (TAIL) {
        fence_proxy_async();  // state tile (generic-proxy stores) -> tensor-core reads
        tc_fence_before();
        mbar_arrive(B_ta_ready + 8u * (it % NTA));
        // pipelined tail stages: outputs of tile it-LAG (frees its hidden
        // tile), then the hidden layer of tile it-1
        if (it >= LAG) tail_out(it - LAG, hs[LAG - 1], ht[LAG - 1]);
        if (it >= 1) tail_hidden(it - 1);
        hs[2] = hs[1];
        ht[2] = ht[1];
        hs[1] = hs[0];
        ht[1] = ht[0];
        hs[0] = slab;
        ht[0] = tile;
      }
      NRX_TADD(t_b, t1);
      ++it;
    }
    if (TAIL) {  // drain, mirroring the MMA warp
      if (it >= LAG) tail_out(it - LAG, hs[LAG - 1], ht[LAG - 1]);
      if (it >= 1) tail_hidden(it - 1);
#pragma unroll
      for (int k = LAG - 2; k >= 0; --k)  // tiles it-1-k, oldest first
        if (it - 1 - k >= 0) tail_out(it - 1 - k, hs[k], ht[k]);
    }
  }
#ifdef NRX_TIMING
  if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x == 0 || threadIdx.x == 32 || threadIdx.x == 64))
    printf("conv NP=%d mode=%d tail=%d c0=%d c1=%d tid=%d all=%lld a=%lld b=%lld c=%lld d=%lld\n", NP, MODE, TAIL,
           p.c0, p.c1, threadIdx.x, clock64() - t_all, t_a, t_b, t_c, t_d);
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}

using KFn = void (*)(const ConvTcParams, const CUtensorMap, const CUtensorMap);

template <typename ET, int TAIL>
static KFn select_conv_tail(const Geom& g, int np, int mode, int c0, int c1, int tpc, bool rt) {
  static const KFn table[4][3] = {
      {k_conv_tc<ET, 16, 0, TAIL>, k_conv_tc<ET, 16, 1, TAIL>, k_conv_tc<ET, 16, 2, TAIL>},
      {k_conv_tc<ET, 32, 0, TAIL>, k_conv_tc<ET, 32, 1, TAIL>, k_conv_tc<ET, 32, 2, TAIL>},
      {k_conv_tc<ET, 48, 0, TAIL>, k_conv_tc<ET, 48, 1, TAIL>, k_conv_tc<ET, 48, 2, TAIL>},
      {k_conv_tc<ET, 64, 0, TAIL>, k_conv_tc<ET, 64, 1, TAIL>, k_conv_tc<ET, 64, 2, TAIL>}};
  KFn fn = table[np / 16 - 1][mode];
  // fully unrolled issue for the 3x3 layers of d_s in (48, 64] (the RT / large models)
  if (g.ks == 3 && np == 64) {
    const int nk0 = c0 / 16, nk1 = c1 / 16;
    if (TAIL == TAIL_NONE && mode == EPI_RELU && nk0 == 2 && nk1 == 0)
      fn = tpc == 3 ? k_conv_tc<ET, 64, EPI_RELU, TAIL, 3, 2, 0, 3> : k_conv_tc<ET, 64, EPI_RELU, TAIL, 3, 2, 0>;
    if (TAIL == TAIL_NONE && mode == EPI_RELU && nk0 == 4 && nk1 == 4) fn = k_conv_tc<ET, 64, EPI_RELU, TAIL, 3, 4, 4>;
    // compile-time RT tail shape (rt); TAIL_NONE has no tail (TH = 0 twice)
    constexpr int TH = TAIL == TAIL_MSG ? 64 : TAIL == TAIL_READOUT ? 128 : 0;
    if (TAIL != TAIL_READOUT && mode == EPI_STATE_INIT && nk0 == 4 && nk1 == 0)
      fn = tpc == 7 ? (rt ? k_conv_tc<ET, 64, EPI_STATE_INIT, TAIL, 3, 4, 0, 7, TH>
                          : k_conv_tc<ET, 64, EPI_STATE_INIT, TAIL, 3, 4, 0, 7>)
                    : k_conv_tc<ET, 64, EPI_STATE_INIT, TAIL, 3, 4, 0>;
    if (mode == EPI_RESIDUAL && nk0 == 4 && nk1 == 0)
      fn = tpc == 7 ? (rt ? k_conv_tc<ET, 64, EPI_RESIDUAL, TAIL, 3, 4, 0, 7, TH>
                          : k_conv_tc<ET, 64, EPI_RESIDUAL, TAIL, 3, 4, 0, 7>)
                    : k_conv_tc<ET, 64, EPI_RESIDUAL, TAIL, 3, 4, 0>;
  }
  return fn;
}

template <typename ET>
static KFn select_conv(const Geom& g, int np, int mode, int tail, int c0, int c1, int tpc, bool rt) {
  if (tail == TAIL_MSG) return select_conv_tail<ET, TAIL_MSG>(g, np, mode, c0, c1, tpc, rt);
  if (tail == TAIL_READOUT) return select_conv_tail<ET, TAIL_READOUT>(g, np, mode, c0, c1, tpc, rt);
  return select_conv_tail<ET, TAIL_NONE>(g, np, mode, c0, c1, tpc, false);
}

static bool racc_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("NRX_RACC");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

struct ConvLaunch {
  const ConvOff* offs;
  int n_off;
  const void* src0;
  int c0;
  const void* src1;
  int c1;
  int src1_xor;
  void* dst;
  int cdst;
  float* dst32;
  int mode;
  int tail;             // ConvTail
  const MlpOff* tail_w;  // per IO set (readout) or one (message MLP)
  int tail_n;
  void* msg;
  float* llr;
  float2* chest;
};

static int launch_conv(const Geom& g, const ConvLaunch& c, const uint8_t* wb, const int32_t* mod_order,
                       cudaStream_t st) {
  ConvTcParams p{};
  p.g = g;
  p.ktap = c.c0 + c.c1;
  p.c0 = c.c0;
  p.c1 = c.c1;
  p.src1_xor = c.src1_xor;
  p.np = rup(g.d, 16);
  p.cdst = c.cdst;
  p.mode = c.mode;
  p.n_io = c.tail == TAIL_READOUT ? c.tail_n : c.n_off;
  p.d4 = rup(g.d, 4);
  // rows per channel chunk in shared memory: the tile plus the halo rounded
  // up to the 16-row TMA granule on both sides (also keeps chunks 256-B aligned)
  p.hup = rup(g.H, 16);
  p.rbox = NRX_TILE_M + 2 * p.hup;
  p.wbytes = (uint32_t)(g.ks * g.ks * p.ktap * p.np * 2);
  p.abytes = (uint32_t)((c.c0 > c.c1 ? c.c0 : c.c1) * p.rbox * 2);  // one source per stage
  p.wbase = wb;
  for (int i = 0; i < p.n_io; ++i) {
    const int k = c.n_off > 1 ? i : 0;  // conv weights: per IO set for the var_io state init only
    p.w_off[i] = c.offs[k].w;
    p.b_off[i] = c.offs[k].b;
  }
  p.mod_order = mod_order;
  p.dst = c.dst;
  p.dst32 = c.dst32;
  if (c.tail) {
    const int hp = rup(g.h, 16);
    p.thp = c.tail == TAIL_MSG ? hp : 2 * hp;
    p.top = c.tail == TAIL_MSG ? rup(g.d, 16) : 32;
    p.tw0bytes = (uint32_t)(g.Cs * p.thp * 2);
    p.tw1bytes = (uint32_t)(p.thp * p.top * 2);
    for (int i = 0; i < p.n_io; ++i) {
      const MlpOff& m = c.tail_w[c.tail_n > 1 ? i : 0];
      p.tw0[i] = m.w0;
      p.tb0[i] = m.b0;
      p.tw1[i] = m.w1;
      p.tb1[i] = m.b1;
    }
    p.msg = c.msg;
    p.llr = c.llr;
    p.chest = c.chest;
    if (p.thp > 256 || p.top > 64) return NRX_ERR_UNSUPPORTED;
  }
  const uint32_t cols = 2 * p.np + (c.tail ? 2 * (p.thp + p.top) : 0);
  p.tmem_cols = cols <= 32 ? 32 : cols <= 64 ? 64 : cols <= 128 ? 128 : cols <= 256 ? 256 : 512;
  if (cols > 512) return NRX_ERR_UNSUPPORTED;
  // tap-pair layers (tp2_chunks; the packer wrote their weights in that K order): state_init.conv0
  // over the feature chunks, the conv1 layers over h; only their data chunks are loaded
  int tpc = 0;
  if (c.c1 == 0 && p.np == 64) {
    if (c.mode == EPI_RELU && c.c0 == g.Cf && tp2_chunks(g.d, g.ks, g.prec, c.c0, g.Cin) == 3) tpc = 3;
    if (c.mode != EPI_RELU && c.c0 == g.Ch && tp2_layer(g.d, g.ks, g.prec)) tpc = 7;
  }
  // the RT tail shape (message: hidden 64 -> 64; readout: hidden 128 -> 32) as compile-time sizes
  bool rt = tpc == 7 && g.Cs == 64 && g.Ca == 64 && g.ks == 3 &&
            ((c.tail == TAIL_MSG && p.thp == 64 && p.top == 64) || (c.tail == TAIL_READOUT && p.thp == 128));
  // fp16 residual update with the RT tail: the residual through the accumulator (conv_racc;
  // NRX_RACC=0 selects the epilogue residual add instead, for A/B runs)
  p.racc = rt && g.prec == NRX_FP16 && c.mode == EPI_RESIDUAL && g.d == 56;
  if (p.racc && !racc_enabled()) rt = false, p.racc = 0;
  auto fit = [&]() {  // pipeline stages that fit next to the resident weights (at least 2)
    int stages = 8;
    p.stages = stages;
    while (stages > 2 && conv_smem_layout(p, c.tail).total > SMEM_LIMIT) p.stages = --stages;
    return conv_smem_layout(p, c.tail).total <= SMEM_LIMIT;
  };
  bool fits = fit();
  if (p.racc && !fits) {  // the third state tile + identity do not fit next to two stages: epilogue add
    p.racc = 0;
    rt = false;
    fits = fit();
  }
  if (!fits || p.rbox > 256) return NRX_ERR_UNSUPPORTED;
  const size_t smem = conv_smem_layout(p, c.tail).total;
  CUtensorMap m0, m1;
  int rc = make_map(&m0, c.src0, g, c.c0, p.rbox, tpc);
  if (rc) return rc;
  if (p.racc)  // source 1 = the previous state: 128-row tiles of its 7 state chunks, no halo
    rc = make_map(&m1, c.dst, g, c.cdst, NRX_TILE_M, 7);
  else
    rc = make_map(&m1, c.src1 ? c.src1 : c.src0, g, c.c1 ? c.c1 : c.c0, p.rbox);
  if (rc) return rc;
  if (p.np % 16 || p.np < 16 || p.np > 64 || c.mode < 0 || c.mode > 2) return NRX_ERR_UNSUPPORTED;
  const KFn fn = g.prec == NRX_FP16 ? select_conv<__half>(g, p.np, c.mode, c.tail, c.c0, c.c1, tpc, rt)
                                    : select_conv<__nv_bfloat16>(g, p.np, c.mode, c.tail, c.c0, c.c1, tpc, rt);
  if (set_smem((const void*)fn, SMEM_LIMIT)) return NRX_ERR_CUDA;
  const int total = g.NU * g.tiles;
  dim3 grid(total < num_sms() ? total : num_sms(), p.n_io);
  if (launch_pdl(fn, grid, dim3(conv_threads(p.np)), smem, st, p, m0, m1) != cudaSuccess) return NRX_ERR_CUDA;
  return cudaPeekAtLastError() == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

}  // namespace tc

#define NRX_TRY_TC(x)            \
  do {                           \
    int _s = (x);                \
    if (_s != NRX_OK) return _s; \
  } while (0)

int launch_msg(const Geom& g, const PackLayout& L, const uint8_t* wb, const void* state, void* agg,
               cudaStream_t st);
int launch_readout(const Geom& g, const PackLayout& L, const uint8_t* wb, const void* state,
                   const int32_t* mod_order, float* llr, float2* chest, cudaStream_t st);

// U = 2: message MLP fused into every conv1, partner-slab messages as the
// update conv's second source; any U: readout fused into the last conv1.
bool tc_fused_messages(const Geom& g) { return g.U == 2; }

static bool pair16_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("NRX_PAIR16");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

int launch_forward_tc(const Geom& g, const PackLayout& L, const WsLayout& W, int n_it, const uint8_t* wb,
                      const int32_t* mod_order, uint8_t* ws, float* llr, float2* chest, cudaStream_t st) {
  using namespace tc;
  if (g.d > 64 || g.h > 128) return NRX_ERR_UNSUPPORTED;
  void* feats = ws + W.feats;
  void* h = ws + W.h;
  void* state = ws + W.state;
  void* agg = ws + W.agg;  // aggregate (U != 2) or own-slab messages (U = 2)
  // bf16 keeps an fp32 copy of the residual state stream; fp16 updates the state in place
  float* state32 = g.prec == NRX_BF16 ? reinterpret_cast<float*>(ws + W.state32) : nullptr;
  const bool fused = tc_fused_messages(g);

  // update.conv0 (tail-less ReLU) on CTA pairs when the blob carries the pair
  // copies (np 32 / 64); NRX_PAIR16=0 keeps it single-CTA
  const bool pair = L.upd0p.w != 0 && pair16_enabled();
  auto relu_layer = [&](const ConvLaunch& c1, const ConvOff* pair_offs) -> int {
    if (!pair) return launch_conv(g, c1, wb, mod_order, st);
    ConvX3Launch x{};
    x.offs = pair_offs;
    x.n_off = c1.n_off;
    x.src0 = c1.src0;
    x.c0 = c1.c0;
    x.src1 = c1.src1;
    x.c1 = c1.c1;
    x.src1_xor = c1.src1_xor;
    x.dst = c1.dst;
    x.cdst = c1.cdst;
    x.mode = EPI_RELU;
    x.prec = g.prec;
    const int rc = launch_conv_x3(g, x, wb, mod_order, st);
    return rc == NRX_ERR_UNSUPPORTED ? launch_conv(g, c1, wb, mod_order, st) : rc;
  };
  ConvLaunch c{};
  c.offs = L.init0;
  c.n_off = g.n_io;
  c.src0 = feats;
  c.c0 = g.Cf;
  c.dst = h;
  c.cdst = g.Ch;
  c.mode = EPI_RELU;
  {
    // state_init.conv0 (K = 32) stays single-CTA: its pair version is slower (0.160 vs 0.138 ms / 32 slots)
    ProfScope ps(KID_INIT0, st);
    NRX_TRY_TC(launch_conv(g, c, wb, mod_order, st));
  }
  c = ConvLaunch{};
  c.offs = L.init1;
  c.n_off = g.n_io;
  c.src0 = h;
  c.c0 = g.Ch;
  c.dst = state;
  c.cdst = g.Cs;
  c.dst32 = state32;
  c.mode = EPI_STATE_INIT;
  if (fused) {
    c.tail = TAIL_MSG;
    c.tail_w = &L.msg;
    c.tail_n = 1;
    c.msg = agg;
  }
  {
    ProfScope ps(KID_INIT1, st);
    NRX_TRY_TC(launch_conv(g, c, wb, mod_order, st));
  }
  for (int it = 0; it < n_it; ++it) {
    if (!fused) {
      ProfScope ps(KID_MSG, st);
      NRX_TRY_TC(launch_msg(g, L, wb, state, agg, st));
    }
    c = ConvLaunch{};
    c.offs = &L.upd0;
    c.n_off = 1;
    c.src0 = state;
    c.c0 = g.Cs;
    c.src1 = agg;
    c.c1 = g.Ca;
    c.src1_xor = fused ? 1 : 0;  // U = 2: the partner UE's messages are the aggregate
    c.dst = h;
    c.cdst = g.Ch;
    c.mode = EPI_RELU;
    {
      ProfScope ps(KID_UPD0, st);
      NRX_TRY_TC(relu_layer(c, &L.upd0p));
    }
    const bool last = it + 1 == n_it;
    c = ConvLaunch{};
    c.offs = &L.upd1;
    c.n_off = 1;
    c.src0 = h;
    c.c0 = g.Ch;
    c.dst = state;
    c.cdst = g.Cs;
    c.dst32 = state32;
    c.mode = EPI_RESIDUAL;
    if (last) {
      c.tail = TAIL_READOUT;
      c.tail_w = L.llr;
      c.tail_n = g.n_io;
      c.llr = llr;
      c.chest = chest;
    } else if (fused) {
      c.tail = TAIL_MSG;
      c.tail_w = &L.msg;
      c.tail_n = 1;
      c.msg = agg;
    }
    ProfScope ps(KID_UPD1, st);
    NRX_TRY_TC(launch_conv(g, c, wb, mod_order, st));
  }
  return NRX_OK;
}

int tc_launch_count(int n_it, int num_ues) { return 2 + (num_ues == 2 ? 2 : 3) * n_it; }

}  // namespace nrx
