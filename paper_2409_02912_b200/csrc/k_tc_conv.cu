// bf16 tensor-core convolution (NRX_BF16 path) and the launch sequence of
// the tensor-core forward pass.
//
//  k_conv_tc     k x k 'same' convolution as an implicit GEMM on the
//                row-linearised grid (nrx_internal.h).  Per 128-row M tile the
//                producer warp TMA-loads the tile plus +-H halo rows of every
//                input channel chunk ONCE per input source (4-D box
//                {8, 128+2H, C/8, 1}, zero filled outside the slab); tap (a,b)
//                is the same shared-memory tile viewed at a row offset
//                (a-r)*Tp + (b-r), which the no-swizzle K-major UMMA descriptor
//                addresses directly (16-byte granular start address).  The whole
//                layer's weights stay resident in shared memory (bulk copy once
//                per CTA).  One thread issues taps * C/16 MMAs (M=128,
//                N=rup(d,16), K=16) into one of two TMEM accumulators; eight
//                epilogue warps drain the other (tcgen05.ld) and apply bias /
//                ReLU / positional channels / fp32 residual while the next
//                tile's MMAs run.
#include "nrx_profile.h"
#include "tc_common.cuh"

namespace nrx {
namespace tc {

// ---------------------------------------------------------------------------
// K2/K3b/K3c: convolution
// ---------------------------------------------------------------------------

struct ConvTcParams {
  Geom g;
  int ktap, c0, c1;     // A channels per tap = c0 (source 0) + c1 (source 1)
  int np, cdst, mode, stages;
  int n_io, d4;
  uint32_t wbytes, abytes, tmem_cols, rbox;
  int hup;              // halo rows loaded on each side (H rounded up to 16)
  const uint8_t* wbase;
  uint64_t w_off[NRX_MAX_IO], b_off[NRX_MAX_IO];
  const int32_t* mod_order;
  void* dst;            // bf16 / fp16 output buffer (element type = kernel's ET)
  float* dst32;         // fp32 master state (bf16 STATE_INIT / RESIDUAL), or null
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

// KS > 0 selects the fully unrolled MMA issue for kernel size KS with NK0 /
// NK1 K=16 steps per tap from source 0 / 1 (host picks it when the layer
// matches); KS = 0 is the generic runtime-loop version.
// ET = __nv_bfloat16 or __half: operand/activation element type.
template <typename ET, int NP, int MODE, int KS = 0, int NK0 = 0, int NK1 = 0>
__global__ void __launch_bounds__(CONV_THREADS, 1)
    k_conv_tc(const __grid_constant__ ConvTcParams p, const __grid_constant__ CUtensorMap map0,
              const __grid_constant__ CUtensorMap map1) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const Geom& g = p.g;
  ET* const dst = static_cast<ET*>(p.dst);
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
#ifdef NRX_TIMING
  long long t_a = 0, t_b = 0, t_c = 0, t_all = clock64();
#endif

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      load_weights(Ws, p.wbase + p.w_off[io], p.wbytes, wbar);
      // one pipeline stage per (tile, input source): finer-grained stages keep
      // more loads in flight next to the resident weights
      WorkIter w(g, g.NU, g.tiles, p.n_io, p.mod_order);
      int slab, tile, st = 0;
      uint32_t ph = 0;
      while (w.next(slab, tile)) {
        const int grp0 = (tile * NRX_TILE_M - p.hup) / 16;  // 16-row groups
        for (int src = 0; src < (p.c1 ? 2 : 1); ++src) {
          NRX_T(t0);
          mbar_wait(&empty[st], ph ^ 1);
          NRX_TADD(t_a, t0);
          mbar_expect_tx(&full[st], (uint32_t)(src ? p.c1 : p.c0) * R * 2);
          tma_load_4d(As + (size_t)st * p.abytes, src ? &map1 : &map0, &full[st], 0, grp0, 0, slab);
          if (++st == p.stages) { st = 0; ph ^= 1; }
        }
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
    mbar_wait(wbar, 0);
    tc_fence_after();
    WorkIter w(g, g.NU, g.tiles, p.n_io, p.mod_order);
    int slab, tile, st = 0, it = 0;
    uint32_t ph = 0;
    while (w.next(slab, tile)) {
      const int acc = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      NRX_T(t0);
      mbar_wait(&tempty[acc], aph ^ 1);
      NRX_TADD(t_a, t0);
      tc_fence_after();
      const uint32_t d = tmem_base + acc * NP;
      if constexpr (KS > 0) {
        // Specialised issue: taps and K steps fully unrolled with constant
        // descriptor offsets (48 cycles per N=64 MMA, the shared-memory
        // operand floor, vs 74 for the runtime loop; scripts/mma_bench_conv_loop.cu).
#pragma unroll
        for (int src = 0; src < (NK1 > 0 ? 2 : 1); ++src) {
          NRX_T(t1);
          mbar_wait(&full[st], ph);
          NRX_TADD(t_b, t1);
          tc_fence_after();
          const uint64_t a_stage = a_desc0 + ((smem_u32(As + (size_t)st * p.abytes) >> 4) + p.hup);
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
          mma_commit_warp(&empty[st]);
          if (++st == p.stages) { st = 0; ph ^= 1; }
        }
      } else {
        for (int src = 0; src < (p.c1 ? 2 : 1); ++src) {
          NRX_T(t1);
          mbar_wait(&full[st], ph);
          NRX_TADD(t_b, t1);
          tc_fence_after();
          const uint32_t a_stage = (smem_u32(As + (size_t)st * p.abytes) >> 4) + p.hup;
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
          mma_commit_warp(&empty[st]);
          if (++st == p.stages) { st = 0; ph ^= 1; }
        }
      }
      mma_commit_warp(&tfull[acc]);
      ++it;
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
      NRX_T(t0);
      mbar_wait(&tfull[acc], aph);
      NRX_TADD(t_a, t0);
      NRX_T(t1);
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
      if (MODE == EPI_RESIDUAL) {  // residual input: issue every load before use
        if (p.dst32) {             // bf16 path: fp32 residual stream
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
        } else {                   // fp16 path: the state buffer itself
          uint4 raw[NC / 8];
#pragma unroll
          for (int c8 = 0; c8 < NC / 8; ++c8) {
            const int cc = cbase / 8 + c8;
            raw[c8] = (valid && cc < nd) ? *reinterpret_cast<const uint4*>(chunk_ptr(dst, slab, nd, cc, row, g))
                                         : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
          for (int c8 = 0; c8 < NC / 8; ++c8) unpack_chunk(raw[c8], static_cast<const ET*>(nullptr), old + 8 * c8);
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
        if (p.dst32) {
#pragma unroll
          for (int c4 = 0; c4 < NC / 4; ++c4) {
            const int cc = cbase / 4 + c4;
            if (cc < n32) store_chunk(chunk_ptr(p.dst32, slab, n32, cc, row, g), x + 4 * c4);
          }
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
        if (cc < nd) store_chunk(chunk_ptr(dst, slab, nd, cc, row, g), x + 8 * c8);
      }
      if (half == 1) {  // buffer channels beyond the accumulator: positional / zero only
        for (int cc = NP / 8; cc < nd; ++cc) {
          float o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            o[e] = (valid && MODE != EPI_RELU) ? state_extra(8 * cc + e, s, t, slab % g.U, g) : 0.f;
          store_chunk(chunk_ptr(dst, slab, nd, cc, row, g), o);
        }
      }
      NRX_TADD(t_b, t1);
      ++it;
    }
  }
#ifdef NRX_TIMING
  if (blockIdx.x == 0 && blockIdx.y == 0 && (threadIdx.x == 0 || threadIdx.x == 32 || threadIdx.x == 64))
    printf("conv NP=%d mode=%d c0=%d c1=%d tid=%d all=%lld a=%lld b=%lld c=%lld\n", NP, MODE, p.c0, p.c1,
           threadIdx.x, clock64() - t_all, t_a, t_b, t_c);
#endif
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, p.tmem_cols);
  }
}


using KFn = void (*)(const ConvTcParams, const CUtensorMap, const CUtensorMap);

template <typename ET>
static KFn select_conv(const Geom& g, int np, int mode, int c0, int c1) {
  static const KFn table[4][3] = {
      {k_conv_tc<ET, 16, 0>, k_conv_tc<ET, 16, 1>, k_conv_tc<ET, 16, 2>},
      {k_conv_tc<ET, 32, 0>, k_conv_tc<ET, 32, 1>, k_conv_tc<ET, 32, 2>},
      {k_conv_tc<ET, 48, 0>, k_conv_tc<ET, 48, 1>, k_conv_tc<ET, 48, 2>},
      {k_conv_tc<ET, 64, 0>, k_conv_tc<ET, 64, 1>, k_conv_tc<ET, 64, 2>}};
  KFn fn = table[np / 16 - 1][mode];
  // fully unrolled issue for the 3x3 layers of d_s in (48, 64] (the RT / large models)
  if (g.ks == 3 && np == 64) {
    const int nk0 = c0 / 16, nk1 = c1 / 16;
    if (mode == EPI_RELU && nk0 == 2 && nk1 == 0) fn = k_conv_tc<ET, 64, EPI_RELU, 3, 2, 0>;
    if (mode == EPI_RELU && nk0 == 4 && nk1 == 4) fn = k_conv_tc<ET, 64, EPI_RELU, 3, 4, 4>;
    if (mode == EPI_STATE_INIT && nk0 == 4 && nk1 == 0) fn = k_conv_tc<ET, 64, EPI_STATE_INIT, 3, 4, 0>;
    if (mode == EPI_RESIDUAL && nk0 == 4 && nk1 == 0) fn = k_conv_tc<ET, 64, EPI_RESIDUAL, 3, 4, 0>;
  }
  return fn;
}

static int launch_conv(const Geom& g, const PackLayout& L, const ConvOff* offs, int n_off, const void* src0,
                       int c0, const void* src1, int c1, void* dst, int cdst, float* dst32, int mode,
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
  // rows per channel chunk in shared memory: the tile plus the halo rounded
  // up to the 16-row TMA granule on both sides (also keeps chunks 256-B aligned)
  p.hup = rup(g.H, 16);
  p.rbox = NRX_TILE_M + 2 * p.hup;
  p.wbytes = (uint32_t)(g.ks * g.ks * p.ktap * p.np * 2);
  p.abytes = (uint32_t)((c0 > c1 ? c0 : c1) * p.rbox * 2);  // one source per stage
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
  int stages = 8;
  while (stages > 2 && fixed + (size_t)stages * p.abytes > SMEM_LIMIT) --stages;
  if (fixed + (size_t)stages * p.abytes > SMEM_LIMIT || p.rbox > 256) return NRX_ERR_UNSUPPORTED;
  p.stages = stages;
  const size_t smem = fixed + (size_t)stages * p.abytes;
  CUtensorMap m0, m1;
  int rc = make_map(&m0, src0, g, c0, p.rbox);
  if (rc) return rc;
  rc = make_map(&m1, src1 ? src1 : src0, g, c1 ? c1 : c0, p.rbox);
  if (rc) return rc;
  if (p.np % 16 || p.np < 16 || p.np > 64 || mode < 0 || mode > 2) return NRX_ERR_UNSUPPORTED;
  const KFn fn = g.prec == NRX_FP16 ? select_conv<__half>(g, p.np, mode, c0, c1)
                                    : select_conv<__nv_bfloat16>(g, p.np, mode, c0, c1);
  if (set_smem((const void*)fn, SMEM_LIMIT)) return NRX_ERR_CUDA;
  const int total = g.NU * g.tiles;
  dim3 grid(total < num_sms() ? total : num_sms(), n_off);
  fn<<<grid, CONV_THREADS, smem, st>>>(p, m0, m1);
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

int launch_forward_tc(const Geom& g, const PackLayout& L, const WsLayout& W, int n_it, const uint8_t* wb,
                      const int32_t* mod_order, uint8_t* ws, float* llr, float2* chest, cudaStream_t st) {
  using namespace tc;
  if (g.d > 64 || g.h > 128) return NRX_ERR_UNSUPPORTED;
  void* feats = ws + W.feats;
  void* h = ws + W.h;
  void* state = ws + W.state;
  void* agg = ws + W.agg;
  // bf16 keeps an fp32 copy of the residual state stream; fp16 updates the state in place
  float* state32 = g.prec == NRX_BF16 ? reinterpret_cast<float*>(ws + W.state32) : nullptr;
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
