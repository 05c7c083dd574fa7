// Training convolutions on the tensor cores at fp32 accuracy (SURVEY.md
// §8(f) row 3; the reference: autodiff.py:302-350 conv2d and its VJPs).
//
// Each of the three convolution operators of a training step is one GEMM
//   fwd    y  [p][o]          = sum_{tap,i} x[p + shift(tap)][i] w[tap][i][o]
//   dgrad  dx [p][i]          = sum_{tap,o} dy[p - shift(tap)][o] w[tap][i][o]
//   wgrad  dw [tap][i][o]     = sum_p x[p + shift(tap)][i] dy[p][o]
// C[M][N] = sum_k A[m][k] B[n][k], with both operands materialised by a pack
// kernel in the K-major core-matrix layout the MMA reads ([plane][K/8][rows][8]
// fp16, plane 0 = hi, plane 1 = lo') -- im2col rows for fwd / dgrad, pixel-major
// rows for wgrad.  The fp32x3 split of DESIGN.md §3b with per-tensor power-of-two
// scales (max |v| 2^E in [2^13, 2^14), from a device max-reduction):
//   v 2^E = hi + lo' 2^-11,  hi = fp16(v 2^E),  lo' = fp16((v 2^E - hi) 2^11)
//   A B = Ahi Bhi + 2^-11 (Alo' Bhi + Ahi Blo')            (lo' lo' dropped: 2^-22)
// accumulated in two TMEM accumulators (big = hi hi, small = the cross terms at
// scale 2^11) that the epilogue combines in fp32 round-to-nearest and descales
// by 2^-(Ea+Eb).  Streaming K needs no ordering between the two, unlike the
// inference kernels' scale-input-d fold.  wgrad's K (pixels) is split over CTAs
// (partials summed by a reduction kernel), which also bounds how many truncating
// MMA accumulations (~0.2 ulp each, scripts/acc_probe.cu) any sum sees.
//
// GEMM kernel roles: warp 0 TMA producer (A hi / lo, B hi / lo per 64-wide K
// stage), warp 1 MMA issuer (M = 128, N = Np <= 128, 3 MMAs per K=16 step), warps
// 2-9 epilogue (two per TMEM lane quarter, half the columns each), two
// accumulator sets so the epilogue of one tile overlaps the next tile's MMAs.
#include "tc_common.cuh"
#include "../../include/nrx_train.h"

namespace nrx {
namespace ttc {
using namespace tc;

constexpr int KSTAGE = 64;  // K per pipeline stage (8 chunks of 8)
constexpr int GEMM_THREADS = 64 + 256;

struct TShape {
  int n, S, T, cin, cout, k, r;
  __host__ __device__ int pixels() const { return n * S * T; }
};

// flattened pixel p = (img, s, t) shifted by (ds, dt); -1 outside the image
__device__ __forceinline__ int shift_px(const TShape& g, int p, int ds, int dt) {
  const int t = p % g.T, s = (p / g.T) % g.S;
  const int s2 = s + ds, t2 = t + dt;
  if (s2 < 0 || s2 >= g.S || t2 < 0 || t2 >= g.T) return -1;
  return p + ds * g.T + dt;
}

enum PackKind { PK_FWD_A = 0, PK_FWD_B = 1, PK_DGRAD_A = 2, PK_DGRAD_B = 3, PK_WGRAD_A = 4, PK_WGRAD_B = 5 };

struct PackArgs {
  TShape g;
  int kind;
  const float* src;
  __half* dst;          // [2][Kp/8][Rp][8]
  int R, Rp, K, Kp;     // valid / padded rows and K
  int cp;               // channel stride of a tap in K (fwd / dgrad) or of a tap in rows (wgrad A)
  const uint32_t* amax; // max |src| as float bits
};

// power-of-two scale 2^E with max 2^E in [2^13, 2^14) (split_exponent on the device)
__device__ __forceinline__ int scale_exp(uint32_t maxbits) {
  const int ex = (int)((maxbits >> 23) & 0xff);
  if (maxbits == 0 || ex == 0xff) return 0;
  const int e = ex == 0 ? -126 : ex - 126;  // max < 2^e
  int E = 14 - e;
  return E < -100 ? -100 : E > 100 ? 100 : E;
}

// max |x| as float bits (non-negative floats order like their bit patterns):
// float4 loads where aligned, one atomic per block
__global__ void __launch_bounds__(256) k_absmax(const float* __restrict__ x, size_t n, uint32_t* out) {
  __shared__ float wm[8];
  float m = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x, t0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if ((reinterpret_cast<uintptr_t>(x) & 15) == 0) {
    const size_t n4 = n / 4;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (size_t i = t0; i < n4; i += stride) {
      const float4 v = x4[i];
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    }
    for (size_t i = 4 * n4 + t0; i < n; i += stride) m = fmaxf(m, fabsf(x[i]));
  } else {
    for (size_t i = t0; i < n; i += stride) m = fmaxf(m, fabsf(x[i]));
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) m = fmaxf(m, wm[w]);
    if (m > 0.f) atomicMax(out, __float_as_uint(m));
  }
}

__device__ __forceinline__ void store_split(const PackArgs& a, int kc, int row, float* v, float sc) {
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] *= sc;
  uint4 hi, lo;
  split_chunk(v, hi, lo);
  const size_t plane = (size_t)(a.Kp / 8) * a.Rp * 8;
  __half* d = a.dst + ((size_t)kc * a.Rp + row) * 8;
  *reinterpret_cast<uint4*>(d) = hi;
  *reinterpret_cast<uint4*>(d + plane) = lo;
}

// im2col operands of fwd / dgrad: one thread per (pixel row, tap) writes the
// tap's cp/8 chunks (the pixel's shifted source row read once, vectorised when
// the channel count allows); consecutive threads = consecutive rows, so every
// chunk store of a warp is 512 contiguous bytes per plane.  Rows >= R and the
// K padding beyond taps * cp are written as zeros by k_pack_kpad / here.
__global__ void k_pack_im2col(PackArgs a) {
  const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const int row = (int)(idx % a.Rp);
  const int tap = (int)(idx / a.Rp);
  const TShape& g = a.g;
  if (tap >= g.k * g.k) return;
  const float sc = ldexpf(1.f, scale_exp(*a.amax));
  const int sgn = a.kind == PK_FWD_A ? 1 : -1;
  const int cs = a.kind == PK_FWD_A ? g.cin : g.cout;
  const int src = row < a.R ? shift_px(g, row, sgn * (tap / g.k - g.r), sgn * (tap % g.k - g.r)) : -1;
  const float* p = a.src + (size_t)(src < 0 ? 0 : src) * cs;
  const bool v4 = (cs & 3) == 0 && (reinterpret_cast<uintptr_t>(a.src) & 15) == 0;
  for (int c0 = 0; c0 < a.cp; c0 += 8) {
    float v[8];
    if (src >= 0 && v4 && c0 + 8 <= cs) {
      const float4 x0 = *reinterpret_cast<const float4*>(p + c0), x1 = *reinterpret_cast<const float4*>(p + c0 + 4);
      v[0] = x0.x; v[1] = x0.y; v[2] = x0.z; v[3] = x0.w;
      v[4] = x1.x; v[5] = x1.y; v[6] = x1.z; v[7] = x1.w;
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = (src >= 0 && c0 + e < cs) ? p[c0 + e] : 0.f;
    }
    store_split(a, (tap * a.cp + c0) / 8, row, v, sc);
  }
}

// zero chunks of the K padding [taps * cp, Kp) of an im2col operand
__global__ void k_pack_kpad(PackArgs a, int kc0) {
  const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const int row = (int)(idx % a.Rp);
  const int kc = kc0 + (int)(idx / a.Rp);
  if (kc >= a.Kp / 8) return;
  float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  store_split(a, kc, row, v, 1.f);
}

// One thread per (16-byte chunk of 8 K values, row): gather, scale, split, store both planes.
__global__ void k_pack(PackArgs a) {
  const size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const int row = (int)(idx % a.Rp);
  const int kc = (int)(idx / a.Rp);
  if (kc >= a.Kp / 8) return;
  const TShape& g = a.g;
  const float sc = ldexpf(1.f, scale_exp(*a.amax));
  float v[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = 0.f;
  const int k0 = 8 * kc;
  if (row < a.R && k0 < a.K) {
    switch (a.kind) {
      case PK_FWD_A:
      case PK_DGRAD_A: {  // row = pixel, k = tap * cp + channel (a chunk never straddles two taps)
        const int tap = k0 / a.cp, c0 = k0 - tap * a.cp;
        const int sgn = a.kind == PK_FWD_A ? 1 : -1;
        const int cs = a.kind == PK_FWD_A ? g.cin : g.cout;
        const int src = shift_px(g, row, sgn * (tap / g.k - g.r), sgn * (tap % g.k - g.r));
        if (src >= 0) {
          const float* p = a.src + (size_t)src * cs;
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (c0 + e < cs) v[e] = p[c0 + e];
        }
        break;
      }
      case PK_FWD_B:
      case PK_DGRAD_B: {  // fwd: row = o, k = tap cinp + i;  dgrad: row = i, k = tap coutp + o
        const int tap = k0 / a.cp, c0 = k0 - tap * a.cp;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int c = c0 + e;
          if (a.kind == PK_FWD_B) {
            if (c < g.cin) v[e] = a.src[((size_t)tap * g.cin + c) * g.cout + row];
          } else {
            if (c < g.cout) v[e] = a.src[((size_t)tap * g.cin + row) * g.cout + c];
          }
        }
        break;
      }
      case PK_WGRAD_A: {  // row = tap * cinp + i, k = pixel
        const int tap = row / a.cp, i = row - tap * a.cp;
        if (i < g.cin) {
          const int ds = tap / g.k - g.r, dt = tap % g.k - g.r;
          int t = k0 % g.T, s = (k0 / g.T) % g.S;  // (s, t) of pixel k0, stepped below
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int p = k0 + e, s2 = s + ds, t2 = t + dt;
            if (p < a.K && s2 >= 0 && s2 < g.S && t2 >= 0 && t2 < g.T)
              v[e] = a.src[(size_t)(p + ds * g.T + dt) * g.cin + i];
            if (++t == g.T) {
              t = 0;
              if (++s == g.S) s = 0;
            }
          }
        }
        break;
      }
      default: {  // PK_WGRAD_B: row = o, k = pixel
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (k0 + e < a.K) v[e] = a.src[(size_t)(k0 + e) * g.cout + row];
        break;
      }
    }
  }
  store_split(a, kc, row, v, sc);
}

struct GemmParams {
  int M, N, Np, Kp;        // valid rows / columns, padded N, padded K
  int m_tiles, nsplit, ksplit;  // work items = m_tiles x nsplit; K per split (multiple of KSTAGE)
  int stages;
  float* C;                // row-major fp32, leading dimension ldc (split s at C + s * split_stride)
  int ldc;
  size_t split_stride;
  const uint32_t* amax_a;
  const uint32_t* amax_b;
};

__host__ __device__ inline uint32_t gemm_stage_bytes(int Np) { return 2u * 128 * KSTAGE * 2 + 2u * Np * KSTAGE * 2; }

__global__ void __launch_bounds__(GEMM_THREADS, 1)
    k_gemm_x3(const __grid_constant__ GemmParams p, const __grid_constant__ CUtensorMap mapA,
              const __grid_constant__ CUtensorMap mapB) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbytes = gemm_stage_bytes(p.Np);
  const uint32_t abytes = 128u * KSTAGE * 2, bbytes = (uint32_t)p.Np * KSTAGE * 2;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.stages * sbytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + 8;
  uint64_t* tfull = bars + 16;
  uint64_t* tempty = bars + 18;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(bars + 20);
  const uint32_t S0 = smem_u32(smem);
  const int warp = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
  const uint32_t tmem_cols = tmem_cols_pow2(4u * p.Np);
  if (warp == 0) tmem_alloc(tmem_ptr, tmem_cols);
  if (threadIdx.x == 32) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 256);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_ptr, 0);
  const int items = p.m_tiles * p.nsplit;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int st = 0;
      uint32_t ph = 0;
      for (int w = blockIdx.x; w < items; w += gridDim.x) {
        const int mt = w % p.m_tiles, sp = w / p.m_tiles;
        const int k0 = sp * p.ksplit, k1 = min(p.Kp, k0 + p.ksplit);
        for (int k = k0; k < k1; k += KSTAGE) {
          mbar_wait(smem_u32(&empty[st]), ph ^ 1);
          mbar_expect_tx(&full[st], sbytes);
          const uint32_t base = S0 + st * sbytes;
          const int kc = k / 8;
          tma_load_4d(base, &mapA, smem_u32(&full[st]), 0, mt * 8, kc, 0);
          tma_load_4d(base + abytes, &mapA, smem_u32(&full[st]), 0, mt * 8, p.Kp / 8 + kc, 0);
          tma_load_4d(base + 2 * abytes, &mapB, smem_u32(&full[st]), 0, 0, kc, 0);
          tma_load_4d(base + 2 * abytes + bbytes, &mapB, smem_u32(&full[st]), 0, 0, p.Kp / 8 + kc, 0);
          if (++st == p.stages) { st = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {  // ---------------- MMA issuer
    const uint32_t idesc = idesc_f16kind<__half>(128, p.Np);
    const uint64_t a_desc0 = smem_desc(0, 128 * 16, 128);
    const uint64_t b_desc0 = smem_desc(0, (uint32_t)p.Np * 16, 128);
    int st = 0, it = 0;
    uint32_t ph = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
      const int sp = w / p.m_tiles;
      const int k0 = sp * p.ksplit, k1 = min(p.Kp, k0 + p.ksplit);
      const int acc = it & 1;
      mbar_wait(smem_u32(&tempty[acc]), ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_big = tmem_base + acc * 2 * p.Np, d_small = d_big + p.Np;
      for (int k = k0; k < k1; k += KSTAGE) {
        mbar_wait(smem_u32(&full[st]), ph);
        tc_fence_after();
        const uint32_t base = (S0 + st * sbytes) >> 4;
        const uint64_t ahi = a_desc0 + base, alo = ahi + (abytes >> 4);
        const uint64_t bhi = b_desc0 + base + (2 * abytes >> 4), blo = bhi + (bbytes >> 4);
#pragma unroll
        for (int j = 0; j < KSTAGE / 16; ++j) {
          const uint32_t acc_on = (k > k0 || j > 0) ? 1u : 0u;
          const uint32_t ao = j * 2 * 128, bo = j * 2 * p.Np;  // two 8-wide chunks per K=16 step (16-B units)
          mma_bf16_warp(d_big, ahi + ao, bhi + bo, idesc, acc_on);
          mma_bf16_warp(d_small, alo + ao, bhi + bo, idesc, acc_on);
          mma_bf16_warp(d_small, ahi + ao, blo + bo, idesc, 1u);
        }
        mma_commit_warp(&empty[st]);
        if (++st == p.stages) { st = 0; ph ^= 1; }
      }
      mma_commit_warp(&tfull[acc]);
    }
  } else {  // ---------------- epilogue: warps 2..9
    const int q = warp & 3, half = (warp - 2) >> 2;
    const int r = 32 * q + lane;
    const uint32_t lane_off = static_cast<uint32_t>(32 * q) << 16;
    const float descale = ldexpf(1.f, -(scale_exp(*p.amax_a) + scale_exp(*p.amax_b)));
    const int cspan = p.Np / 2, cbeg = half * cspan;
    int it = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
      const int mt = w % p.m_tiles, sp = w / p.m_tiles;
      const int acc = it & 1;
      mbar_wait(smem_u32(&tfull[acc]), (it >> 1) & 1);
      tc_fence_after();
      const int row = mt * 128 + r;
      float* crow = p.C + sp * p.split_stride + (size_t)row * p.ldc;
      const uint32_t tb = tmem_base + lane_off + acc * 2 * p.Np;
      for (int c = cbeg; c < cbeg + cspan; c += 8) {
        float big[8], small[8];
        tmem_ld8(tb + c, big);
        tmem_ld8(tb + p.Np + c, small);
        tmem_wait_ld();
        if (row < p.M) {
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (c + e < p.N) crow[c + e] = fmaf(small[e], 1.f / 2048.f, big[e]) * descale;
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, tmem_cols);
  }
}

// dw[tap][i][o] = sum over splits of partial[s][tap cinp + i][o]
__global__ void k_wgrad_reduce(const float* __restrict__ part, int nsplit, size_t split_stride, int ldp, TShape g,
                               int cinp, float* __restrict__ dw) {
  const int n = g.k * g.k * g.cin * g.cout;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  const int o = idx % g.cout, i = (idx / g.cout) % g.cin, tap = idx / (g.cout * g.cin);
  const size_t off = (size_t)(tap * cinp + i) * ldp + o;
  float s = 0.f;
  for (int sp = 0; sp < nsplit; ++sp) s += part[sp * split_stride + off];
  dw[idx] = s;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

inline int rup_i(int a, int b) { return (a + b - 1) / b * b; }
inline size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

// 4-D map over an operand [2][Kp/8][Rp][8] fp16, viewed as {128 (16 rows x 8), Rp/16, 2 Kp/8, 1};
// box {128, box_rows/16, 8, 1} = one K stage of box_rows rows.
static int make_operand_map(CUtensorMap* m, const void* base, int Rp, int Kp, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return 3;
  const cuuint64_t dims[4] = {128, (cuuint64_t)(Rp / 16), (cuuint64_t)(2 * Kp / 8), 1};
  const cuuint64_t strides[3] = {256, (cuuint64_t)Rp * 16, (cuuint64_t)(2 * Kp / 8) * Rp * 16};
  const cuuint32_t box[4] = {128, (cuuint32_t)(box_rows / 16), KSTAGE / 8, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 4;
}

// Shapes of one operator's GEMM
struct GemmShape {
  int M, N, K, Mp, Np, Kp, cpA, cpB, kindA, kindB;
  int m_tiles, nsplit, ksplit;
  size_t a_bytes, b_bytes, part_bytes;
};

static int gemm_shape(const TShape& g, int op, GemmShape* s) {
  const int taps = g.k * g.k, P = g.pixels();
  const int cinp = rup_i(g.cin, 8), coutp = rup_i(g.cout, 8);
  if (op == 0) {  // fwd: M = pixels, N = cout, K = taps cinp
    *s = GemmShape{P, g.cout, taps * cinp, 0, 0, 0, cinp, cinp, PK_FWD_A, PK_FWD_B, 0, 1, 0, 0, 0, 0};
  } else if (op == 1) {  // dgrad: M = pixels, N = cin, K = taps coutp
    *s = GemmShape{P, g.cin, taps * coutp, 0, 0, 0, coutp, coutp, PK_DGRAD_A, PK_DGRAD_B, 0, 1, 0, 0, 0, 0};
  } else {  // wgrad: M = taps cinp (rows tap, i), N = cout, K = pixels
    *s = GemmShape{taps * cinp, g.cout, P, 0, 0, 0, cinp, 0, PK_WGRAD_A, PK_WGRAD_B, 0, 1, 0, 0, 0, 0};
  }
  s->Mp = rup_i(s->M, 128);
  s->Np = rup_i(s->N, 16);
  s->Kp = rup_i(s->K, KSTAGE);
  if (s->Np > 128 || s->M <= 0 || s->N <= 0 || s->K <= 0) return 1;
  s->m_tiles = s->Mp / 128;
  if (op == 2) {  // split K over enough CTAs to fill the GPU, at most 64 stages (4096 pixels) per split
    int ns = (2 * num_sms() + s->m_tiles - 1) / s->m_tiles;
    const int min_ns = (s->Kp / KSTAGE + 63) / 64;
    if (ns < min_ns) ns = min_ns;
    if (ns > s->Kp / KSTAGE) ns = s->Kp / KSTAGE;
    s->ksplit = rup_i((s->Kp + ns - 1) / ns, KSTAGE);
    s->nsplit = (s->Kp + s->ksplit - 1) / s->ksplit;
  } else {
    s->ksplit = s->Kp;
    s->nsplit = 1;
  }
  s->a_bytes = align256((size_t)2 * s->Kp * s->Mp * 2);
  s->b_bytes = align256((size_t)2 * s->Kp * s->Np * 2);
  s->part_bytes = op == 2 ? align256((size_t)s->nsplit * s->Mp * s->Np * 4) : 0;
  return 0;
}

static size_t op_workspace(const GemmShape& s) { return 256 + s.a_bytes + s.b_bytes + s.part_bytes; }

static int check_shape(const TShape& g) {
  if (g.n <= 0 || g.S <= 0 || g.T <= 0 || g.cin <= 0 || g.cout <= 0 || g.k <= 0 || !(g.k & 1)) return 1;
  if (g.cin > 128 || g.cout > 128) return 1;
  if ((long long)g.n * g.S * g.T >= (1ll << 31) / 16) return 1;
  return 0;
}

static int run_op(const TShape& g, int op, const float* a_src, size_t a_n, const float* b_src, size_t b_n,
                  float* out, void* ws, size_t ws_bytes, cudaStream_t st) {
  GemmShape s;
  if (gemm_shape(g, op, &s)) return 1;
  if (!ws || ws_bytes < op_workspace(s)) return 1;
  uint8_t* w8 = static_cast<uint8_t*>(ws);
  uint32_t* amax = reinterpret_cast<uint32_t*>(w8);
  __half* A = reinterpret_cast<__half*>(w8 + 256);
  __half* B = reinterpret_cast<__half*>(w8 + 256 + s.a_bytes);
  float* part = reinterpret_cast<float*>(w8 + 256 + s.a_bytes + s.b_bytes);
  if (cudaMemsetAsync(amax, 0, 8, st) != cudaSuccess) return 4;
  const int sms = num_sms();
  auto blocks = [&](size_t n) { const size_t b = (n / 4 + 255) / 256; return (unsigned)(b < 1 ? 1 : b > (size_t)sms * 4 ? sms * 4 : b); };
  k_absmax<<<blocks(a_n), 256, 0, st>>>(a_src, a_n, amax);
  k_absmax<<<blocks(b_n), 256, 0, st>>>(b_src, b_n, amax + 1);
  PackArgs pa{g, s.kindA, a_src, A, s.M, s.Mp, s.K, s.Kp, s.cpA, amax};
  PackArgs pb{g, s.kindB, b_src, B, s.N, s.Np, s.K, s.Kp, s.cpB, amax + 1};
  if (op == 2) {  // wgrad: K = pixels on both operands
    pa.K = pb.K = s.K;
    pb.cp = 0;
  }
  const size_t na = (size_t)s.Mp * (s.Kp / 8), nb = (size_t)s.Np * (s.Kp / 8);
  if (op == 2) {
    k_pack<<<(unsigned)((na + 255) / 256), 256, 0, st>>>(pa);
  } else {
    const int taps = g.k * g.k, kc_used = taps * s.cpA / 8;
    const size_t ni = (size_t)s.Mp * taps, npad = (size_t)s.Mp * (s.Kp / 8 - kc_used);
    k_pack_im2col<<<(unsigned)((ni + 255) / 256), 256, 0, st>>>(pa);
    if (npad) k_pack_kpad<<<(unsigned)((npad + 255) / 256), 256, 0, st>>>(pa, kc_used);
  }
  k_pack<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(pb);
  CUtensorMap ma, mb;
  if (make_operand_map(&ma, A, s.Mp, s.Kp, 128) || make_operand_map(&mb, B, s.Np, s.Kp, s.Np)) return 4;
  GemmParams p{};
  p.M = s.M;
  p.N = s.N;
  p.Np = s.Np;
  p.Kp = s.Kp;
  p.m_tiles = s.m_tiles;
  p.nsplit = s.nsplit;
  p.ksplit = s.ksplit;
  p.amax_a = amax;
  p.amax_b = amax + 1;
  if (op == 2) {
    p.C = part;
    p.ldc = s.Np;
    p.split_stride = (size_t)s.Mp * s.Np;
  } else {
    p.C = out;
    p.ldc = s.N;
    p.split_stride = 0;
  }
  const size_t sb = gemm_stage_bytes(s.Np), extra = 32 * 8 + 64;
  p.stages = 6;
  while (p.stages > 2 && p.stages * sb + extra > SMEM_LIMIT) --p.stages;
  const size_t smem = p.stages * sb + extra;
  if (set_smem((const void*)k_gemm_x3, SMEM_LIMIT)) return 4;
  const int items = s.m_tiles * s.nsplit;
  k_gemm_x3<<<items < sms ? items : sms, GEMM_THREADS, smem, st>>>(p, ma, mb);
  if (op == 2) {
    const int n = g.k * g.k * g.cin * g.cout;
    k_wgrad_reduce<<<(n + 255) / 256, 256, 0, st>>>(part, s.nsplit, p.split_stride, s.Np, g, s.cpA, out);
  }
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 4;
}

}  // namespace ttc
}  // namespace nrx

using namespace nrx::ttc;

extern "C" {

size_t nrx_train_tc_workspace(int n, int S, int T, int cin, int cout, int k) {
  const TShape g{n, S, T, cin, cout, k, k / 2};
  if (check_shape(g)) return 0;
  size_t need = 0;
  for (int op = 0; op < 3; ++op) {
    GemmShape s;
    if (gemm_shape(g, op, &s)) return 0;
    const size_t b = op_workspace(s);
    if (b > need) need = b;
  }
  return need;
}

int nrx_train_conv_tc_fwd(int n, int S, int T, int cin, int cout, int k, const float* x, const float* w, float* y,
                          void* ws, size_t ws_bytes, void* stream) {
  const TShape g{n, S, T, cin, cout, k, k / 2};
  if (check_shape(g) || !x || !w || !y) return 1;
  return run_op(g, 0, x, (size_t)g.pixels() * cin, w, (size_t)k * k * cin * cout, y, ws, ws_bytes,
                (cudaStream_t)stream);
}

int nrx_train_conv_tc_dgrad(int n, int S, int T, int cin, int cout, int k, const float* dy, const float* w,
                            float* dx, void* ws, size_t ws_bytes, void* stream) {
  const TShape g{n, S, T, cin, cout, k, k / 2};
  if (check_shape(g) || !dy || !w || !dx) return 1;
  return run_op(g, 1, dy, (size_t)g.pixels() * cout, w, (size_t)k * k * cin * cout, dx, ws, ws_bytes,
                (cudaStream_t)stream);
}

int nrx_train_conv_tc_wgrad(int n, int S, int T, int cin, int cout, int k, const float* x, const float* dy,
                            float* dw, void* ws, size_t ws_bytes, void* stream) {
  const TShape g{n, S, T, cin, cout, k, k / 2};
  if (check_shape(g) || !x || !dy || !dw) return 1;
  return run_op(g, 2, x, (size_t)g.pixels() * cin, dy, (size_t)g.pixels() * cout, dw, ws, ws_bytes,
                (cudaStream_t)stream);
}

}  // extern "C"
