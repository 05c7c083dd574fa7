// Device helpers shared by all kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "nrx_internal.h"

namespace nrx {

// Programmatic dependent launch (PDL).  A kernel launched with programmatic
// stream serialization may start while its predecessor still runs: it does its
// prologue (barriers, TMEM, resident weights), then pdl_wait() blocks until the
// predecessor grid has completed and its writes are visible.  Every read or
// write of activation memory must come after pdl_wait().
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Lets the next PDL-launched kernel be scheduled (on SMs this grid frees).
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }

// Distance from subcarrier s to the nearest comb subcarrier of UE u
// (positional_encoding, nrx.py:165-167).
__device__ __forceinline__ int comb_dist(int s, int u, const Geom& g) {
  const int o = u;  // the UE's comb offset: u < U <= comb (validate(), slot.py:60)
  if (s <= o) return o - s;
  const int q = g.comb == 1 ? s - o : (int)__umulhi((unsigned)(s - o), g.comb_magic);  // exact (make_geom)
  const int lo = o + q * g.comb;
  int d = s - lo;
  const int hi = lo + g.comb;
  if (hi < g.S && hi - s < d) d = hi - s;
  return d;
}

// float32(dist / S) as numpy computes it (int/int true-divide in float64,
// then cast).  For integers below 2^24 the correctly rounded fp32 quotient is
// identical: the float64 quotient can never fall on (or across) a float32
// rounding midpoint, since any midpoint differs from a/b by >= 1/(b 2^k)
// while the float64 error is < 2^-28 / 2^k.
// combs wider than 16 (not in any reference configuration): an out-of-line
// IEEE division instead of the table, kept out of the unrolled epilogues
static __device__ __noinline__ float df_div(int k, int S) { return __fdiv_rn((float)k, (float)S); }
__device__ __forceinline__ float pos_df(int s, int u, const Geom& g) {
  if (!g.freq_enc) return 0.f;
  const int k = comb_dist(s, u, g);  // < comb
  return g.comb <= 16 ? g.df_tab[k] : df_div(k, g.S);
}

// Value a producer writes into state channel c >= d (pos encoding / zero).
__device__ __forceinline__ float state_extra(int c, int s, int t, int u, const Geom& g) {
  if (c == g.d) return g.dt[t];
  if (c == g.d + 1) return pos_df(s, u, g);
  return 0.f;
}

// Grid row -> (subcarrier s, padded symbol t).  floor((row + 1/2) / Tp) by
// one float multiply: the fractional part of (row + 1/2) / Tp stays >= 1/(2 Tp)
// from an integer and the product's error is below row / Tp * 2^-22, so the
// result is exact for rows < 2^21 (make_geom enforces it).
__device__ __forceinline__ void row_to_st(int row, const Geom& g, int& s, int& t) {
  s = __float2int_rz((static_cast<float>(row) + 0.5f) * g.inv_Tp);
  t = row - s * g.Tp;
}

// Address of the 16-byte chunk (slab, chunk, row) of a chunk-planar buffer.
template <typename T>
__device__ __forceinline__ T* chunk_ptr(T* base, int slab, int nchunks, int chunk, int row, const Geom& g) {
  constexpr int cw = 16 / sizeof(T);
  return base + (((size_t)slab * nchunks + chunk) * g.rows_slab + row) * cw;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float2 unpack_bf16x2(uint32_t v) {
  __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&v);
  return __bfloat1622float2(b);
}

// Write 4 (fp32) or 8 (bf16) channel values as one 16-byte chunk.
__device__ __forceinline__ void store_chunk(float* p, const float* v) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void store_chunk(__nv_bfloat16* p, const float* v) {
  uint4 q;
  q.x = pack_bf16x2(v[0], v[1]);
  q.y = pack_bf16x2(v[2], v[3]);
  q.z = pack_bf16x2(v[4], v[5]);
  q.w = pack_bf16x2(v[6], v[7]);
  *reinterpret_cast<uint4*>(p) = q;
}

__device__ __forceinline__ void store_chunk(__half* p, const float* v) {
  uint4 q;
  __half2 h0 = __floats2half2_rn(v[0], v[1]), h1 = __floats2half2_rn(v[2], v[3]);
  __half2 h2 = __floats2half2_rn(v[4], v[5]), h3 = __floats2half2_rn(v[6], v[7]);
  q.x = *reinterpret_cast<uint32_t*>(&h0);
  q.y = *reinterpret_cast<uint32_t*>(&h1);
  q.z = *reinterpret_cast<uint32_t*>(&h2);
  q.w = *reinterpret_cast<uint32_t*>(&h3);
  *reinterpret_cast<uint4*>(p) = q;
}

// 8 channel values as one packed 16-byte half-precision chunk, and a store
// of it to a shared-memory address (no generic-to-shared conversion).
__device__ __forceinline__ uint4 pack_chunk(const float* v, const __nv_bfloat16*) {
  return make_uint4(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]), pack_bf16x2(v[4], v[5]),
                    pack_bf16x2(v[6], v[7]));
}
__device__ __forceinline__ uint4 pack_chunk(const float* v, const __half*) {
  __half2 h[4] = {__floats2half2_rn(v[0], v[1]), __floats2half2_rn(v[2], v[3]), __floats2half2_rn(v[4], v[5]),
                  __floats2half2_rn(v[6], v[7])};
  return make_uint4(*reinterpret_cast<uint32_t*>(&h[0]), *reinterpret_cast<uint32_t*>(&h[1]),
                    *reinterpret_cast<uint32_t*>(&h[2]), *reinterpret_cast<uint32_t*>(&h[3]));
}
// The reference's ReLU, np.maximum(x, 0) (autodiff.py:203-205): NaN propagates
// (fmaxf would return 0 and hide a non-finite input from CHECK_FINITE).
__device__ __forceinline__ float relu_f(float x) { return x < 0.f ? 0.f : x; }
// max(x, 0) on a packed chunk (exact: rounding commutes with the clamp; NaN propagates)
__device__ __forceinline__ uint4 relu_chunk(uint4 q, const __half*) {
  uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __half2 h = __hmax2_nan(*reinterpret_cast<__half2*>(&w[i]), __float2half2_rn(0.f));
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ __forceinline__ uint4 relu_chunk(uint4 q, const __nv_bfloat16*) {
  uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h = __hmax2_nan(*reinterpret_cast<__nv_bfloat162*>(&w[i]), __float2bfloat162_rn(0.f));
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}
// zero a packed chunk on invalid (pad) rows: mask = 0 or ~0
__device__ __forceinline__ uint4 mask_chunk(uint4 q, uint32_t m) {
  return make_uint4(q.x & m, q.y & m, q.z & m, q.w & m);
}
__device__ __forceinline__ void st_shared_u4(uint32_t addr, uint4 q) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(q.x), "r"(q.y), "r"(q.z), "r"(q.w)
               : "memory");
}

// Unpack one 16-byte chunk of 8 half-precision channels (type tag selects
// bf16 or fp16) into floats.
__device__ __forceinline__ void unpack_chunk(uint4 q, const __nv_bfloat16*, float* v) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = unpack_bf16x2(w[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void unpack_chunk(uint4 q, const __half*, float* v) {
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}

// fp32x3 operand split (NRX_FP32X3): a = hi + lo 2^-11 with hi = fp16(a) and
// lo = fp16((a - hi) 2^11).  a - hi is exact in fp32 and |lo| <= |a|, so lo
// never overflows where hi does not; lo keeps 11 more bits for |a| >= 2^-13.
constexpr float X3_LO_SCALE = 2048.f;
constexpr float X3_LO_INV = 1.f / 2048.f;
__device__ __forceinline__ void split_chunk(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __half2 hh = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
    const float2 hf = __half22float2(hh);
    const __half2 ll = __floats2half2_rn((v[2 * i] - hf.x) * X3_LO_SCALE, (v[2 * i + 1] - hf.y) * X3_LO_SCALE);
    h[i] = *reinterpret_cast<const uint32_t*>(&hh);
    l[i] = *reinterpret_cast<const uint32_t*>(&ll);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}
// split_chunk that also records a range violation at every split (the
// earliest point an overflowed plane can be seen): a hi half that is inf or
// NaN (|v| >= 65520 rounds to inf; below that hi + lo 2^-11 still represents v).
// Exponent field all ones, two halves per word: (e & 0x7c00) + 0x0400 carries
// into the half's sign bit only for 0x7c00.
__device__ __forceinline__ void split_chunk(const float* v, uint4& hi, uint4& lo, uint32_t& bad) {
  split_chunk(v, hi, lo);
  const uint32_t h[4] = {hi.x, hi.y, hi.z, hi.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) bad |= ((h[i] & 0x7c007c00u) + 0x04000400u) & 0x80008000u;
}
// the range-guard word (Geom::flag, NRX_WS_FLAG_OFFSET): one atomic per offending thread
__device__ __forceinline__ void report_range(uint32_t bad, uint32_t* flag) {
  if (bad && flag) atomicOr(flag, 1u);
}

// hi + lo 2^-11 in fp32 (exact: both terms fit the 24-bit significand)
__device__ __forceinline__ void unsplit_chunk(uint4 hi, uint4 lo, float* v) {
  const uint32_t h[4] = {hi.x, hi.y, hi.z, hi.w}, l[4] = {lo.x, lo.y, lo.z, lo.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&h[i]));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&l[i]));
    v[2 * i] = fmaf(b.x, X3_LO_INV, a.x);
    v[2 * i + 1] = fmaf(b.y, X3_LO_INV, a.y);
  }
}

__device__ __forceinline__ int io_index(const int32_t* mod_order, int slab, const Geom& g) {
  if (g.n_io == 1 || mod_order == nullptr) return 0;
  const int m = mod_order[slab];
  for (int i = 0; i < g.n_io; ++i)
    if (g.io_orders[i] == m) return i;
  return -1;
}

}  // namespace nrx
