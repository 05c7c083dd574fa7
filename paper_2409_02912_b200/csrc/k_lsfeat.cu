// K1: DMRS least-squares channel estimate fused with input-feature assembly.
//
// Replaces ls_features (nrx.py:205-213) -> classical.ls_estimate
// (classical.py:40-78) and assemble_features + positional_encoding
// (nrx.py:159-202).  One thread per (slab, row): it reads the 4-antenna
// received sample at its RE, the (up to 2) comb pilots that bracket its
// subcarrier at its nearest pilot symbol, and writes the C_in feature
// channels of that row as 16-byte chunks into the chunk-planar feature
// buffer.  Pad rows (t >= T, s >= S) are written as zeros, which provides
// the convolution's zero padding downstream.  The LS arithmetic runs in
// float64 with the reference's operation order (no FMA contraction) and
// is rounded to float32 once, as assemble_features does.
//
// HBM-bound: per RE-slab it reads 8*B bytes of y (c64) and writes
// Cf * sizeof(out) bytes; pilot samples are re-read from L1/L2.
#include <type_traits>

#include "nrx_device.cuh"
#include "nrx_kernels.h"

namespace nrx {

template <typename C>
__device__ __forceinline__ double2 ld_c(const C* p);
template <>
__device__ __forceinline__ double2 ld_c<float2>(const float2* p) {
  float2 v = __ldg(p);
  return make_double2((double)v.x, (double)v.y);
}
template <>
__device__ __forceinline__ double2 ld_c<double2>(const double2* p) {
  return __ldg(p);
}
template <typename C>
__device__ __forceinline__ float2 ld_c_f(const C* p);
template <>
__device__ __forceinline__ float2 ld_c_f<float2>(const float2* p) { return __ldg(p); }
template <>
__device__ __forceinline__ float2 ld_c_f<double2>(const double2* p) {
  double2 v = __ldg(p);
  return make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
}

// conj(p)/|p|^2 the way numpy evaluates it for complex128 / float64:
// Smith division by (|p|^2 + 0j) degenerates to multiplication with the
// reciprocal 1/|p|^2 (classical.py:46).
__device__ __forceinline__ double2 pilot_scale(double2 p) {
  const double a = hypot(p.x, p.y);
  const double rec = __ddiv_rn(1.0, __dmul_rn(a, a));
  return make_double2(__dmul_rn(p.x, rec), __dmul_rn(-p.y, rec));
}

__device__ __forceinline__ double2 cmul_nofma(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

// BT > 0: the rx antenna count fixed at compile time, so the feature row
// stays in registers (BT = 0: runtime B, the row lives in local memory).
// X3: fp32x3 output, every chunk written as its fp16 hi plane (chunks
// [0, Cf/8)) and lo plane (chunks [Cf/8, 2 Cf/8)).
template <typename OutT, typename YT, typename PT, int BT, bool X3 = false>
__global__ void __launch_bounds__(128) k_ls_feat(Geom g, const YT* __restrict__ y, const PT* __restrict__ pilots,
                                                 int n_pilot_sets, const float* __restrict__ noise_feat,
                                                 OutT* __restrict__ feats) {
  constexpr int CW = 16 / sizeof(OutT);
  pdl_launch_dependents();  // the first conv's prologue may overlap this kernel's last wave
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int slab = blockIdx.y;
  if (row >= g.rows_slab) return;
  const int n = slab / g.U, u = slab - n * g.U;
  const int s = row / g.Tp, t = row - s * g.Tp;
  const bool valid = s < g.S && t < g.T;

  float f[48];
#pragma unroll
  for (int c = 0; c < 48; ++c) f[c] = 0.f;

  if (valid) {
    const int B = BT > 0 ? BT : g.B;
    const YT* yrow = y + (((size_t)n * g.S + s) * g.T + t) * B;
#pragma unroll
    for (int b = 0; b < (BT > 0 ? BT : 8); ++b) {
      if (b >= B) break;
      float2 v = ld_c_f(yrow + b);
      f[2 * b] = v.x;
      f[2 * b + 1] = v.y;
    }
    // LS on UE u's comb at its nearest pilot symbol, linear interpolation in s.
    const int k = g.nearest[t];
    const int pt = g.ps[k];
    const int o = u % g.comb;
    const int F = (g.S - o + g.comb - 1) / g.comb;
    const int Fmax = (g.S + g.comb - 1) / g.comb;
    const int pset = n_pilot_sets > 1 ? n : 0;
    const PT* pil = pilots + (((size_t)pset * g.U + u) * Fmax) * g.K;
    int j = 0;
    double frac = 0.0;
    if (F > 1) {
      const int diff = s - o;
      int q = diff >= 0 ? diff / g.comb : -1;  // python floor division
      j = q < 0 ? 0 : (q > F - 2 ? F - 2 : q);
      frac = __ddiv_rn((double)(s - (o + j * g.comb)), (double)g.comb);
    }
    const double2 q0 = pilot_scale(ld_c(pil + (size_t)j * g.K + k));
    const double2 q1 = F > 1 ? pilot_scale(ld_c(pil + (size_t)(j + 1) * g.K + k)) : q0;
    const YT* y0 = y + (((size_t)n * g.S + (o + j * g.comb)) * g.T + pt) * B;
    const YT* y1 = y + (((size_t)n * g.S + (o + (j + 1) * g.comb)) * g.T + pt) * B;
#pragma unroll
    for (int b = 0; b < (BT > 0 ? BT : 8); ++b) {
      if (b >= B) break;
      const double2 r0 = cmul_nofma(ld_c(y0 + b), q0);
      double2 h = r0;
      if (F > 1) {
        const double2 r1 = cmul_nofma(ld_c(y1 + b), q1);
        h.x = __dadd_rn(r0.x, __dmul_rn(frac, __dsub_rn(r1.x, r0.x)));
        h.y = __dadd_rn(r0.y, __dmul_rn(frac, __dsub_rn(r1.y, r0.y)));
      }
      f[2 * B + 2 * b] = __double2float_rn(h.x);
      f[2 * B + 2 * b + 1] = __double2float_rn(h.y);
    }
    f[4 * B] = g.dt[t];
    f[4 * B + 1] = pos_df(s, u, g);
    if (g.noise_plane) f[4 * B + 2] = noise_feat[n];
  }
  const int nch = g.Cf / CW;
  if constexpr (X3) {
    uint32_t bad = 0;
#pragma unroll
    for (int c = 0; c < 48 / CW; ++c)
      if (c < nch) {
        uint4 hi, lo;
        split_chunk(f + c * CW, hi, lo, bad);
        *reinterpret_cast<uint4*>(chunk_ptr(feats, slab, 2 * nch, c, row, g)) = hi;
        *reinterpret_cast<uint4*>(chunk_ptr(feats, slab, 2 * nch, nch + c, row, g)) = lo;
      }
    report_range(bad, g.flag);
  } else {
#pragma unroll
    for (int c = 0; c < 48 / CW; ++c)
      if (c < nch) store_chunk(chunk_ptr(feats, slab, nch, c, row, g), f + c * CW);
    if (std::is_same<OutT, __half>::value) {  // fp16 features: the same range guard
      uint32_t bad = 0;
#pragma unroll
      for (int c = 0; c < 48; ++c) bad |= (__float_as_uint(f[c]) & 0x7fffffffu) > 0x477fe000u;
      report_range(bad, g.flag);
    }
  }
}

template <typename OutT, bool X3 = false>
int launch_ls_feat_t(const Geom& g, const void* y, int y_c128, const void* pil, int pil_c128, int n_sets,
                     const float* noise, OutT* feats, cudaStream_t st) {
  dim3 grid(cdiv(g.rows_slab, 128), g.NU);
  const bool b4 = g.B == 4;
#define NRX_LSF(YT, PT)                                                                                         \
  do {                                                                                                          \
    if (b4)                                                                                                     \
      k_ls_feat<OutT, YT, PT, 4, X3><<<grid, 128, 0, st>>>(g, (const YT*)y, (const PT*)pil, n_sets, noise, feats);  \
    else                                                                                                        \
      k_ls_feat<OutT, YT, PT, 0, X3><<<grid, 128, 0, st>>>(g, (const YT*)y, (const PT*)pil, n_sets, noise, feats);  \
  } while (0)
  if (y_c128 && pil_c128)
    NRX_LSF(double2, double2);
  else if (y_c128)
    NRX_LSF(double2, float2);
  else if (pil_c128)
    NRX_LSF(float2, double2);
  else
    NRX_LSF(float2, float2);
#undef NRX_LSF
  return cudaPeekAtLastError() == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

int launch_ls_feat(const Geom& g, const void* y, int y_c128, const void* pil, int pil_c128, int n_sets,
                   const float* noise, void* feats, cudaStream_t st) {
  if (g.prec == NRX_BF16)
    return launch_ls_feat_t(g, y, y_c128, pil, pil_c128, n_sets, noise, (__nv_bfloat16*)feats, st);
  if (g.prec == NRX_FP32X3)
    return launch_ls_feat_t<__half, true>(g, y, y_c128, pil, pil_c128, n_sets, noise, (__half*)feats, st);
  if (g.prec == NRX_FP16)
    return launch_ls_feat_t(g, y, y_c128, pil, pil_c128, n_sets, noise, (__half*)feats, st);
  return launch_ls_feat_t(g, y, y_c128, pil, pil_c128, n_sets, noise, (float*)feats, st);
}

}  // namespace nrx
