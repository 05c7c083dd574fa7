// Training kernels: the NRX training step's
// convolutions and dense layers, forward and backward, and the Adam update,
// in fp32 like the reference's numpy autodiff (autodiff.py:302-350 conv2d /
// matmul and their VJPs, 428-525 Adam).
//
// Tensors are NHWC float32: x (n, S, T, cin), y (n, S, T, cout), kernel
// w (k, k, cin, cout) with 'same' zero padding (odd k).  A dense layer is the
// k = 1, T = 1 case (x (rows, cin) @ w (cin, cout)).
//
//   fwd    y[p, o]  = sum_{a,b,i} x[p + (a-r, b-r), i] w[a, b, i, o]   (+ bias)
//   dgrad  dx[p, i] = sum_{a,b,o} dy[p - (a-r, b-r), o] w[a, b, i, o]
//   wgrad  dw[a, b, i, o] = sum_p x[p + (a-r, b-r), i] dy[p, o],  db[o] = sum_p dy[p, o]
//
// Each kernel tiles 64 pixels per block: per tap the block stages the tap's
// weights and the 64 shifted pixel rows in shared memory, and every thread
// accumulates a strip of outputs of one pixel in registers (fwd / dgrad), or
// a strip of (i, o) weight-gradient entries over a chunk of pixels (wgrad,
// one block per (tap, pixel chunk), partials added with fp32 atomics).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "../../include/nrx_train.h"

namespace nrx {
namespace train {

constexpr int TP = 64;         // pixels per block
constexpr int THREADS = 256;   // 16 pixel groups x 16 channel groups
constexpr int PPT = 4;         // pixels per thread (fwd / dgrad)
constexpr int MAXC = 128;      // channel limit (update.conv0 has 2 d + 2 = 114 inputs)

struct Shape {
  int n, S, T, cin, cout, k, r;
  __host__ __device__ int pixels() const { return n * S * T; }
};

// flattened pixel p = (img, s, t) shifted by (ds, dt); -1 outside the image
__device__ __forceinline__ int shifted(const Shape& g, int p, int ds, int dt) {
  const int t = p % g.T, s = (p / g.T) % g.S;
  const int s2 = s + ds, t2 = t + dt;
  if (s2 < 0 || s2 >= g.S || t2 < 0 || t2 >= g.T) return -1;
  return p + ds * g.T + dt;
}

// Forward (DGRAD = false): out[p, c] = sum_{tap, j} in[p + shift(tap), j] W[tap][j][c]
// with (in, out, j, c) = (x, y, i, o).  Input gradient (DGRAD = true): the same
// contraction with (in, out, j, c) = (dy, dx, o, i), the tap shift negated and
// W read transposed.  Register micro-tile: 4 pixels x CPT channels per thread.
template <bool DGRAD, int CPT>
__global__ void __launch_bounds__(THREADS) k_conv_tile(Shape g, const float* __restrict__ in,
                                                       const float* __restrict__ w, const float* __restrict__ b,
                                                       float* __restrict__ out) {
  extern __shared__ __align__(16) float sm[];
  const int cj = DGRAD ? g.cout : g.cin;   // contraction channels
  const int co = DGRAD ? g.cin : g.cout;   // output channels
  const int cop = (co + 3) & ~3;           // padded to a float4
  const int cjp = cj | 1;                  // odd row stride: a thread's 4 pixels hit distinct banks (<= 2-way)
  float* Ws = sm;                          // [cj][cop]
  float* Xs = sm + cj * cop;               // [TP][cjp]
  __shared__ int s_st[TP];                 // (s << 16 | t) of the block's pixels, -1 past the end
  const int pg = threadIdx.x & 15, og = threadIdx.x >> 4;  // 16 pixel groups x 16 channel groups
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = g.pixels();
  const int pbase = blockIdx.x * TP;
  if (threadIdx.x < TP) {
    const int pp = pbase + threadIdx.x;
    s_st[threadIdx.x] = pp < P ? (((pp / g.T) % g.S) << 16) | (pp % g.T) : -1;
  }
  float acc[PPT][CPT];
#pragma unroll
  for (int a = 0; a < PPT; ++a)
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[a][c] = 0.f;
  for (int a = 0; a < g.k; ++a)
    for (int bb = 0; bb < g.k; ++bb) {
      __syncthreads();
      const float* wt = w + (size_t)(a * g.k + bb) * g.cin * g.cout;
      // staging without integer division: warps over rows, lanes over channels
      for (int j = warp; j < cj; j += THREADS / 32)
        for (int c = lane; c < cop; c += 32) {
          float v = 0.f;
          if (c < co) v = DGRAD ? wt[(size_t)c * g.cout + j] : wt[(size_t)j * g.cout + c];
          Ws[j * cop + c] = v;
        }
      const int ds = DGRAD ? g.r - a : a - g.r, dt = DGRAD ? g.r - bb : bb - g.r;
      for (int px = warp; px < TP; px += THREADS / 32) {
        const int st = s_st[px];
        const int s2 = (st >> 16) + ds, t2 = (st & 0xffff) + dt;
        const bool ok = st >= 0 && s2 >= 0 && s2 < g.S && t2 >= 0 && t2 < g.T;
        const float* src = in + (size_t)(pbase + px + ds * g.T + dt) * cj;
        for (int j = lane; j < cj; j += 32) Xs[px * cjp + j] = ok ? src[j] : 0.f;  // coalesced, conflict-free
      }
      __syncthreads();
#pragma unroll 2
      for (int j = 0; j < cj; ++j) {
        const float* xr = Xs + 4 * pg * cjp + j;
        float wv[CPT];
#pragma unroll
        for (int c4 = 0; c4 < CPT; c4 += 4) {
          const float4 t4 = *reinterpret_cast<const float4*>(Ws + j * cop + og * CPT + c4);
          wv[c4] = t4.x;
          wv[c4 + 1] = t4.y;
          wv[c4 + 2] = t4.z;
          wv[c4 + 3] = t4.w;
        }
        const float xa[PPT] = {xr[0], xr[cjp], xr[2 * cjp], xr[3 * cjp]};
#pragma unroll
        for (int a2 = 0; a2 < PPT; ++a2)
#pragma unroll
          for (int c = 0; c < CPT; ++c) acc[a2][c] = fmaf(xa[a2], wv[c], acc[a2][c]);
      }
    }
#pragma unroll
  for (int a2 = 0; a2 < PPT; ++a2) {
    const int p = pbase + 4 * pg + a2;
    if (p >= P) continue;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int ch = og * CPT + c;
      if (ch < co) out[(size_t)p * co + ch] = (!DGRAD && b) ? acc[a2][c] + b[ch] : acc[a2][c];
    }
  }
}

constexpr int WCHUNK = 1024;  // max pixels per wgrad block (fewer when there are few taps)
constexpr int WTP = 32;       // pixels staged per step

// dw[tap] (+)= sum over a pixel chunk of x[p + shift(tap)] (outer) dy[p]; thread
// (ti, to) owns i in [8 ti, 8 ti + 8), o in [ob + 4 to, ob + 4 to + 4) with
// ob = 64 blockIdx.z (outputs beyond 64 in a second grid plane).  Tap-0 blocks
// also accumulate db.  Partials are added with fp32 atomics.
__global__ void __launch_bounds__(THREADS) k_conv_wgrad(Shape g, int chunk, const float* __restrict__ x,
                                                        const float* __restrict__ dy, float* __restrict__ dw,
                                                        float* __restrict__ db) {
  extern __shared__ __align__(16) float sm[];
  const int cip = (g.cin + 7) & ~7, cop = (g.cout + 3) & ~3;
  float* Xs = sm;                  // [WTP][cip]
  float* Ds = sm + WTP * cip;      // [WTP][cop]
  const int tap = blockIdx.y, a = tap / g.k, bb = tap % g.k;
  const int P = g.pixels();
  const int p0 = blockIdx.x * chunk;  // chunk: a multiple of WTP
  const int ti = threadIdx.x >> 4, to = threadIdx.x & 15;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ds = a - g.r, dt = bb - g.r;
  const int ob = 64 * blockIdx.z + 4 * to;  // first output channel of this thread
  const bool active = 8 * ti < g.cin && ob < g.cout;
  float acc[8][4], bacc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int o = 0; o < 4; ++o) acc[i][o] = 0.f;
  for (int pt = p0; pt < p0 + chunk && pt < P; pt += WTP) {
    __syncthreads();
    for (int px = warp; px < WTP; px += THREADS / 32) {  // warps over pixels, lanes over channels
      const int pp = pt + px;
      const int src = pp < P ? shifted(g, pp, ds, dt) : -1;
      for (int i = lane; i < cip; i += 32)
        Xs[px * cip + i] = (src >= 0 && i < g.cin) ? x[(size_t)src * g.cin + i] : 0.f;
      for (int o = lane; o < cop; o += 32)
        Ds[px * cop + o] = (pp < P && o < g.cout) ? dy[(size_t)pp * g.cout + o] : 0.f;
    }
    __syncthreads();
    if (!active) continue;
#pragma unroll 4
    for (int px = 0; px < WTP; ++px) {
      const float4 x0 = *reinterpret_cast<const float4*>(Xs + px * cip + 8 * ti);
      const float4 x1 = *reinterpret_cast<const float4*>(Xs + px * cip + 8 * ti + 4);
      const float4 d4 = *reinterpret_cast<const float4*>(Ds + px * cop + ob);
      const float xi[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
      const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int o = 0; o < 4; ++o) acc[i][o] = fmaf(xi[i], dv[o], acc[i][o]);
      if (tap == 0 && ti == 0)
#pragma unroll
        for (int o = 0; o < 4; ++o) bacc[o] += dv[o];
    }
  }
  if (!active) return;
  const int nio = g.cin * g.cout;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      const int ii = 8 * ti + i, oo = ob + o;
      if (ii < g.cin && oo < g.cout) atomicAdd(dw + (size_t)tap * nio + (size_t)ii * g.cout + oo, acc[i][o]);
    }
  if (db && tap == 0 && ti == 0)
#pragma unroll
    for (int o = 0; o < 4; ++o)
      if (ob + o < g.cout) atomicAdd(db + ob + o, bacc[o]);
}

// Adam with the reference's bias-corrected update (autodiff.py:485-525)
__global__ void k_adam(int n, float* __restrict__ p, const float* __restrict__ grad, float* __restrict__ m,
                       float* __restrict__ v, float lr_c1, float b1, float b2, float c2, float eps) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float g = grad[i];
  const float mi = b1 * m[i] + (1.f - b1) * g;
  const float vi = b2 * v[i] + (1.f - b2) * g * g;
  m[i] = mi;
  v[i] = vi;
  p[i] -= lr_c1 * mi / (sqrtf(vi / c2) + eps);
}

template <bool DGRAD>
static int launch_tile(const Shape& g, const float* in, const float* w, const float* b, float* out,
                       cudaStream_t st) {
  const int co = DGRAD ? g.cin : g.cout, cj = DGRAD ? g.cout : g.cin;
  const int cop = (co + 3) & ~3;
  const size_t smem = (size_t)(cj * cop + TP * (cj | 1)) * 4;
  const int blocks = (g.pixels() + TP - 1) / TP;
  auto run = [&](auto kern) -> int {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 4;
    kern<<<blocks, THREADS, smem, st>>>(g, in, w, b, out);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : 4;
  };
  if (co <= 64) return run(k_conv_tile<DGRAD, 4>);
  return run(k_conv_tile<DGRAD, 8>);
}

static bool shape_ok(const Shape& g) {
  return g.n > 0 && g.S > 0 && g.T > 0 && g.cin > 0 && g.cout > 0 && g.k > 0 && (g.k & 1) && g.cin <= MAXC &&
         g.cout <= MAXC;
}

}  // namespace train
}  // namespace nrx

using namespace nrx::train;

extern "C" {

int nrx_train_conv_fwd(int n, int S, int T, int cin, int cout, int k, const float* x, const float* w,
                       const float* b, float* y, void* stream) {
  const Shape g{n, S, T, cin, cout, k, k / 2};
  if (!shape_ok(g) || !x || !w || !y) return 1;
  return launch_tile<false>(g, x, w, b, y, (cudaStream_t)stream);
}

int nrx_train_conv_dgrad(int n, int S, int T, int cin, int cout, int k, const float* dy, const float* w,
                         float* dx, void* stream) {
  const Shape g{n, S, T, cin, cout, k, k / 2};
  if (!shape_ok(g) || !dy || !w || !dx) return 1;
  return launch_tile<true>(g, dy, w, nullptr, dx, (cudaStream_t)stream);
}

int nrx_train_conv_wgrad(int n, int S, int T, int cin, int cout, int k, const float* x, const float* dy, float* dw,
                         float* db, void* stream) {
  const Shape g{n, S, T, cin, cout, k, k / 2};
  if (!shape_ok(g) || !x || !dy || !dw) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(dw, 0, (size_t)k * k * cin * cout * 4, st) != cudaSuccess) return 4;
  if (db && cudaMemsetAsync(db, 0, (size_t)cout * 4, st) != cudaSuccess) return 4;
  const int cip = (cin + 7) & ~7, cop = (cout + 3) & ~3;
  const size_t smem = (size_t)WTP * (cip + cop) * 4;
  // >= ~4 blocks per SM: chunks of WCHUNK pixels, smaller (multiples of WTP) for few taps
  const int want = (4 * 148 + k * k - 1) / (k * k);
  int chunks = (g.pixels() + WCHUNK - 1) / WCHUNK;
  if (chunks < want) chunks = want;
  const int per = ((g.pixels() + chunks - 1) / chunks + WTP - 1) / WTP * WTP;
  chunks = (g.pixels() + per - 1) / per;
  dim3 grid(chunks, k * k, (cout + 63) / 64);
  k_conv_wgrad<<<grid, THREADS, smem, st>>>(g, per, x, dy, dw, db);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 4;
}

int nrx_train_adam(int n, float* p, const float* grad, float* m, float* v, float lr, float beta1, float beta2,
                   float eps, int step, void* stream) {
  if (n < 0 || !p || !grad || !m || !v || step < 1) return 1;
  if (n == 0) return 0;
  const double c1 = 1.0 - std::pow((double)beta1, step), c2 = 1.0 - std::pow((double)beta2, step);
  k_adam<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n, p, grad, m, v, (float)(lr / c1), beta1, beta2,
                                                             (float)c2, eps);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : 4;
}

}  // extern "C"
