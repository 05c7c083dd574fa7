// fp32 SIMT kernels: the parity mode (NRX_FP32).
//
// They reproduce the reference's float32 arithmetic (autodiff.py conv2d /
// matmul / sum_others) with fp32 FFMA accumulation, so the LLRs agree with
// the CPU reference to ~1e-6 relative (only the summation order differs
// from OpenBLAS).  The tensor-core path (k_tc.cu) is the fast mode.
//
//  k_conv_simt     'same' k x k convolution as an implicit GEMM over the
//                  row-linearised grid (see nrx_internal.h): the 128-row
//                  tile plus its +-H halo rows is staged once in shared
//                  memory (channel-major, conflict-free), every tap is a
//                  row-shifted view of it; one warp owns 8 output channels,
//                  one lane 4 rows.  Epilogues: bias+ReLU (conv0), bias +
//                  positional channels (state init conv1), bias + residual
//                  (iteration conv1, nrx.py:263).
//  k_msg_agg_simt  message MLP of every UE of one slot on a 128-RE tile and
//                  the float64 sum-of-others (autodiff.py:276-294).
//  k_readout_simt  LLR MLP (per-slab IO set for var_io) + channel MLP,
//                  writing the user-facing (N,U,S,T,W) LLR and planar-decoded
//                  complex64 chest layouts directly.
#include <mutex>

#include "nrx_device.cuh"
#include "nrx_kernels.h"

namespace nrx {

constexpr int SIMT_NB = 64;  // output channels per conv block (8 warps x 8)

__global__ void __launch_bounds__(256, 2) k_conv_simt(Geom g, ConvArgs a) {
  extern __shared__ float4 smem4[];
  float* smem = reinterpret_cast<float*>(smem4);
  const int R = NRX_TILE_M + 2 * g.H;
  const int ktap = a.c0 + a.c1;
  float* As = smem;             // [ktap][R]
  float* Ws = smem + ktap * R;  // [ktap][64]
  const int tile = blockIdx.x, slab = blockIdx.y, nb0 = blockIdx.z * SIMT_NB;
  const int p0 = tile * NRX_TILE_M;
  const int nch0 = a.c0 / 4, nch1 = a.c1 / 4, nch = nch0 + nch1;
  const float* s0 = static_cast<const float*>(a.src0);
  const float* s1 = static_cast<const float*>(a.src1);

  for (int idx = threadIdx.x; idx < nch * R; idx += blockDim.x) {
    const int c = idx / R, r = idx - c * R;
    const int row = p0 - g.H + r;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row >= 0 && row < g.rows_slab) {
      const float* p = c < nch0 ? chunk_ptr(s0, slab, nch0, c, row, g) : chunk_ptr(s1, slab, nch1, c - nch0, row, g);
      v = *reinterpret_cast<const float4*>(p);
    }
    As[(4 * c + 0) * R + r] = v.x;
    As[(4 * c + 1) * R + r] = v.y;
    As[(4 * c + 2) * R + r] = v.z;
    As[(4 * c + 3) * R + r] = v.w;
  }

  int io = 0;
  if (a.n_off > 1) {
    io = io_index(a.mod_order, slab, g);
    if (io < 0) io = 0;
  }
  const float* W = reinterpret_cast<const float*>(a.wbase + a.off[io].w);
  const float* bias = reinterpret_cast<const float*>(a.wbase + a.off[io].b);
  const int nw = (a.cdst + 7) / 8 * 8;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = nb0 + warp * 8;
  const bool active = n0 < nw;  // warp-uniform

  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  const int taps = g.ks * g.ks;
  for (int tap = 0; tap < taps; ++tap) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < ktap * 16; idx += blockDim.x) {
      const int k = idx >> 4, q = idx & 15, col = nb0 + q * 4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (col < nw) v = __ldg(reinterpret_cast<const float4*>(W + ((size_t)tap * ktap + k) * nw + col));
      reinterpret_cast<float4*>(Ws)[k * 16 + q] = v;
    }
    __syncthreads();
    if (active) {
      const int ta = tap / g.ks, tb = tap - ta * g.ks;
      const int shift = (ta - g.r) * g.Tp + (tb - g.r);
      const float* Ab = As + g.H + shift + lane;
      const float4* Wb = reinterpret_cast<const float4*>(Ws) + warp * 2;
#pragma unroll 4
      for (int k = 0; k < ktap; ++k) {
        float av[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = Ab[k * R + 32 * i];
        const float4 w0 = Wb[k * 16], w1 = Wb[k * 16 + 1];
        const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], wv[j], acc[i][j]);
      }
    }
  }
  if (!active) return;

  const int u = slab % g.U;
  float* dst = static_cast<float*>(a.dst);
  const int ndst = a.cdst / 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = p0 + lane + 32 * i;
    const int s = row / g.Tp, t = row - s * g.Tp;
    const bool valid = row < g.rows_data && t < g.T;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int c0 = n0 + 4 * half;
      if (c0 >= a.cdst) continue;
      float* p = chunk_ptr(dst, slab, ndst, c0 / 4, row, g);
      float old[4] = {0.f, 0.f, 0.f, 0.f};
      if (a.mode == EPI_RESIDUAL) {
        const float4 o = *reinterpret_cast<const float4*>(p);
        old[0] = o.x; old[1] = o.y; old[2] = o.z; old[3] = o.w;
      }
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = c0 + e;
        float val = 0.f;
        if (valid) {
          if (c < g.d) {
            float x = acc[i][4 * half + e] + bias[c];
            if (a.mode == EPI_RELU) x = relu_f(x);
            else if (a.mode == EPI_RESIDUAL) x = old[e] + x;
            val = x;
          } else if (a.mode != EPI_RELU) {
            val = state_extra(c, s, t, u, g);
          }
        }
        v[e] = val;
      }
      store_chunk(p, v);
    }
  }
}

static size_t conv_simt_smem(const Geom& g, int ktap) {
  return (size_t)ktap * (NRX_TILE_M + 2 * g.H + SIMT_NB) * sizeof(float);
}

int launch_conv_simt(const Geom& g, const ConvArgs& a, cudaStream_t st) {
  static std::once_flag once[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(once[dev & 63], [] {
    cudaFuncSetAttribute(k_conv_simt, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  const size_t smem = conv_simt_smem(g, a.c0 + a.c1);
  if (smem > 200 * 1024) return NRX_ERR_UNSUPPORTED;
  dim3 grid(g.tiles, g.NU, cdiv(rup(a.cdst, 8), SIMT_NB));
  k_conv_simt<<<grid, 256, smem, st>>>(g, a);
  return cudaPeekAtLastError() == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

// ---------------------------------------------------------------------------
// message MLP + float64 sum of the other UEs' messages
// ---------------------------------------------------------------------------

template <int DM>
__device__ __forceinline__ void load_state_row(const Geom& g, const float* state, int slab, int row, float* x) {
  const int nch = g.Cs / 4;
#pragma unroll
  for (int c4 = 0; c4 < DM / 4; ++c4) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c4 * 4 < g.d) v = *reinterpret_cast<const float4*>(chunk_ptr(state, slab, nch, c4, row, g));
    x[4 * c4 + 0] = 4 * c4 + 0 < g.d ? v.x : 0.f;
    x[4 * c4 + 1] = 4 * c4 + 1 < g.d ? v.y : 0.f;
    x[4 * c4 + 2] = 4 * c4 + 2 < g.d ? v.z : 0.f;
    x[4 * c4 + 3] = 4 * c4 + 3 < g.d ? v.w : 0.f;
  }
}

template <int DM>
__global__ void __launch_bounds__(128) k_msg_agg_simt(Geom g, const uint8_t* __restrict__ wb, MlpOff o,
                                                      const float* __restrict__ state, float* __restrict__ agg) {
  extern __shared__ double smd[];
  double* tot = smd;                                   // [DM][128]
  float* W0 = reinterpret_cast<float*>(smd + DM * 128);  // [DM][h]
  float* b0 = W0 + DM * g.h;
  float* W1 = b0 + g.h;                                // [h][DM]
  float* b1 = W1 + g.h * DM;
  {
    const float* s0 = reinterpret_cast<const float*>(wb + o.w0);
    const float* sb0 = reinterpret_cast<const float*>(wb + o.b0);
    const float* s1 = reinterpret_cast<const float*>(wb + o.w1);
    const float* sb1 = reinterpret_cast<const float*>(wb + o.b1);
    for (int i = threadIdx.x; i < DM * g.h; i += blockDim.x) W0[i] = s0[i];
    for (int i = threadIdx.x; i < g.h; i += blockDim.x) b0[i] = sb0[i];
    for (int i = threadIdx.x; i < g.h * DM; i += blockDim.x) W1[i] = s1[i];
    for (int i = threadIdx.x; i < DM; i += blockDim.x) b1[i] = sb1[i];
  }
  __syncthreads();
  const int row = blockIdx.x * NRX_TILE_M + threadIdx.x;
  const int n = blockIdx.y;
  const int s = row / g.Tp, t = row - s * g.Tp;
  const bool valid = row < g.rows_data && t < g.T;
  const int ncha = g.Ca / 4;

  for (int u = 0; u < g.U; ++u) {
    const int slab = n * g.U + u;
    float msg[DM];
#pragma unroll
    for (int c = 0; c < DM; ++c) msg[c] = 0.f;
    if (valid) {
      float x[DM];
      load_state_row<DM>(g, state, slab, row, x);
      for (int j = 0; j < g.h; ++j) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < DM; ++i) acc = fmaf(x[i], W0[i * g.h + j], acc);
        const float hj = relu_f(acc + b0[j]);
#pragma unroll
        for (int c = 0; c < DM; ++c) msg[c] = fmaf(hj, W1[j * DM + c], msg[c]);
      }
#pragma unroll
      for (int c = 0; c < DM; ++c) msg[c] = msg[c] + b1[c];
    }
#pragma unroll
    for (int c4 = 0; c4 < DM / 4; ++c4)
      if (c4 < ncha) store_chunk(chunk_ptr(agg, slab, ncha, c4, row, g), msg + 4 * c4);
#pragma unroll
    for (int c = 0; c < DM; ++c) {
      const double v = (double)msg[c];
      tot[c * NRX_TILE_M + threadIdx.x] = u == 0 ? v : tot[c * NRX_TILE_M + threadIdx.x] + v;
    }
  }
  // agg_u = f32(sum_v f64(m_v) - f64(m_u)); exactly 0 for a single UE
  for (int u = 0; u < g.U; ++u) {
    const int slab = n * g.U + u;
#pragma unroll
    for (int c4 = 0; c4 < DM / 4; ++c4) {
      if (c4 >= ncha) continue;
      float* p = chunk_ptr(agg, slab, ncha, c4, row, g);
      const float4 m = *reinterpret_cast<const float4*>(p);
      const float mv[4] = {m.x, m.y, m.z, m.w};
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int c = 4 * c4 + e;
        v[e] = (valid && c < g.d) ? (float)(tot[c * NRX_TILE_M + threadIdx.x] - (double)mv[e]) : 0.f;
      }
      store_chunk(p, v);
    }
  }
}

template <int DM>
static int launch_msg_agg_t(const Geom& g, const PackLayout& L, const uint8_t* wb, const float* state, float* agg,
                            cudaStream_t st) {
  const size_t smem = DM * NRX_TILE_M * sizeof(double) + (size_t)(2 * DM * g.h + g.h + DM) * sizeof(float);
  static std::once_flag once[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(once[dev & 63], [] {
    cudaFuncSetAttribute(k_msg_agg_simt<DM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  if (smem > 200 * 1024) return NRX_ERR_UNSUPPORTED;
  k_msg_agg_simt<DM><<<dim3(g.tiles, g.N), NRX_TILE_M, smem, st>>>(g, wb, L.msg, state, agg);
  return cudaPeekAtLastError() == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

int launch_msg_agg_simt(const Geom& g, const PackLayout& L, const uint8_t* wb, const float* state, float* agg,
                        cudaStream_t st) {
  switch (L.dmax) {
    case 16: return launch_msg_agg_t<16>(g, L, wb, state, agg, st);
    case 32: return launch_msg_agg_t<32>(g, L, wb, state, agg, st);
    case 64: return launch_msg_agg_t<64>(g, L, wb, state, agg, st);
    default: return NRX_ERR_UNSUPPORTED;
  }
}

// ---------------------------------------------------------------------------
// readouts: LLR MLP (IO set per slab) + channel-estimate MLP
// ---------------------------------------------------------------------------

struct ReadoutOff {
  MlpOff llr[NRX_MAX_IO];
  MlpOff chest;
};

template <int DM>
__global__ void __launch_bounds__(128) k_readout_simt(Geom g, const uint8_t* __restrict__ wb, ReadoutOff ro,
                                                      const float* __restrict__ state,
                                                      const int32_t* __restrict__ mod_order,
                                                      float* __restrict__ llr, float2* __restrict__ chest) {
  extern __shared__ float4 smr4[];
  float* sm = reinterpret_cast<float*>(smr4);
  const int slab = blockIdx.y;
  const int io = io_index(mod_order, slab, g);
  const MlpOff lo = ro.llr[io < 0 ? 0 : io];
  const MlpOff co = ro.chest;
  const int h = g.h;
  float* lW0 = sm;               // [DM][h]
  float* lb0 = lW0 + DM * h;
  float* lW1 = lb0 + h;          // [h][8]
  float* lb1 = lW1 + h * 8;
  float* cW0 = lb1 + 8;          // [DM][h]
  float* cb0 = cW0 + DM * h;
  float* cW1 = cb0 + h;          // [h][16]
  float* cb1 = cW1 + h * 16;
  auto cp = [&](float* d, size_t off, int n) {
    const float* s = reinterpret_cast<const float*>(wb + off);
    for (int i = threadIdx.x; i < n; i += blockDim.x) d[i] = s[i];
  };
  cp(lW0, lo.w0, DM * h); cp(lb0, lo.b0, h); cp(lW1, lo.w1, h * 8); cp(lb1, lo.b1, 8);
  cp(cW0, co.w0, DM * h); cp(cb0, co.b0, h); cp(cW1, co.w1, h * 16); cp(cb1, co.b1, 16);
  __syncthreads();

  const int row = blockIdx.x * NRX_TILE_M + threadIdx.x;
  const int s = row / g.Tp, t = row - s * g.Tp;
  if (row >= g.rows_data || t >= g.T) return;
  float x[DM];
  load_state_row<DM>(g, state, slab, row, x);
  float ol[8], oc[16];
#pragma unroll
  for (int c = 0; c < 8; ++c) ol[c] = 0.f;
#pragma unroll
  for (int c = 0; c < 16; ++c) oc[c] = 0.f;
  for (int j = 0; j < h; ++j) {
    float al = 0.f, ac = 0.f;
#pragma unroll
    for (int i = 0; i < DM; ++i) {
      al = fmaf(x[i], lW0[i * h + j], al);
      ac = fmaf(x[i], cW0[i * h + j], ac);
    }
    const float hl = relu_f(al + lb0[j]), hc = relu_f(ac + cb0[j]);
#pragma unroll
    for (int c = 0; c < 8; ++c) ol[c] = fmaf(hl, lW1[j * 8 + c], ol[c]);
#pragma unroll
    for (int c = 0; c < 16; ++c) oc[c] = fmaf(hc, cW1[j * 16 + c], oc[c]);
  }
  const size_t re = ((size_t)slab * g.S + s) * g.T + t;
  const int width = io < 0 ? 0 : g.io_width[io];
  float* lp = llr + re * g.llr_width;
  for (int c = 0; c < g.llr_width; ++c) {
    float v = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q == c) v = ol[q] + lb1[q];
    lp[c] = io < 0 ? __int_as_float(0x7fc00000) : (c < width ? v : 0.f);
  }
  float2* cp2 = chest + re * g.B;
  for (int b = 0; b < g.B; ++b) {
    float re_v = 0.f, im_v = 0.f;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (q == b) re_v = oc[q] + cb1[q];
      if (q == g.B + b) im_v = oc[q] + cb1[q];
    }
    cp2[b] = make_float2(re_v, im_v);
  }
}

template <int DM>
static int launch_readout_t(const Geom& g, const PackLayout& L, const uint8_t* wb, const float* state,
                            const int32_t* mod_order, float* llr, float2* chest, cudaStream_t st) {
  ReadoutOff ro;
  for (int i = 0; i < NRX_MAX_IO; ++i) ro.llr[i] = L.llr[i];
  ro.chest = L.chest;
  const size_t smem = (size_t)(2 * DM * g.h + 2 * g.h + 8 * g.h + 8 + 16 * g.h + 16) * sizeof(float);
  static std::once_flag once[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(once[dev & 63], [] {
    cudaFuncSetAttribute(k_readout_simt<DM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  if (smem > 200 * 1024) return NRX_ERR_UNSUPPORTED;
  k_readout_simt<DM><<<dim3(g.tiles, g.NU), NRX_TILE_M, smem, st>>>(g, wb, ro, state, mod_order, llr, chest);
  return cudaPeekAtLastError() == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

int launch_readout_simt(const Geom& g, const PackLayout& L, const uint8_t* wb, const float* state,
                        const int32_t* mod_order, float* llr, float2* chest, cudaStream_t st) {
  switch (L.dmax) {
    case 16: return launch_readout_t<16>(g, L, wb, state, mod_order, llr, chest, st);
    case 32: return launch_readout_t<32>(g, L, wb, state, mod_order, llr, chest, st);
    case 64: return launch_readout_t<64>(g, L, wb, state, mod_order, llr, chest, st);
    default: return NRX_ERR_UNSUPPORTED;
  }
}

}  // namespace nrx
