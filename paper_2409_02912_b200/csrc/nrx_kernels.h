// Launchers of the device kernels (host-callable, no exceptions).
#pragma once
#include <cuda_runtime.h>

#include "nrx_internal.h"

namespace nrx {

enum ConvEpilogue { EPI_RELU = 0, EPI_STATE_INIT = 1, EPI_RESIDUAL = 2 };

// Arguments of one convolution layer (chunk-planar buffers, see nrx_internal.h).
struct ConvArgs {
  const void* src0; int c0;          // first input buffer and its channel count
  const void* src1; int c1;          // optional second input (concatenated after src0)
  void* dst; int cdst;               // output buffer and its channel count
  float* dst32;                      // bf16 path: fp32 master copy of the state (or null)
  const uint8_t* wbase;              // packed weight blob (device)
  ConvOff off[NRX_MAX_IO];           // per-IO-set weight offsets (1 unless var_io state init)
  int n_off;
  const int32_t* mod_order;          // per-slab modulation order (var_io weight select)
  int mode;                          // ConvEpilogue
};

// One CTA-pair convolution (k_tc_conv_x3.cu): the fp32x3 layers, or a
// bf16 / fp16 ReLU layer without a tail (prec = NRX_FP16 / NRX_BF16).
struct ConvX3Launch {
  const ConvOff* offs;
  int n_off;
  const void* src0;
  int c0;
  const void* src1;
  int c1;
  int src1_xor;
  void* dst;
  int cdst;
  int mode;
  int prec = NRX_FP32X3;
  bool posf = false;  // update.conv0 with the positional channels folded out of K (upd0_posf)
};
int launch_conv_x3(const Geom& g, const ConvX3Launch& c, const uint8_t* wb, const int32_t* mod_order,
                   cudaStream_t st);

int launch_ls_feat(const Geom& g, const void* y, int y_c128, const void* pil, int pil_c128, int n_sets,
                   const float* noise, void* feats, cudaStream_t st);

// fp32 SIMT parity kernels
int launch_conv_simt(const Geom& g, const ConvArgs& a, cudaStream_t st);
int launch_msg_agg_simt(const Geom& g, const PackLayout& L, const uint8_t* wbase, const float* state,
                        float* agg, cudaStream_t st);
int launch_readout_simt(const Geom& g, const PackLayout& L, const uint8_t* wbase, const float* state,
                        const int32_t* mod_order, float* llr, float2* chest, cudaStream_t st);

}  // namespace nrx
