/*
 * nrx_train.h — C ABI of the hand-written training kernels (libnrx_b200.so).
 *
 * The reference trains the NRX with its own numpy autodiff on the CPU
 * (/root/reference/pkg/src/nrxsim/training.py:180-234 train_step,
 * autodiff.py:302-350 conv2d + its VJP, autodiff.py:428-525 Adam).  These
 * entry points are that step's heavy operators on the GPU, in fp32:
 *
 *   nrx_train_conv_fwd    conv2d 'same' (autodiff.py:302-350), NHWC x (n,S,T,cin),
 *                         w (k,k,cin,cout), optional bias; a dense layer x @ w
 *                         (autodiff matmul) is the k = 1, T = 1 case
 *   nrx_train_conv_dgrad  its input gradient (the conv2d VJP w.r.t. x)
 *   nrx_train_conv_wgrad  its kernel / bias gradients (VJP w.r.t. w, b), overwritten
 *   nrx_train_adam        one bias-corrected Adam update of a parameter tensor
 *                         (AdamState / adam_step, autodiff.py:485-525)
 *
 * All pointers are device pointers; each call enqueues on `stream` (a
 * cudaStream_t) and returns 0, 1 (bad argument / shape beyond the limits:
 * cin, cout <= 128, odd k) or 4 (CUDA error).
 *
 * Tensor-core versions (csrc/k_train_tc.cu): the same three operators as
 * fp32x3 GEMMs on tcgen05 (fp16 hi / lo operand planes with per-tensor
 * power-of-two scales, fp32 accumulation) over a caller-owned
 * device workspace of nrx_train_tc_workspace(...) bytes (0: unsupported
 * shape; cin, cout <= 128, odd k).  No bias: the graph adds it.
 */
#ifndef NRX_TRAIN_H_
#define NRX_TRAIN_H_

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

int nrx_train_conv_fwd(int n, int S, int T, int cin, int cout, int k, const float* x, const float* w,
                       const float* b, float* y, void* stream);
int nrx_train_conv_dgrad(int n, int S, int T, int cin, int cout, int k, const float* dy, const float* w,
                         float* dx, void* stream);
int nrx_train_conv_wgrad(int n, int S, int T, int cin, int cout, int k, const float* x, const float* dy, float* dw,
                         float* db, void* stream);
int nrx_train_adam(int n, float* p, const float* grad, float* m, float* v, float lr, float beta1, float beta2,
                   float eps, int step, void* stream);

size_t nrx_train_tc_workspace(int n, int S, int T, int cin, int cout, int k);
int nrx_train_conv_tc_fwd(int n, int S, int T, int cin, int cout, int k, const float* x, const float* w, float* y,
                          void* workspace, size_t workspace_bytes, void* stream);
int nrx_train_conv_tc_dgrad(int n, int S, int T, int cin, int cout, int k, const float* dy, const float* w,
                            float* dx, void* workspace, size_t workspace_bytes, void* stream);
int nrx_train_conv_tc_wgrad(int n, int S, int T, int cin, int cout, int k, const float* x, const float* dy,
                            float* dw, void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NRX_TRAIN_H_ */
