// tcgen05 (bf16) path — placeholder until the tensor-core kernels land.
#include "nrx_kernels.h"

namespace nrx {
int launch_forward_tc(const Geom&, const PackLayout&, const WsLayout&, int, const uint8_t*, const int32_t*,
                      uint8_t*, float*, float2*, cudaStream_t) {
  return NRX_ERR_UNSUPPORTED;
}
int tc_launch_count(int n_it) { return 2 + 3 * n_it + 1; }
}  // namespace nrx
