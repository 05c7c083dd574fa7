// RAII bracket that records CUDA events around one kernel launch when
// nrx_profile_enable() selected its kernel id.
#pragma once
#include <cuda_runtime.h>

#include "nrx_internal.h"

namespace nrx {

enum KernelId { KID_LSFEAT = 0, KID_INIT0 = 1, KID_INIT1 = 2, KID_MSG = 3, KID_UPD0 = 4, KID_UPD1 = 5, KID_READOUT = 6 };

class ProfScope {
 public:
  ProfScope(int kid, cudaStream_t st);
  ~ProfScope();
  ProfScope(const ProfScope&) = delete;
  ProfScope& operator=(const ProfScope&) = delete;

 private:
  int kid_;
  cudaStream_t st_;
  int rec_;
};

// NVTX range (domain "nrx") around a host-side scope, e.g. one nrx_forward call.
class NvtxScope {
 public:
  explicit NvtxScope(const char* name);
  ~NvtxScope();
  NvtxScope(const NvtxScope&) = delete;
  NvtxScope& operator=(const NvtxScope&) = delete;
};

}  // namespace nrx
