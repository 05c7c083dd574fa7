// Optional per-launch CUDA-event timing (nrx_profile_* in include/nrx_b200.h),
// and NVTX ranges (domain "nrx", one per layer launch) that Nsight tools show
// on the host timeline; without an attached tool an NVTX push is a no-op call.
#include <nvtx3/nvToolsExt.h>

#include <mutex>
#include <vector>

#include "nrx_profile.h"

namespace nrx {

namespace {
struct Record {
  int kid;
  cudaEvent_t a, b;
};
std::mutex g_mu;
bool g_on = false;
uint32_t g_mask = 0;
std::vector<cudaEvent_t> g_pool;
std::vector<Record> g_recs;
size_t g_next = 0;

const char* const kNames[] = {"ls_feat", "state_init.conv0", "state_init.conv1", "msg", "update.conv0",
                              "update.conv1", "readout"};

nvtxDomainHandle_t domain() {
  static nvtxDomainHandle_t d = nvtxDomainCreateA("nrx");
  return d;
}

void range_push(const char* name) {
  nvtxEventAttributes_t a = {};
  a.version = NVTX_VERSION;
  a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
  a.messageType = NVTX_MESSAGE_TYPE_ASCII;
  a.message.ascii = name;
  nvtxDomainRangePushEx(domain(), &a);
}
}  // namespace

NvtxScope::NvtxScope(const char* name) { range_push(name); }
NvtxScope::~NvtxScope() { nvtxDomainRangePop(domain()); }

ProfScope::ProfScope(int kid, cudaStream_t st) : kid_(kid), st_(st), rec_(-1) {
  range_push(kid >= 0 && kid < 7 ? kNames[kid] : "kernel");
  if (!g_on) return;  // racy read is fine: enable/disable are not concurrent with forwards
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_on || !(g_mask >> kid & 1u) || g_next + 2 > g_pool.size()) return;
  Record r{kid, g_pool[g_next], g_pool[g_next + 1]};
  g_next += 2;
  cudaEventRecord(r.a, st);
  rec_ = (int)g_recs.size();
  g_recs.push_back(r);
}

ProfScope::~ProfScope() {
  nvtxDomainRangePop(domain());
  if (rec_ < 0) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEventRecord(g_recs[rec_].b, st_);
}

}  // namespace nrx

using namespace nrx;

extern "C" int nrx_profile_enable(uint32_t kernel_mask, int max_records) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (max_records < 1) return NRX_ERR_INVALID;
  while ((int)g_pool.size() < 2 * max_records) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return NRX_ERR_CUDA;
    g_pool.push_back(e);
  }
  g_recs.clear();
  g_next = 0;
  g_mask = kernel_mask;
  g_on = true;
  return NRX_OK;
}

extern "C" int nrx_profile_collect(int32_t* kernel_ids, float* ms, int cap) {
  std::lock_guard<std::mutex> lk(g_mu);
  int n = 0;
  for (const Record& r : g_recs) {
    if (n >= cap) break;
    if (cudaEventSynchronize(r.b) != cudaSuccess) return -NRX_ERR_CUDA;
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    kernel_ids[n] = r.kid;
    ms[n] = t;
    ++n;
  }
  g_recs.clear();
  g_next = 0;
  return n;
}

extern "C" void nrx_profile_disable(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_on = false;
  g_recs.clear();
  g_next = 0;
}

extern "C" const char* nrx_kernel_name(int kid) {
  static const char* names[] = {"ls_feat", "conv_state_init0", "conv_state_init1", "msg_agg",
                                "conv_update0", "conv_update1", "readout"};
  return (kid >= 0 && kid < 7) ? names[kid] : "unknown";
}
