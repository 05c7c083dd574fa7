// nrx_forward: the C-ABI entry point (include/nrx_b200.h) — enqueues the
// whole receiver forward pass for a batch of slots on one stream.
//
// Launch sequence (nrx_forward_graph, nrx.py:302-342, training=False):
//   K1  ls_feat                      LS + features            (nrx.py:205-213, 184-202)
//   K2  conv  feats -> h             state_init conv0 + ReLU  (nrx.py:232-234, 237-249)
//   K2  conv  h -> state             state_init conv1 (+ pos channels)
//   per iteration (nrx.py:252-263, weights shared across iterations):
//   K3a msg_agg  state -> agg        message MLP + fp64 sum of others
//   K3b conv  [state|agg] -> h       update conv0 + ReLU (concat never materialised)
//   K3c conv  h -> state             update conv1 + bias + residual
//   K4  readout state -> llr, chest  (nrx.py:266-281, 382-384)
#include <cstring>

#include "nrx_kernels.h"
#include "nrx_profile.h"

namespace nrx {
int make_geom(const nrx_model_desc* m, const nrx_slot_desc* s, int n_slots, int prec, Geom* g);
void pack_layout(const nrx_model_desc* m, int prec, PackLayout* L);
void ws_layout(const Geom& g, WsLayout* w);
int launch_forward_tc(const Geom& g, const PackLayout& L, const WsLayout& W, int n_it, const uint8_t* wb,
                      const int32_t* mod_order, uint8_t* ws, float* llr, float2* chest, cudaStream_t st);
int tc_launch_count(int n_it, int num_ues);
int launch_forward_x3(const Geom& g, const PackLayout& L, const WsLayout& W, int n_it, const uint8_t* wb,
                      const int32_t* mod_order, uint8_t* ws, float* llr, float2* chest, cudaStream_t st);
}  // namespace nrx

using namespace nrx;

#define NRX_TRY(x)          \
  do {                      \
    int _s = (x);           \
    if (_s != NRX_OK) return _s; \
  } while (0)

static int forward_simt(const Geom& g, const PackLayout& L, const WsLayout& W, int n_it, const uint8_t* wb,
                        const int32_t* mod_order, uint8_t* ws, float* llr, float2* chest, cudaStream_t st) {
  float* feats = reinterpret_cast<float*>(ws + W.feats);
  float* h = reinterpret_cast<float*>(ws + W.h);
  float* state = reinterpret_cast<float*>(ws + W.state);
  float* agg = reinterpret_cast<float*>(ws + W.agg);

  ConvArgs a{};
  a.wbase = wb;
  a.mod_order = mod_order;
  // state init, conv0: feats -> h
  a.src0 = feats; a.c0 = g.Cf; a.src1 = nullptr; a.c1 = 0;
  a.dst = h; a.cdst = g.Ch; a.mode = EPI_RELU;
  a.n_off = g.n_io;
  for (int i = 0; i < g.n_io; ++i) a.off[i] = L.init0[i];
  { ProfScope p(KID_INIT0, st); NRX_TRY(launch_conv_simt(g, a, st)); }
  // state init, conv1: h -> state
  a.src0 = h; a.c0 = g.Ch; a.dst = state; a.cdst = g.Cs; a.mode = EPI_STATE_INIT;
  for (int i = 0; i < g.n_io; ++i) a.off[i] = L.init1[i];
  { ProfScope p(KID_INIT1, st); NRX_TRY(launch_conv_simt(g, a, st)); }
  for (int it = 0; it < n_it; ++it) {
    { ProfScope p(KID_MSG, st); NRX_TRY(launch_msg_agg_simt(g, L, wb, state, agg, st)); }
    ConvArgs c{};
    c.wbase = wb; c.n_off = 1;
    c.src0 = state; c.c0 = g.Cs; c.src1 = agg; c.c1 = g.Ca;
    c.dst = h; c.cdst = g.Ch; c.mode = EPI_RELU; c.off[0] = L.upd0;
    { ProfScope p(KID_UPD0, st); NRX_TRY(launch_conv_simt(g, c, st)); }
    c.src0 = h; c.c0 = g.Ch; c.src1 = nullptr; c.c1 = 0;
    c.dst = state; c.cdst = g.Cs; c.mode = EPI_RESIDUAL; c.off[0] = L.upd1;
    { ProfScope p(KID_UPD1, st); NRX_TRY(launch_conv_simt(g, c, st)); }
  }
  ProfScope p(KID_READOUT, st);
  return launch_readout_simt(g, L, wb, state, mod_order, llr, chest, st);
}

extern "C" int nrx_forward(const nrx_model_desc* model, const nrx_slot_desc* slot, int n_slots, int precision,
                           int num_iterations, const void* y, int y_c128, const void* pilots, int pilots_c128,
                           int n_pilot_sets, const float* noise_feat, const int32_t* mod_order,
                           const void* packed_weights, float* llr_out, int llr_width, void* chest_out,
                           void* workspace, size_t workspace_bytes, void* stream) {
  NvtxScope range("nrx_forward");
  Geom g;
  NRX_TRY(make_geom(model, slot, n_slots, precision, &g));
  if (num_iterations < 1 || num_iterations > model->num_iterations) return NRX_ERR_DEPTH;
  if (!y || !pilots || !packed_weights || !llr_out || !chest_out || !workspace) return NRX_ERR_INVALID;
  if (model->include_noise_plane && !noise_feat) return NRX_ERR_INVALID;
  if (model->variant == NRX_VAR_IO && !mod_order) return NRX_ERR_INVALID;
  if (n_pilot_sets != 1 && n_pilot_sets != n_slots) return NRX_ERR_INVALID;
  if (llr_width < 1 || llr_width > 8) return NRX_ERR_INVALID;
  g.llr_width = llr_width;
  WsLayout W;
  ws_layout(g, &W);
  if (workspace_bytes < W.total) return NRX_ERR_WORKSPACE;
  PackLayout L;
  pack_layout(model, precision, &L);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const uint8_t* wb = static_cast<const uint8_t*>(packed_weights);
  // range guard of the half-precision operand modes: the readouts set this
  // word when an output is not finite (fp16 planes overflow above 65504)
  g.flag = precision == NRX_FP32 ? nullptr : reinterpret_cast<uint32_t*>(ws + W.flag);
  if (g.flag && cudaMemsetAsync(g.flag, 0, 4, st) != cudaSuccess) return NRX_ERR_CUDA;

  {
    ProfScope p(KID_LSFEAT, st);
    NRX_TRY(launch_ls_feat(g, y, y_c128, pilots, pilots_c128, n_pilot_sets, noise_feat, ws + W.feats, st));
  }
  if (precision == NRX_FP32)
    return forward_simt(g, L, W, num_iterations, wb, mod_order, ws, llr_out, static_cast<float2*>(chest_out), st);
  if (precision == NRX_FP32X3)
    return launch_forward_x3(g, L, W, num_iterations, wb, mod_order, ws, llr_out, static_cast<float2*>(chest_out),
                             st);
  return launch_forward_tc(g, L, W, num_iterations, wb, mod_order, ws, llr_out, static_cast<float2*>(chest_out), st);
}

extern "C" int nrx_forward_launch_count(const nrx_model_desc* model, const nrx_slot_desc* slot, int precision,
                                        int num_iterations) {
  if (!model || !slot || num_iterations < 1) return -1;
  if (precision == NRX_FP32 || precision == NRX_FP32X3) return 1 + 2 + 3 * num_iterations + 1;
  return 1 + tc_launch_count(num_iterations, slot->num_ues);
}

extern "C" int nrx_buffer_geometry(const nrx_model_desc* model, const nrx_slot_desc* slot, int precision,
                                   int32_t* out8) {
  Geom g;
  NRX_TRY(make_geom(model, slot, 1, precision, &g));
  if (!out8) return NRX_ERR_INVALID;
  const int32_t v[8] = {g.rows_slab, g.Tp, g.Cf, g.Cs, g.Ch, g.Ca, g.cw, g.tiles};
  std::memcpy(out8, v, sizeof(v));
  return NRX_OK;
}

extern "C" int nrx_ls_features(const nrx_model_desc* model, const nrx_slot_desc* slot, int n_slots,
                               int precision, const void* y, int y_c128, const void* pilots, int pilots_c128,
                               int n_pilot_sets, const float* noise_feat, void* feats_out, void* stream) {
  Geom g;
  NRX_TRY(make_geom(model, slot, n_slots, precision, &g));
  if (!y || !pilots || !feats_out || (model->include_noise_plane && !noise_feat)) return NRX_ERR_INVALID;
  if (n_pilot_sets != 1 && n_pilot_sets != n_slots) return NRX_ERR_INVALID;
  return launch_ls_feat(g, y, y_c128, pilots, pilots_c128, n_pilot_sets, noise_feat, feats_out,
                        reinterpret_cast<cudaStream_t>(stream));
}
