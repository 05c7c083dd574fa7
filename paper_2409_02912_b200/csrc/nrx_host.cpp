// Host-side pieces of the C ABI that need no GPU: descriptor validation,
// geometry, canonical weight naming (expected_shapes, nrx.py:92-120), the
// packed-weight layout + repacker, and the workspace layout.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "nrx_internal.h"

namespace nrx {

namespace {

struct TensorSpec {
  std::string name;
  std::vector<int> shape;
};

int input_channels(const nrx_model_desc* m) {
  return 4 * m->num_rx_ant + 2 + (m->include_noise_plane ? 1 : 0);
}

int llr_width_of(const nrx_model_desc* m, int io) {
  return m->variant == NRX_VAR_IO ? m->io_orders[io] : m->m_max;
}

// Canonical tensor list, documented in include/nrx_b200.h.
std::vector<TensorSpec> canonical(const nrx_model_desc* m) {
  std::vector<TensorSpec> v;
  const int k = m->kernel_size, d = m->d_s, h = m->hidden, cin = input_channels(m);
  auto conv_block = [&](const std::string& p, int c0) {
    v.push_back({p + ".conv0.w", {k, k, c0, d}});
    v.push_back({p + ".conv0.b", {d}});
    v.push_back({p + ".conv1.w", {k, k, d, d}});
    v.push_back({p + ".conv1.b", {d}});
  };
  auto mlp = [&](const std::string& p, int out) {
    v.push_back({p + ".fc0.w", {d, h}});
    v.push_back({p + ".fc0.b", {h}});
    v.push_back({p + ".fc1.w", {h, out}});
    v.push_back({p + ".fc1.b", {out}});
  };
  for (int i = 0; i < m->n_io; ++i) {
    std::string tag = m->variant == NRX_VAR_IO ? ".m" + std::to_string(m->io_orders[i]) : "";
    conv_block("state_init" + tag, cin);
    mlp("readout_llr" + tag, llr_width_of(m, i));
  }
  mlp("iteration.msg", d);
  conv_block("iteration.update", 2 * d + 2);
  mlp("readout_chest", 2 * m->num_rx_ant);
  return v;
}

int64_t numel(const TensorSpec& t) {
  int64_t n = 1;
  for (int s : t.shape) n *= s;
  return n;
}

}  // namespace

int validate(const nrx_model_desc* m, const nrx_slot_desc* s) {
  if (!m) return NRX_ERR_INVALID;
  if (m->d_s < 4 || m->num_iterations < 1 || m->kernel_size < 1 || m->kernel_size % 2 == 0)
    return NRX_ERR_INVALID;
  if (m->variant < 0 || m->variant > 2 || m->n_io < 1 || m->n_io > NRX_MAX_IO) return NRX_ERR_INVALID;
  if (m->variant != NRX_VAR_IO && m->n_io != 1) return NRX_ERR_INVALID;
  if (m->hidden < 1 || m->num_rx_ant < 1 || m->m_max < 1) return NRX_ERR_INVALID;
  for (int i = 0; i < m->n_io; ++i)
    if (m->io_orders[i] < 1 || m->io_orders[i] > m->m_max) return NRX_ERR_INVALID;
  // implementation limits
  if (m->d_s > 64 || m->hidden > 256 || m->num_rx_ant > 8 || m->m_max > 8) return NRX_ERR_UNSUPPORTED;
  if (m->kernel_size > 5) return NRX_ERR_UNSUPPORTED;
  if (!s) return NRX_OK;
  if (s->num_subcarriers < 1 || s->num_symbols < 1 || s->num_ues < 1 || s->comb_size < 1) return NRX_ERR_INVALID;
  if (s->num_ues > s->comb_size) return NRX_ERR_INVALID;
  if (s->num_pilot_symbols < 1 || s->num_pilot_symbols > NRX_MAX_PILOT_SYMBOLS) return NRX_ERR_INVALID;
  for (int i = 0; i < s->num_pilot_symbols; ++i)
    if (s->pilot_symbols[i] < 0 || s->pilot_symbols[i] >= s->num_symbols) return NRX_ERR_INVALID;
  if (s->num_subcarriers < s->comb_size) return NRX_ERR_UNSUPPORTED;  // every UE needs a pilot
  if (s->num_symbols > 32 || s->num_ues > 8) return NRX_ERR_UNSUPPORTED;
  return NRX_OK;
}

int quantum(int prec) { return prec == NRX_FP32 ? 4 : 16; }

// Largest padded MLP hidden width per mode: the message / readout MLPs keep two
// hidden tiles and the readout's N = 2 hidden GEMM in TMEM and shared memory
// (fp16 / bf16: the fused readout tail next to the convolution accumulators;
// fp32x3: hi and lo planes of the hidden tile).
int hidden_limit(int prec) { return prec == NRX_FP32 ? 256 : prec == NRX_FP32X3 ? 96 : 64; }
constexpr size_t kResidentLimit = 170 * 1024;
size_t resident_conv_bytes(int ks, int d, int prec) {
  const int np = prec == NRX_FP32X3 ? x3_np(d) : rup(d, 16);
  return (size_t)ks * ks * (rup(d + 2, 16) + rup(d, 16)) * np * 2;
}

int make_geom(const nrx_model_desc* m, const nrx_slot_desc* s, int n_slots, int prec, Geom* g) {
  int st = validate(m, s);
  if (st) return st;
  if (n_slots < 1) return NRX_ERR_INVALID;
  if (prec != NRX_FP32 && prec != NRX_BF16 && prec != NRX_FP16 && prec != NRX_FP32X3) return NRX_ERR_INVALID;
  if (hidden_limit(prec) < rup(m->hidden, 16)) return NRX_ERR_UNSUPPORTED;
  std::memset(g, 0, sizeof(*g));
  g->N = n_slots;
  g->U = s->num_ues;
  g->NU = n_slots * s->num_ues;
  g->S = s->num_subcarriers;
  g->T = s->num_symbols;
  g->B = m->num_rx_ant;
  g->comb = s->comb_size;
  // (s - o) / comb as __umulhi(s - o, ceil(2^32 / comb)) is exact while (s - o) * comb^2 < 2^32
  if ((uint64_t)s->num_subcarriers * (uint64_t)s->comb_size * (uint64_t)s->comb_size >= (1ull << 32))
    return NRX_ERR_UNSUPPORTED;
  g->comb_magic = s->comb_size > 1 ? (uint32_t)(((1ull << 32) + s->comb_size - 1) / s->comb_size) : 0u;
  for (int k = 0; k < 16; ++k)  // IEEE float division, as __fdiv_rn((float)k, (float)S) on the device
    g->df_tab[k] = (float)k / (float)s->num_subcarriers;
  g->K = s->num_pilot_symbols;
  for (int i = 0; i < g->K; ++i) g->ps[i] = s->pilot_symbols[i];
  g->ks = m->kernel_size;
  g->r = m->kernel_size / 2;
  g->Tp = g->T + g->r;
  g->inv_Tp = 1.0f / (float)g->Tp;
  g->H = g->r * g->Tp + g->r;
  g->rows_data = g->S * g->Tp;
  g->rows_slab = rup(g->rows_data, NRX_TILE_M);
  g->tiles = g->rows_slab / NRX_TILE_M;
  if (g->rows_slab >= (1 << 21)) return NRX_ERR_UNSUPPORTED;   // row_to_st exactness bound
  g->d = m->d_s;
  g->h = m->hidden;
  g->prec = prec;
  g->cw = prec == NRX_FP32 ? 4 : 8;
  const int q = quantum(prec);
  g->Cin = input_channels(m);
  g->Cf = rup(g->Cin, q);
  g->Cs = rup(g->d + 2, q);
  g->Ch = rup(g->d, q);
  g->Ca = rup(g->d, q);
  // tensor-core modes keep a layer's weights resident in shared memory: update.conv0
  // (taps x (Cs + Ca) x np fp16, the largest layer) must leave room for two pipeline
  // stages (e.g. 5x5 kernels fit up to d_s = 32)
  if (prec != NRX_FP32 && resident_conv_bytes(g->ks, g->d, prec) > kResidentLimit) return NRX_ERR_UNSUPPORTED;
  // the standalone message kernel (fp32x3: every U; bf16 / fp16: U != 2) holds two
  // hidden tiles and the U message tiles of a slot in TMEM (512 columns)
  if (prec != NRX_FP32 && (prec == NRX_FP32X3 || g->U != 2) &&
      2 * rup(m->hidden, 16) + 2 * g->U * rup(g->d, 16) > 512)
    return NRX_ERR_UNSUPPORTED;
  g->n_io = m->n_io;
  int w = 0;
  for (int i = 0; i < m->n_io; ++i) {
    g->io_orders[i] = m->io_orders[i];
    g->io_width[i] = llr_width_of(m, i);
    if (g->io_width[i] > w) w = g->io_width[i];
  }
  g->llr_width = w;
  g->noise_plane = m->include_noise_plane;
  g->freq_enc = m->include_freq_encoding;
  // positional encoding along t (nrx.py:164): float32(min|t - ps| / T)
  for (int t = 0; t < g->T; ++t) {
    int best = 1 << 30, arg = 0;
    for (int k = 0; k < g->K; ++k) {
      int dd = std::abs(t - g->ps[k]);
      if (dd < best) { best = dd; arg = k; }  // strict: ties keep the earlier symbol
    }
    g->dt[t] = (float)((double)best / (double)g->T);
    g->nearest[t] = arg;
  }
  return NRX_OK;
}

int dmax_of(int d) { return d <= 16 ? 16 : d <= 32 ? 32 : 64; }

// ---- packed weight layout ------------------------------------------------
//
// FP32 (SIMT kernels):
//   conv  w: [tap][ktap][nw] float, ktap = buffer input channels, nw = output
//         buffer channels rounded to 8; b: [nw]
//   mlp   w0: [dmax][h], b0: [h], w1: [h][outp], b1: [outp]
//         (outp = dmax for msg, 8 for the LLR readout, 16 for the chest)
// BF16 (tcgen05 kernels): every GEMM operand B is stored as W^T in the
// K-major no-swizzle core-matrix layout the MMA reads from shared memory,
// [K/8][N][8] bf16 (element (n, k) at ((k/8)*N + n)*8 + k%8); biases fp32.
//   conv      w: K = taps*ktap (tap-major, then buffer channel), N = np
//   msg       w0: K = Cs, N = hp;  w1: K = hp, N = np
//   readout   (per IO set, LLR and chest MLPs fused) w0: K = Cs, N = 2hp
//             ([llr hidden | chest hidden]);  w1: K = 2hp, N = 32 block
//             diagonal (outputs 0..7 LLR, 8..8+2B chest)
// with np = rup(d,16), hp = rup(h,16).
void pack_layout(const nrx_model_desc* m, int prec, PackLayout* L) {
  Geom g;
  nrx_slot_desc s{};
  s.num_subcarriers = 64; s.num_symbols = 14; s.num_ues = 1; s.comb_size = 1;
  s.num_pilot_symbols = 1; s.pilot_symbols[0] = 0;
  make_geom(m, &s, 1, prec, &g);
  std::memset(L, 0, sizeof(*L));
  const int taps = m->kernel_size * m->kernel_size;
  const int dmax = dmax_of(m->d_s);
  L->dmax = dmax;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
  if (prec == NRX_FP32X3) {  // fp16 hi/lo operand pairs, CTA-pair convolutions
    const int npx = x3_np(m->d_s), np = rup(m->d_s, 16), hp = rup(m->hidden, 16);
    auto conv = [&](ConvOff& c, int ktap, bool posf = false) {
      c.ktap = ktap;
      c.w = take((size_t)taps * ktap * npx * 2 * 2);  // [rank 0: W_hi | rank 1: W_lo][K/8][npx][8]
      c.b = take((size_t)(posw_off(npx) + (posf ? 2 * taps * npx : 0)) * 4);  // bias, descale 2^-E, pos weights
    };
    auto mlp = [&](MlpOff& o, int k0, int n0, int n1) {
      o.out = n1;
      o.w0 = take((size_t)k0 * n0 * 2 * 2);  // [hi|lo][K/8][N][8]
      o.b0 = take((size_t)(n0 + 4) * 4);
      o.w1 = take((size_t)n0 * n1 * 2 * 2);
      o.b1 = take((size_t)(n1 + 4) * 4);
    };
    for (int i = 0; i < m->n_io; ++i) {
      conv(L->init0[i], g.Cf);
      conv(L->init1[i], g.Ch);
      mlp(L->llr[i], g.Cs, 2 * hp, 32);
    }
    mlp(L->msg, g.Cs, hp, np);
    const bool posf = upd0_posf(m->d_s, m->kernel_size, NRX_FP32X3);
    conv(L->upd0, posf ? 2 * m->d_s : g.Cs + g.Ca, posf);
    conv(L->upd1, g.Ch);
    L->total = off;
    return;
  }
  if (prec != NRX_FP32) {  // bf16 / fp16 tensor-core operands
    const int np = rup(m->d_s, 16), hp = rup(m->hidden, 16);
    auto conv = [&](ConvOff& c, int ktap) {
      c.ktap = ktap;
      c.w = take((size_t)taps * ktap * np * 2);
      c.b = take((size_t)np * 4);
    };
    auto mlp = [&](MlpOff& o, int k0, int n0, int n1) {
      o.out = n1;
      o.w0 = take((size_t)k0 * n0 * 2);
      o.b0 = take((size_t)n0 * 4);
      o.w1 = take((size_t)n0 * n1 * 2);
      o.b1 = take((size_t)n1 * 4);
    };
    for (int i = 0; i < m->n_io; ++i) {
      conv(L->init0[i], g.Cf);
      conv(L->init1[i], g.Ch);
      mlp(L->llr[i], g.Cs, 2 * hp, 32);
    }
    mlp(L->msg, g.Cs, hp, np);
    conv(L->upd0, g.Cs + g.Ca);
    conv(L->upd1, g.Ch);
    if (np >= 32) {  // pair copies (same byte size: two ranks of np/2 columns)
      for (int i = 0; i < m->n_io; ++i) conv(L->init0p[i], g.Cf);
      conv(L->upd0p, g.Cs + g.Ca);
    }
    L->total = off;
    return;
  }
  auto conv = [&](ConvOff& c, int ktap, int cdst) {
    int nw = rup(cdst, 8);
    c.ktap = ktap;
    c.w = take((size_t)taps * ktap * nw * 4);
    c.b = take((size_t)nw * 4);
  };
  auto mlp = [&](MlpOff& o, int outp) {
    o.out = outp;
    o.w0 = take((size_t)dmax * m->hidden * 4);
    o.b0 = take((size_t)m->hidden * 4);
    o.w1 = take((size_t)m->hidden * outp * 4);
    o.b1 = take((size_t)outp * 4);
  };
  for (int i = 0; i < m->n_io; ++i) {
    conv(L->init0[i], g.Cf, g.Ch);
    conv(L->init1[i], g.Ch, g.Cs);
    mlp(L->llr[i], 8);
  }
  mlp(L->msg, dmax);
  conv(L->upd0, g.Cs + g.Ca, g.Ch);
  conv(L->upd1, g.Ch, g.Cs);
  mlp(L->chest, 16);
  L->total = off;
}

namespace {

// Map a buffer input channel j of a conv to the reference Cin index (-1: zero).
using ChanMap = int (*)(int j, const Geom& g);
int map_identity_feats(int j, const Geom& g) { return j < g.Cin ? j : -1; }
int map_identity_hidden(int j, const Geom& g) { return j < g.d ? j : -1; }
// update conv0 input = [state (d) | pos (2) | pad][agg (d) | pad]; the
// reference concat order is [state, agg, pos] (nrx.py:262).
int map_update(int j, const Geom& g) {
  if (j < g.d) return j;
  if (j == g.d) return 2 * g.d;
  if (j == g.d + 1) return 2 * g.d + 1;
  if (j < g.Cs) return -1;
  int a = j - g.Cs;
  return a < g.d ? g.d + a : -1;
}
// update conv0 with the positional channels folded out (upd0_posf): [state (d) | agg (d)]
int map_update_posf(int j, const Geom& g) { return j < 2 * g.d ? j : -1; }

// fp32 weights of the two positional input channels (reference Cin 2d, 2d+1)
// as [channel][tap][np] after the bias block (posw_off)
void pack_posw(const Geom& g, int k, const ConvOff& c, int np, const float* w, uint8_t* base) {
  const int taps = k * k, cout = g.d, cin_ref = 2 * g.d + 2;
  float* pw = (float*)(base + c.b) + posw_off(np);
  for (int p = 0; p < 2; ++p)
    for (int tap = 0; tap < taps; ++tap)
      for (int o = 0; o < np; ++o)
        pw[((size_t)p * taps + tap) * np + o] = o < cout ? w[((size_t)tap * cin_ref + 2 * g.d + p) * cout + o] : 0.f;
}

void pack_conv_f32(const Geom& g, int k, const ConvOff& c, int cdst, int cin_ref, const float* w,
                   const float* b, ChanMap map, uint8_t* base) {
  const int nw = rup(cdst, 8), taps = k * k, cout = g.d;
  float* dw = (float*)(base + c.w);
  float* db = (float*)(base + c.b);
  for (int tap = 0; tap < taps; ++tap)
    for (int j = 0; j < c.ktap; ++j) {
      int src = map(j, g);
      for (int o = 0; o < nw; ++o)
        dw[((size_t)tap * c.ktap + j) * nw + o] =
            (src >= 0 && o < cout) ? w[((size_t)tap * cin_ref + src) * cout + o] : 0.f;
    }
  for (int o = 0; o < nw; ++o) db[o] = o < cout ? b[o] : 0.f;
}

void pack_mlp_f32(int din, int dmax, int h, int out, const MlpOff& o, const float* w0, const float* b0,
                  const float* w1, const float* b1, uint8_t* base) {
  float* p0 = (float*)(base + o.w0);
  for (int i = 0; i < dmax; ++i)
    for (int j = 0; j < h; ++j) p0[(size_t)i * h + j] = i < din ? w0[(size_t)i * h + j] : 0.f;
  std::memcpy(base + o.b0, b0, (size_t)h * 4);
  float* p1 = (float*)(base + o.w1);
  float* q1 = (float*)(base + o.b1);
  for (int j = 0; j < h; ++j)
    for (int c = 0; c < o.out; ++c) p1[(size_t)j * o.out + c] = c < out ? w1[(size_t)j * out + c] : 0.f;
  for (int c = 0; c < o.out; ++c) q1[c] = c < out ? b1[c] : 0.f;
}

uint16_t f32_to_bf16(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  if ((x & 0x7f800000u) == 0x7f800000u && (x & 0x007fffffu)) return (uint16_t)((x >> 16) | 0x40);  // quiet NaN
  x += 0x7fffu + ((x >> 16) & 1u);  // round to nearest even
  return (uint16_t)(x >> 16);
}

uint16_t f32_to_f16(float f) {  // IEEE binary16, round to nearest even (GCC _Float16)
  const _Float16 h = (_Float16)f;
  uint16_t bits;
  std::memcpy(&bits, &h, 2);
  return bits;
}

// B operand writer: element (n, k) of a [N][K] K-major matrix, bf16 or fp16.
struct BOperand {
  uint16_t* p;
  int N;
  bool f16;
  void set(int n, int k, float v) {
    p[((size_t)(k / 8) * N + n) * 8 + (k % 8)] = f16 ? f32_to_f16(v) : f32_to_bf16(v);
  }
};

void pack_conv_bf16(const Geom& g, int k, const ConvOff& c, int cin_ref, const float* w, const float* b,
                    ChanMap map, uint8_t* base) {
  const int np = rup(g.d, 16), taps = k * k, cout = g.d;
  BOperand B{(uint16_t*)(base + c.w), np, g.prec == NRX_FP16};
  for (int tap = 0; tap < taps; ++tap)
    for (int j = 0; j < c.ktap; ++j) {
      const int src = map(j, g);
      for (int o = 0; o < np; ++o)
        B.set(o, tap * c.ktap + j, (src >= 0 && o < cout) ? w[((size_t)tap * cin_ref + src) * cout + o] : 0.f);
    }
  float* db = (float*)(base + c.b);
  for (int o = 0; o < np; ++o) db[o] = o < cout ? b[o] : 0.f;
}

// bf16 / fp16 single-CTA convolution in the tap-pair K order (tp2_slot) over C data chunks
void pack_conv_bf16_tp2(const Geom& g, int C, const ConvOff& c, int cin_ref, const float* w, const float* b,
                        uint8_t* base) {
  const int np = rup(g.d, 16), cout = g.d;
  BOperand B{(uint16_t*)(base + c.w), np, g.prec == NRX_FP16};
  for (int slot = 0; slot < 2 * tp2_steps(C); ++slot) {
    int tap, ch;
    tp2_slot(C, slot, &tap, &ch);
    for (int j = 0; j < 8; ++j) {
      const int src = 8 * ch + j;
      for (int o = 0; o < np; ++o)
        B.set(o, 8 * slot + j, (src < cin_ref && o < cout) ? w[((size_t)tap * cin_ref + src) * cout + o] : 0.f);
    }
  }
  float* db = (float*)(base + c.b);
  for (int o = 0; o < np; ++o) db[o] = o < cout ? b[o] : 0.f;
}

float f16_to_f32(uint16_t b) {
  _Float16 h;
  std::memcpy(&h, &b, 2);
  return (float)h;
}

// Power-of-two operand scale 2^E with max|W| 2^E in [2^13, 2^14): the hi
// halves stay far below the fp16 limit and the lo halves (|lo| <= 2^-11 |hi|)
// keep all 11 bits down to weights 2^-16 of the largest.
int split_exponent(float maxabs) {
  if (!(maxabs > 0.f) || !std::isfinite(maxabs)) return 0;
  int e = 0;
  std::frexp(maxabs, &e);  // maxabs < 2^e
  int E = 14 - e;
  return E < -100 ? -100 : E > 100 ? 100 : E;
}

// fp32-grade B operand: W 2^E = hi + lo (both fp16), K-major core-matrix
// layout [K/8][N][8] for each half; `lo_off` elements separate the halves.
struct SplitB {
  uint16_t* p;
  int N;
  size_t lo_off;
  float scale;
  void set(int n, int k, float v) {
    const float s = v * scale;
    const uint16_t h = f32_to_f16(s);
    const size_t i = ((size_t)(k / 8) * N + n) * 8 + (k % 8);
    p[i] = h;
    p[lo_off + i] = f32_to_f16(s - f16_to_f32(h));
  }
};

// Convolution for the CTA pair: the pair MMA (N = 2 npx) reads its B operand
// as rank 0's rows followed by rank 1's, so rank 0 holds W_hi and rank 1 W_lo,
// each for every output channel ([taps*ktap/8][npx][8] fp16): one MMA gives
// [a*W_hi | a*W_lo] in adjacent TMEM column blocks.
void pack_conv_x3(const Geom& g, int k, const ConvOff& c, int cin_ref, const float* w, const float* b,
                  ChanMap map, uint8_t* base) {
  const int npx = x3_np(g.d), taps = k * k, cout = g.d;
  float mx = 0.f;
  for (size_t i = 0; i < (size_t)taps * cin_ref * cout; ++i) mx = std::fmax(mx, std::fabs(w[i]));
  const int E = split_exponent(mx);
  const size_t half = (size_t)taps * c.ktap * npx;  // elements of one rank's block
  SplitB B{(uint16_t*)(base + c.w), npx, half, std::ldexp(1.f, E)};
  for (int tap = 0; tap < taps; ++tap)
    for (int j = 0; j < c.ktap; ++j) {
      const int src = map(j, g);
      for (int o = 0; o < npx; ++o)
        B.set(o, tap * c.ktap + j, (src >= 0 && o < cout) ? w[((size_t)tap * cin_ref + src) * cout + o] : 0.f);
    }
  float* db = (float*)(base + c.b);
  for (int o = 0; o < npx; ++o) db[o] = o < cout ? b[o] : 0.f;
  db[npx] = std::ldexp(1.f, -E);
}

// The same in the tap-pair K order (tp2_slot) for an input of C data chunks
// (cin_ref reference channels); the block keeps the taps x ktap size, the
// unused slots at its end stay zero.
void pack_conv_x3_tp2(const Geom& g, int C, const ConvOff& c, int cin_ref, const float* w, const float* b,
                      uint8_t* base) {
  const int npx = x3_np(g.d), taps = 9, cout = g.d;
  float mx = 0.f;
  for (size_t i = 0; i < (size_t)taps * cin_ref * cout; ++i) mx = std::fmax(mx, std::fabs(w[i]));
  const int E = split_exponent(mx);
  const size_t half = (size_t)taps * c.ktap * npx;
  SplitB B{(uint16_t*)(base + c.w), npx, half, std::ldexp(1.f, E)};
  for (int slot = 0; slot < 2 * tp2_steps(C); ++slot) {
    int tap, ch;
    tp2_slot(C, slot, &tap, &ch);
    for (int j = 0; j < 8; ++j) {
      const int src = 8 * ch + j;
      for (int o = 0; o < npx; ++o)
        B.set(o, 8 * slot + j, (src < cin_ref && o < cout) ? w[((size_t)tap * cin_ref + src) * cout + o] : 0.f);
    }
  }
  float* db = (float*)(base + c.b);
  for (int o = 0; o < npx; ++o) db[o] = o < cout ? b[o] : 0.f;
  db[npx] = std::ldexp(1.f, -E);
}

// Half-precision convolution for the CTA pair: rank r holds output channels
// [r np/2, (r+1) np/2) as [K/8][np/2][8] (the pair MMA reads B as rank 0's
// rows followed by rank 1's).
void pack_conv_pair16(const Geom& g, int k, const ConvOff& c, int cin_ref, const float* w, const float* b,
                      ChanMap map, uint8_t* base) {
  const int np = rup(g.d, 16), nh = np / 2, taps = k * k, cout = g.d;
  const size_t block = (size_t)taps * c.ktap * nh;
  for (int r = 0; r < 2; ++r) {
    BOperand B{(uint16_t*)(base + c.w) + (size_t)r * block, nh, g.prec == NRX_FP16};
    for (int tap = 0; tap < taps; ++tap)
      for (int j = 0; j < c.ktap; ++j) {
        const int src = map(j, g);
        for (int n = 0; n < nh; ++n) {
          const int o = r * nh + n;
          B.set(n, tap * c.ktap + j, (src >= 0 && o < cout) ? w[((size_t)tap * cin_ref + src) * cout + o] : 0.f);
        }
      }
  }
  float* db = (float*)(base + c.b);
  for (int o = 0; o < np; ++o) db[o] = o < cout ? b[o] : 0.f;
}

}  // namespace

// fp32-grade tensor-core packing (NRX_FP32X3): same GEMM shapes as
// pack_weights_tc, every B operand as scaled fp16 [hi | lo] halves and the
// descale 2^-E stored after each bias vector.
int pack_weights_x3(const nrx_model_desc* m, const float* const* t, uint8_t* base) {
  PackLayout L;
  pack_layout(m, NRX_FP32X3, &L);
  std::memset(base, 0, L.total);
  Geom g;
  nrx_slot_desc s{};
  s.num_subcarriers = 64; s.num_symbols = 14; s.num_ues = 1; s.comb_size = 1;
  s.num_pilot_symbols = 1;
  make_geom(m, &s, 1, NRX_FP32X3, &g);
  const int k = m->kernel_size, d = m->d_s, h = m->hidden, B2 = 2 * m->num_rx_ant;
  const int np = rup(d, 16), hp = rup(h, 16);
  const int i_msg = 8 * m->n_io, i_upd = i_msg + 4, i_chest = i_upd + 4;
  auto maxabs = [](const float* a, size_t n) {
    float mx = 0.f;
    for (size_t i = 0; i < n; ++i) mx = std::fmax(mx, std::fabs(a[i]));
    return mx;
  };
  for (int io = 0; io < m->n_io; ++io) {
    const int i = 8 * io;
    if (tp2_chunks(d, k, NRX_FP32X3, g.Cf, g.Cin) == 3)  // the 19 feature channels: 3 data chunks of 4
      pack_conv_x3_tp2(g, 3, L.init0[io], g.Cin, t[i], t[i + 1], base);
    else
      pack_conv_x3(g, k, L.init0[io], g.Cin, t[i], t[i + 1], map_identity_feats, base);
    if (tp2_layer(d, k, NRX_FP32X3))
      pack_conv_x3_tp2(g, 7, L.init1[io], d, t[i + 2], t[i + 3], base);
    else
      pack_conv_x3(g, k, L.init1[io], d, t[i + 2], t[i + 3], map_identity_hidden, base);
    const MlpOff& o = L.llr[io];
    const int width = llr_width_of(m, io);
    const float *lw0 = t[i + 4], *lb0 = t[i + 5], *lw1 = t[i + 6], *lb1 = t[i + 7];
    const float *cw0 = t[i_chest], *cb0 = t[i_chest + 1], *cw1 = t[i_chest + 2], *cb1 = t[i_chest + 3];
    const int E0 = split_exponent(std::fmax(maxabs(lw0, (size_t)d * h), maxabs(cw0, (size_t)d * h)));
    SplitB W0{(uint16_t*)(base + o.w0), 2 * hp, (size_t)g.Cs * 2 * hp, std::ldexp(1.f, E0)};
    float* b0 = (float*)(base + o.b0);
    for (int n = 0; n < 2 * hp; ++n) {
      const bool chest = n >= hp;
      const int nn = chest ? n - hp : n;
      for (int kk = 0; kk < g.Cs; ++kk)
        W0.set(n, kk, (kk < d && nn < h) ? (chest ? cw0 : lw0)[(size_t)kk * h + nn] : 0.f);
      b0[n] = nn < h ? (chest ? cb0 : lb0)[nn] : 0.f;
    }
    b0[2 * hp] = std::ldexp(1.f, -E0);
    const int E1 = split_exponent(std::fmax(maxabs(lw1, (size_t)h * width), maxabs(cw1, (size_t)h * B2)));
    SplitB W1{(uint16_t*)(base + o.w1), 32, (size_t)2 * hp * 32, std::ldexp(1.f, E1)};
    float* b1 = (float*)(base + o.b1);
    for (int n = 0; n < 32; ++n) {
      for (int kk = 0; kk < 2 * hp; ++kk) {
        float v = 0.f;
        if (n < width && kk < h) v = lw1[(size_t)kk * width + n];
        if (n >= 8 && n < 8 + B2 && kk >= hp && kk - hp < h) v = cw1[(size_t)(kk - hp) * B2 + (n - 8)];
        W1.set(n, kk, v);
      }
      b1[n] = n < width ? lb1[n] : (n >= 8 && n < 8 + B2) ? cb1[n - 8] : 0.f;
    }
    b1[32] = std::ldexp(1.f, -E1);
  }
  {
    const float *w0 = t[i_msg], *b0 = t[i_msg + 1], *w1 = t[i_msg + 2], *b1 = t[i_msg + 3];
    const int E0 = split_exponent(maxabs(w0, (size_t)d * h)), E1 = split_exponent(maxabs(w1, (size_t)h * d));
    SplitB W0{(uint16_t*)(base + L.msg.w0), hp, (size_t)g.Cs * hp, std::ldexp(1.f, E0)};
    float* pb0 = (float*)(base + L.msg.b0);
    for (int n = 0; n < hp; ++n) {
      for (int kk = 0; kk < g.Cs; ++kk) W0.set(n, kk, (kk < d && n < h) ? w0[(size_t)kk * h + n] : 0.f);
      pb0[n] = n < h ? b0[n] : 0.f;
    }
    pb0[hp] = std::ldexp(1.f, -E0);
    SplitB W1{(uint16_t*)(base + L.msg.w1), np, (size_t)hp * np, std::ldexp(1.f, E1)};
    float* pb1 = (float*)(base + L.msg.b1);
    for (int n = 0; n < np; ++n) {
      for (int kk = 0; kk < hp; ++kk) W1.set(n, kk, (kk < h && n < d) ? w1[(size_t)kk * d + n] : 0.f);
      pb1[n] = n < d ? b1[n] : 0.f;
    }
    pb1[np] = std::ldexp(1.f, -E1);
  }
  if (upd0_posf(d, k, NRX_FP32X3)) {
    pack_conv_x3(g, k, L.upd0, 2 * d + 2, t[i_upd], t[i_upd + 1], map_update_posf, base);
    pack_posw(g, k, L.upd0, x3_np(d), t[i_upd], base);
  } else {
    pack_conv_x3(g, k, L.upd0, 2 * d + 2, t[i_upd], t[i_upd + 1], map_update, base);
  }
  if (tp2_layer(d, k, NRX_FP32X3))
    pack_conv_x3_tp2(g, 7, L.upd1, d, t[i_upd + 2], t[i_upd + 3], base);
  else
    pack_conv_x3(g, k, L.upd1, d, t[i_upd + 2], t[i_upd + 3], map_identity_hidden, base);
  return NRX_OK;
}

int pack_weights_tc(const nrx_model_desc* m, int prec, const float* const* t, uint8_t* base) {
  PackLayout L;
  pack_layout(m, prec, &L);
  std::memset(base, 0, L.total);
  Geom g;
  nrx_slot_desc s{};
  s.num_subcarriers = 64; s.num_symbols = 14; s.num_ues = 1; s.comb_size = 1;
  s.num_pilot_symbols = 1;
  make_geom(m, &s, 1, prec, &g);
  const bool f16 = prec == NRX_FP16;
  const int k = m->kernel_size, d = m->d_s, h = m->hidden, B2 = 2 * m->num_rx_ant;
  const int np = rup(d, 16), hp = rup(h, 16);
  // indices of the shared tensors in the canonical order (include/nrx_b200.h)
  const int i_msg = 8 * m->n_io, i_upd = i_msg + 4, i_chest = i_upd + 4;
  for (int io = 0; io < m->n_io; ++io) {
    const int i = 8 * io;
    if (tp2_chunks(d, k, prec, g.Cf, g.Cin) == 3)
      pack_conv_bf16_tp2(g, 3, L.init0[io], g.Cin, t[i], t[i + 1], base);
    else
      pack_conv_bf16(g, k, L.init0[io], g.Cin, t[i], t[i + 1], map_identity_feats, base);
    if (tp2_layer(d, k, prec))
      pack_conv_bf16_tp2(g, 7, L.init1[io], d, t[i + 2], t[i + 3], base);
    else
      pack_conv_bf16(g, k, L.init1[io], d, t[i + 2], t[i + 3], map_identity_hidden, base);
    // fused readout: fc0 = [llr fc0 | chest fc0], fc1 block diagonal
    const MlpOff& o = L.llr[io];
    const int width = llr_width_of(m, io);
    const float *lw0 = t[i + 4], *lb0 = t[i + 5], *lw1 = t[i + 6], *lb1 = t[i + 7];
    const float *cw0 = t[i_chest], *cb0 = t[i_chest + 1], *cw1 = t[i_chest + 2], *cb1 = t[i_chest + 3];
    BOperand W0{(uint16_t*)(base + o.w0), 2 * hp, f16};
    float* b0 = (float*)(base + o.b0);
    for (int n = 0; n < 2 * hp; ++n) {
      const bool chest = n >= hp;
      const int nn = chest ? n - hp : n;
      for (int kk = 0; kk < g.Cs; ++kk)
        W0.set(n, kk, (kk < d && nn < h) ? (chest ? cw0 : lw0)[(size_t)kk * h + nn] : 0.f);
      b0[n] = nn < h ? (chest ? cb0 : lb0)[nn] : 0.f;
    }
    BOperand W1{(uint16_t*)(base + o.w1), 32, f16};
    float* b1 = (float*)(base + o.b1);
    for (int n = 0; n < 32; ++n) {
      for (int kk = 0; kk < 2 * hp; ++kk) {
        float v = 0.f;
        if (n < width && kk < h) v = lw1[(size_t)kk * width + n];
        if (n >= 8 && n < 8 + B2 && kk >= hp && kk - hp < h) v = cw1[(size_t)(kk - hp) * B2 + (n - 8)];
        W1.set(n, kk, v);
      }
      b1[n] = n < width ? lb1[n] : (n >= 8 && n < 8 + B2) ? cb1[n - 8] : 0.f;
    }
  }
  {
    const float *w0 = t[i_msg], *b0 = t[i_msg + 1], *w1 = t[i_msg + 2], *b1 = t[i_msg + 3];
    BOperand W0{(uint16_t*)(base + L.msg.w0), hp, f16};
    float* pb0 = (float*)(base + L.msg.b0);
    for (int n = 0; n < hp; ++n) {
      for (int kk = 0; kk < g.Cs; ++kk) W0.set(n, kk, (kk < d && n < h) ? w0[(size_t)kk * h + n] : 0.f);
      pb0[n] = n < h ? b0[n] : 0.f;
    }
    BOperand W1{(uint16_t*)(base + L.msg.w1), np, f16};
    float* pb1 = (float*)(base + L.msg.b1);
    for (int n = 0; n < np; ++n) {
      for (int kk = 0; kk < hp; ++kk) W1.set(n, kk, (kk < h && n < d) ? w1[(size_t)kk * d + n] : 0.f);
      pb1[n] = n < d ? b1[n] : 0.f;
    }
  }
  pack_conv_bf16(g, k, L.upd0, 2 * d + 2, t[i_upd], t[i_upd + 1], map_update, base);
  if (tp2_layer(d, k, prec))
    pack_conv_bf16_tp2(g, 7, L.upd1, d, t[i_upd + 2], t[i_upd + 3], base);
  else
    pack_conv_bf16(g, k, L.upd1, d, t[i_upd + 2], t[i_upd + 3], map_identity_hidden, base);
  if (L.upd0p.w) {
    for (int io = 0; io < m->n_io; ++io)
      pack_conv_pair16(g, k, L.init0p[io], g.Cin, t[8 * io], t[8 * io + 1], map_identity_feats, base);
    pack_conv_pair16(g, k, L.upd0p, 2 * d + 2, t[i_upd], t[i_upd + 1], map_update, base);
  }
  return NRX_OK;
}

int pack_weights_f32(const nrx_model_desc* m, const float* const* t, uint8_t* base) {
  PackLayout L;
  pack_layout(m, NRX_FP32, &L);
  std::memset(base, 0, L.total);
  Geom g;
  nrx_slot_desc s{};
  s.num_subcarriers = 64; s.num_symbols = 14; s.num_ues = 1; s.comb_size = 1;
  s.num_pilot_symbols = 1;
  make_geom(m, &s, 1, NRX_FP32, &g);
  const int k = m->kernel_size, d = m->d_s, h = m->hidden;
  int i = 0;
  for (int io = 0; io < m->n_io; ++io) {
    pack_conv_f32(g, k, L.init0[io], g.Ch, g.Cin, t[i], t[i + 1], map_identity_feats, base);
    pack_conv_f32(g, k, L.init1[io], g.Cs, d, t[i + 2], t[i + 3], map_identity_hidden, base);
    pack_mlp_f32(d, L.dmax, h, llr_width_of(m, io), L.llr[io], t[i + 4], t[i + 5], t[i + 6], t[i + 7], base);
    i += 8;
  }
  pack_mlp_f32(d, L.dmax, h, d, L.msg, t[i], t[i + 1], t[i + 2], t[i + 3], base);
  i += 4;
  pack_conv_f32(g, k, L.upd0, g.Ch, 2 * d + 2, t[i], t[i + 1], map_update, base);
  pack_conv_f32(g, k, L.upd1, g.Cs, d, t[i + 2], t[i + 3], map_identity_hidden, base);
  i += 4;
  pack_mlp_f32(d, L.dmax, h, 2 * m->num_rx_ant, L.chest, t[i], t[i + 1], t[i + 2], t[i + 3], base);
  return NRX_OK;
}

void ws_layout(const Geom& g, WsLayout* w) {
  const size_t esz = g.prec == NRX_FP32 ? 4 : 2;
  // fp32x3: every activation buffer holds its hi and lo planes (2x channels)
  const size_t plane = (size_t)g.NU * g.rows_slab * esz * (g.prec == NRX_FP32X3 ? 2 : 1);
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
  w->flag = take(4);  // offset 0 (NRX_WS_FLAG_OFFSET)
  w->feats = take(plane * g.Cf);
  w->h = take(plane * g.Ch);
  w->state = take(plane * g.Cs);
  w->agg = take(plane * g.Ca);
  w->state32 = g.prec == NRX_BF16 ? take((size_t)g.NU * g.rows_slab * 4 * rup(g.d, 4)) : 0;
  w->total = off;
}

}  // namespace nrx

using namespace nrx;

extern "C" {

int nrx_abi_version(void) { return NRX_ABI_VERSION; }

const char* nrx_status_string(int s) {
  switch (s) {
    case NRX_OK: return "ok";
    case NRX_ERR_INVALID: return "invalid descriptor or argument";
    case NRX_ERR_UNSUPPORTED: return "configuration outside the limits of this implementation";
    case NRX_ERR_WORKSPACE: return "workspace too small";
    case NRX_ERR_CUDA: return "CUDA launch or driver error";
    case NRX_ERR_DEPTH: return "inference depth outside [1, N_it]";
    case NRX_ERR_NO_DEVICE: return "no sm_100 device or kernel image";
    default: return "unknown status";
  }
}

int nrx_validate(const nrx_model_desc* m, const nrx_slot_desc* s) { return validate(m, s); }

int nrx_weight_count(const nrx_model_desc* m) {
  if (validate(m, nullptr) == NRX_ERR_INVALID) return -1;
  return (int)canonical(m).size();
}

int nrx_weight_name(const nrx_model_desc* m, int i, char* buf, size_t len) {
  if (validate(m, nullptr) == NRX_ERR_INVALID) return -1;
  auto v = canonical(m);
  if (i < 0 || i >= (int)v.size() || !buf || len == 0) return -1;
  std::snprintf(buf, len, "%s", v[i].name.c_str());
  return (int)v[i].name.size();
}

int64_t nrx_weight_numel(const nrx_model_desc* m, int i) {
  if (validate(m, nullptr) == NRX_ERR_INVALID) return -1;
  auto v = canonical(m);
  if (i < 0 || i >= (int)v.size()) return -1;
  return numel(v[i]);
}

size_t nrx_packed_weight_bytes(const nrx_model_desc* m, int prec) {
  if (validate(m, nullptr) != NRX_OK) return 0;
  PackLayout L;
  pack_layout(m, prec, &L);
  return L.total;
}

int nrx_pack_weights(const nrx_model_desc* m, int prec, const float* const* tensors, int n, void* out) {
  int st = validate(m, nullptr);
  if (st) return st;
  if (!tensors || !out || n != (int)canonical(m).size()) return NRX_ERR_INVALID;
  for (int i = 0; i < n; ++i)
    if (!tensors[i]) return NRX_ERR_INVALID;
  if (prec == NRX_FP32) return pack_weights_f32(m, tensors, (uint8_t*)out);
  if (hidden_limit(prec) < rup(m->hidden, 16)) return NRX_ERR_UNSUPPORTED;
  if (prec == NRX_FP32X3) return pack_weights_x3(m, tensors, (uint8_t*)out);
  if (prec == NRX_BF16 || prec == NRX_FP16) return pack_weights_tc(m, prec, tensors, (uint8_t*)out);
  return NRX_ERR_INVALID;
}

size_t nrx_workspace_bytes(const nrx_model_desc* m, const nrx_slot_desc* s, int n_slots, int prec) {
  Geom g;
  if (make_geom(m, s, n_slots, prec, &g)) return 0;
  WsLayout w;
  ws_layout(g, &w);
  return w.total;
}

}  // extern "C"
