// Internal geometry / layout definitions shared by the host orchestrator,
// the weight packer and the kernels.
//
// HBM layout of every activation tensor ("chunk-planar", slab-major):
//   buf[slab][chunk][row][CW]      CW = 16 bytes / sizeof(element)
// slab = n*U + u (the reference's N*U flattening, nrx.py:321), chunk =
// channel / CW, row = s*Tp + t over the (S, T) grid with the symbol axis
// padded from T to Tp = T + r (r = kernel_size/2).  With that padding the
// k x k 'same' convolution over (s, t) (autodiff.py:324-350) becomes a 1-D
// convolution over `row` with tap offsets (a-r)*Tp + (b-r): the zero rows
// t in [T, Tp) supply the reference's zero padding along T and rows outside
// [0, rows_slab) (zero-filled by TMA / bounds checks) the padding along S.
// rows_slab = S*Tp rounded up to the 128-row tile; rows with s >= S or
// t >= T are kept at zero by every producer.  A 16-byte chunk of one row
// is the unit every kernel moves, so a warp touching 32 consecutive rows of
// one chunk issues fully coalesced 512-byte transactions, and a TMA box
// {CW, rows, chunks} lands as the K-major no-swizzle core-matrix layout
// tcgen05.mma reads directly.
#pragma once
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/nrx_b200.h"

#define NRX_TILE_M 128

namespace nrx {

inline int cdiv(int a, int b) { return (a + b - 1) / b; }
inline int rup(int a, int b) { return cdiv(a, b) * b; }
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
// fp32x3 pair-convolution width: output channels of one [W_hi | W_lo] half
// (the pair MMA's N is twice it, a multiple of 16): d rounded up to 16, but
// 56 for d in (48, 56] (the RT model: N = 112 instead of 128 skips 12.5 % of
// the tensor work).
inline int x3_np(int d) { return (d + 7) / 8 * 8 == 56 ? 56 : rup(d, 16); }
// iteration.update.conv0 with the two positional channels taken out of the
// GEMM (K = 2 d instead of rup(d + 2, 16) + rup(d, 16): 112 instead of 128
// for d = 56, 32 instead of 48 for d = 16); the epilogue adds their
// contribution from 18 x np fp32 weights stored after the bias (POSW_OFF).
// On for the fp32x3 layer where an unrolled instance exists (d = 16, 56):
// update.conv0 0.975 -> 0.887 ms per 32 C2 slots.  The bf16 / fp16 pair copy
// keeps K = 128: there the shared 2-source stage and the table lookups cost
// more than the 12.5 % of MMAs they save (0.341 -> 0.357 ms).
inline bool posf_enabled() {  // NRX_POSF=0: keep the positional channels in K (A/B experiments)
  static const bool on = [] {
    const char* e = std::getenv("NRX_POSF");
    return !(e && e[0] == '0');
  }();
  return on;
}
inline bool upd0_posf(int d, int ks, int prec) {
  if (ks != 3 || d % 8 || !posf_enabled()) return false;
  return prec == NRX_FP32X3 && (d == 56 || d == 16);
}
// float offset of the positional weights [channel dt, df][tap][np] in a conv bias block
inline int posw_off(int np) { return np + 4; }

// fp32x3 3x3 convolutions whose input has an odd number C of 8-channel chunks
// holding data (C = 7: state_init.conv1 / update.conv1 of d_s = 56; C = 3: the
// 19 feature channels of state_init.conv0): a per-tap K = 16 loop reads a zero
// chunk per tap.  "Tap pairs" order the K slots (8 channels each) so that one
// MMA step straddles two taps: taps (t, u = t+1) take C steps instead of C+1 --
// (t,0)(t,1) .. (t,C-3)(t,C-2), then (u,0)(t,C-1), then (u,1)(u,2) .. (u,C-2)(u,C-1)
// -- for the pairs (0,1) (2,3) (4,5) (6,7), then tap 8 alone in (C+1)/2 steps
// whose last pairs a zero-weight slot (A: chunk C-2, which the TMA loads) with
// chunk C-1.  The straddling step's second half sits at another row offset,
// which its A descriptor's leading-byte offset expresses; only C chunks are loaded.
inline int tp2_chunks(int d, int ks, int prec, int cin_buf, int cin) {  // C, or 0: not a tap-pair layer
  if ((prec != NRX_FP32X3 && prec != NRX_FP16 && prec != NRX_BF16) || ks != 3 || cin_buf % 16) return 0;
  const int c = (cin + 7) / 8;
  return (c % 2 == 1 && c + 1 == cin_buf / 8 && (c == 7 || c == 3) && d == 56) ? c : 0;
}
inline bool tp2_layer(int d, int ks, int prec) { return tp2_chunks(d, ks, prec, rup(d, 16), d) == 7; }
inline int tp2_steps(int C) { return 4 * C + (C + 1) / 2; }
inline void tp2_slot(int C, int slot, int* tap, int* chunk) {  // half-slot (8 K values) -> (tap, chunk)
  const int step = slot / 2, h = slot & 1;
  if (step >= 4 * C) {  // tap 8 alone; the last step: zero-weight slot (chunk C, none) then chunk C-1
    const int s = step - 4 * C;
    *tap = 8;
    *chunk = s == (C - 1) / 2 ? (h ? C - 1 : C) : 2 * s + h;
    return;
  }
  const int pr = step / C, s = step % C, t = 2 * pr, half = (C - 1) / 2;
  if (s < half) {
    *tap = t;
    *chunk = 2 * s + h;
  } else if (s == half) {
    *tap = h ? t : t + 1;
    *chunk = h ? C - 1 : 0;
  } else {
    *tap = t + 1;
    *chunk = 2 * (s - half) - 1 + h;
  }
}
// Geometry + channel bookkeeping, passed by value to kernels.
struct Geom {
  int N, U, NU, S, T, B, comb, K;
  uint32_t comb_magic;        // ceil(2^32 / comb): (s - o) / comb by one __umulhi (comb > 1)
  float df_tab[16];           // float32(k / S) for k < comb <= 16 (the frequency encoding)
  int ps[NRX_MAX_PILOT_SYMBOLS];
  int ks, r, Tp, H;           // kernel size, radius, padded symbols, halo rows
  float inv_Tp;               // 1 / Tp: row -> (s, t) by one multiply (rows < 2^21)
  int rows_data, rows_slab, tiles;
  int d, h;                   // state depth, MLP hidden width
  int cw;                     // elements per 16-byte chunk
  int Cin, Cf, Cs, Ch, Ca;    // logical input channels, buffer channel counts
  int nb;                     // conv output width covered by the SIMT kernel
  int n_io;
  int io_orders[NRX_MAX_IO];
  int io_width[NRX_MAX_IO];   // LLR width produced by io set i
  int llr_width;              // output row stride of llr_out
  int noise_plane, freq_enc;
  int prec;
  float dt[32];               // positional encoding, symbol axis (float32, nrx.py:164)
  int nearest[32];            // nearest pilot-symbol index per t (classical.py:71)
  uint32_t* flag;             // workspace word set when a tensor-core readout wrote a non-finite output
};

// Byte offsets of each weight sub-buffer inside the packed blob.
struct ConvOff { size_t w, b; int ktap; };
struct MlpOff { size_t w0, b0, w1, b1; int out; };
struct PackLayout {
  ConvOff init0[NRX_MAX_IO], init1[NRX_MAX_IO];
  MlpOff llr[NRX_MAX_IO];
  MlpOff msg;
  ConvOff upd0, upd1;
  // bf16 / fp16: CTA-pair copies of the tail-less ReLU convolutions (rank r's
  // block holds output channels [r np/2, (r+1) np/2)); w == 0 when absent
  ConvOff init0p[NRX_MAX_IO], upd0p;
  MlpOff chest;
  size_t total;
  int dmax;                   // padded state depth for the SIMT MLP kernels
};

struct WsLayout {
  size_t flag, feats, h, state, agg, state32, total;  // flag: uint32 at workspace offset 0
};

}  // namespace nrx
