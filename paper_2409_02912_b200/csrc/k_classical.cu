// k_classical.cu — the reference's "ls_lmmse" baseline receiver on the GPU:
// comb LS channel estimate, per-RE LMMSE equalisation with unbiased outputs,
// exact APP demapping, clipping.  C ABI in include/nrx_classical.h.
//
// Reference (/root/reference/pkg/src/nrxsim): ls_estimate classical.py:40-78,
// lmmse_equalize :113-143, app_demap (mode "exact") :150-174,
// ReceiverBank.run("ls_lmmse") evaluation.py:130-135 with
// _demap_equalized :79-84.  float64 like the reference (the LS keeps its
// operation order; the U x U solves use Gauss-Jordan with partial pivoting
// where LAPACK uses LU, so LLRs agree to float64 rounding, not bitwise).
//
// One thread per RE (slot, s, t): the LS estimates of all UEs at that RE
// (the comb pilots bracketing s at the nearest pilot symbol), the U x U
// Gram matrix H^H H + n0 I and its inverse, the unbiased symbol estimates
// z_u and noise variances, then for each UE the log-sum-exp of
// -|z - x|^2 / nvar over the 2^m Gray points per bit, written as float32.
// Compute-bound (float64 exp/log over the constellation); HBM traffic is
// y in (32 B) and LLRs out (U * W * 4 B) per RE.

#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "../../include/nrx_classical.h"
#include "../../include/nrx_slotgen.h"

namespace nrx_cl {

constexpr double kVarFloor = 1e-12;   // classical.py:25

struct ClParams {
  int S, T, U, B, comb, K, F, n_pilot_sets, W;
  int ps[NRX_MAX_PILOT_SYMBOLS];
  int nearest[32];
  float clip;
  double2 qam[NRX_SG_QAM_POINTS];
  const void* y;
  int y_c128;
  const void* pilots;
  int p_c128;
  const double* n0;
  const int32_t* mod;
  float* llr;
};

__host__ __device__ inline int qam_offset(int m) { return m == 2 ? 0 : m == 4 ? 4 : m == 6 ? 20 : 84; }

__device__ inline double2 ldc(const void* base, size_t i, int c128) {
  if (c128) return static_cast<const double2*>(base)[i];
  const float2 v = static_cast<const float2*>(base)[i];
  return make_double2(v.x, v.y);
}

__device__ inline double2 cmul(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ inline double2 cconjmul(double2 a, double2 b) {   // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ inline double2 cdiv(double2 a, double2 b) {
  const double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}

// conj(p)/|p|^2 as numpy evaluates it (classical.py:46)
__device__ inline double2 pilot_scale(double2 p) {
  const double a = hypot(p.x, p.y);
  const double rec = __ddiv_rn(1.0, __dmul_rn(a, a));
  return make_double2(__dmul_rn(p.x, rec), __dmul_rn(-p.y, rec));
}

__global__ void __launch_bounds__(128) k_ls_lmmse(ClParams p) {
  const int n = blockIdx.y;
  const int re = blockIdx.x * blockDim.x + threadIdx.x;
  if (re >= p.S * p.T) return;
  const int s = re / p.T, t = re - s * p.T;
  const int B = p.B, U = p.U;
  double2 yv[NRX_CL_MAX_RX_ANT];
  for (int b = 0; b < B; ++b) yv[b] = ldc(p.y, (((size_t)n * p.S + s) * p.T + t) * B + b, p.y_c128);

  // ---- LS estimate of every UE at (s, t)
  double2 h[NRX_CL_MAX_UES][NRX_CL_MAX_RX_ANT];
  const int k = p.nearest[t];
  const int pt = p.ps[k];
  const int pset = p.n_pilot_sets > 1 ? n : 0;
  for (int u = 0; u < U; ++u) {
    const int o = u % p.comb;
    const int F = (p.S - o + p.comb - 1) / p.comb;
    int j = 0;
    double frac = 0.0;
    if (F > 1) {
      const int diff = s - o;
      const int q = diff >= 0 ? diff / p.comb : -1;   // python floor division
      j = q < 0 ? 0 : (q > F - 2 ? F - 2 : q);
      frac = __ddiv_rn((double)(s - (o + j * p.comb)), (double)p.comb);
    }
    const size_t pbase = (((size_t)pset * U + u) * p.F) * p.K;
    const double2 q0 = pilot_scale(ldc(p.pilots, pbase + (size_t)j * p.K + k, p.p_c128));
    const double2 q1 = F > 1 ? pilot_scale(ldc(p.pilots, pbase + (size_t)(j + 1) * p.K + k, p.p_c128)) : q0;
    const size_t y0 = (((size_t)n * p.S + (o + j * p.comb)) * p.T + pt) * B;
    const size_t y1 = (((size_t)n * p.S + (o + (j + 1) * p.comb)) * p.T + pt) * B;
    for (int b = 0; b < B; ++b) {
      const double2 r0 = cmul(ldc(p.y, y0 + b, p.y_c128), q0);
      double2 hv = r0;
      if (F > 1) {
        const double2 r1 = cmul(ldc(p.y, y1 + b, p.y_c128), q1);
        hv.x = __dadd_rn(r0.x, __dmul_rn(frac, __dsub_rn(r1.x, r0.x)));
        hv.y = __dadd_rn(r0.y, __dmul_rn(frac, __dsub_rn(r1.y, r0.y)));
      }
      h[u][b] = hv;
    }
  }

  // ---- LMMSE: A = H^H H + max(n0,0) I, x = A^-1 H^H y, mu_u = 1 - n0 [A^-1]_uu
  const double n0 = p.n0[n];
  double2 a[NRX_CL_MAX_UES][2 * NRX_CL_MAX_UES];   // [A | I] -> [I | A^-1]
  double2 rhs[NRX_CL_MAX_UES];
  for (int u = 0; u < U; ++u) {
    for (int v = 0; v < U; ++v) {
      double2 acc = make_double2(0.0, 0.0);
      for (int b = 0; b < B; ++b) {
        const double2 pr = cconjmul(h[u][b], h[v][b]);
        acc.x += pr.x;
        acc.y += pr.y;
      }
      if (u == v) acc.x += fmax(n0, 0.0);
      a[u][v] = acc;
      a[u][U + v] = make_double2(u == v ? 1.0 : 0.0, 0.0);
    }
    double2 r = make_double2(0.0, 0.0);
    for (int b = 0; b < B; ++b) {
      const double2 pr = cconjmul(h[u][b], yv[b]);
      r.x += pr.x;
      r.y += pr.y;
    }
    rhs[u] = r;
  }
  for (int c = 0; c < U; ++c) {   // Gauss-Jordan, partial pivoting
    int piv = c;
    double best = hypot(a[c][c].x, a[c][c].y);
    for (int r = c + 1; r < U; ++r) {
      const double v = hypot(a[r][c].x, a[r][c].y);
      if (v > best) {
        best = v;
        piv = r;
      }
    }
    if (piv != c)
      for (int q = 0; q < 2 * U; ++q) {
        const double2 tmp = a[c][q];
        a[c][q] = a[piv][q];
        a[piv][q] = tmp;
      }
    if (best == 0.0) a[c][c].x = kVarFloor;   // singular: the reference's +1e-12 I retry
    const double2 inv = cdiv(make_double2(1.0, 0.0), a[c][c]);
    for (int q = 0; q < 2 * U; ++q) a[c][q] = cmul(a[c][q], inv);
    for (int r = 0; r < U; ++r) {
      if (r == c) continue;
      const double2 f = a[r][c];
      for (int q = 0; q < 2 * U; ++q) {
        const double2 pr = cmul(f, a[c][q]);
        a[r][q].x -= pr.x;
        a[r][q].y -= pr.y;
      }
    }
  }
  for (int u = 0; u < U; ++u) {
    double2 x = make_double2(0.0, 0.0);
    for (int v = 0; v < U; ++v) {
      const double2 pr = cmul(a[u][U + v], rhs[v]);
      x.x += pr.x;
      x.y += pr.y;
    }
    double mu = 1.0 - n0 * a[u][U + u].x;
    mu = fmax(mu, kVarFloor);
    const double2 z = make_double2(x.x / mu, x.y / mu);
    const double nvar = fmax((1.0 - mu) / mu, kVarFloor);

    // ---- exact APP demap over the UE's Gray constellation
    const int m = p.mod[n * U + u];
    const double2* pts = p.qam + qam_offset(m);
    const int cnt = 1 << m;
    float* out = p.llr + ((((size_t)n * U + u) * p.S + s) * p.T + t) * p.W;
    // log-sum-exp per bit subset with one shared shift (the largest metric):
    // log(sum_1 e^met) - log(sum_0 e^met) is the reference's per-subset
    // max-shifted form up to float64 rounding; a subset that underflows gives
    // +-inf, clipped like the reference's huge finite value.
    double top = -INFINITY;
    for (int i = 0; i < cnt; ++i) {
      const double d = hypot(z.x - pts[i].x, z.y - pts[i].y);
      top = fmax(top, -(d * d) / nvar);
    }
    double s1[8] = {0, 0, 0, 0, 0, 0, 0, 0}, s0[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < cnt; ++i) {
      const double d = hypot(z.x - pts[i].x, z.y - pts[i].y);
      const double e = exp(-(d * d) / nvar - top);
#pragma unroll
      for (int kb = 0; kb < 8; ++kb) {
        if (kb >= m) break;
        if ((i >> (m - 1 - kb)) & 1) s1[kb] += e;
        else s0[kb] += e;
      }
    }
#pragma unroll
    for (int kb = 0; kb < 8; ++kb) {
      if (kb >= m) break;
      const double llr = log(s1[kb]) - log(s0[kb]);
      out[kb] = fminf(fmaxf(static_cast<float>(llr), -p.clip), p.clip);
    }
    for (int kb = m; kb < p.W; ++kb) out[kb] = 0.f;
  }
}

struct KbParams {
  int S, T, U, B, W, K, ref_pairing;
  int is_pilot[32];
  float clip;
  double2 qam[NRX_SG_QAM_POINTS];
  const void* y;
  int y_c128;
  const void* h;
  int h_c128;
  const double* n0;
  const int32_t* mod;
  float* llr;
};

// One thread per RE: MGS QR of the B x U channel, breadth-first K-Best over
// the streams U-1 .. 0 (the reference's level order), max-log LLRs from the
// final list.  Partial-path metrics are invariant to the per-column phase
// of the QR, so MGS (positive real diagonal) and LAPACK's Householder QR
// give the same metrics up to float64 rounding.
__global__ void __launch_bounds__(128) k_kbest(KbParams p) {
  const int n = blockIdx.y;
  const int re = blockIdx.x * blockDim.x + threadIdx.x;
  if (re >= p.S * p.T) return;
  const int s = re / p.T, t = re - s * p.T;
  const int B = p.B, U = p.U;
  if (p.is_pilot[t]) {
    for (int u = 0; u < U; ++u) {
      float* out = p.llr + ((((size_t)n * U + u) * p.S + s) * p.T + t) * p.W;
      for (int j = 0; j < p.W; ++j) out[j] = 0.f;
    }
    return;
  }
  double2 q[NRX_CL_MAX_RX_ANT][NRX_CL_MAX_UES], r[NRX_CL_MAX_UES][NRX_CL_MAX_UES], yt[NRX_CL_MAX_UES];
  for (int u = 0; u < U; ++u) {
    double2 v[NRX_CL_MAX_RX_ANT];
    for (int b = 0; b < B; ++b) v[b] = ldc(p.h, ((((size_t)n * U + u) * p.S + s) * p.T + t) * B + b, p.h_c128);
    for (int j = 0; j < u; ++j) {
      double2 d = make_double2(0.0, 0.0);
      for (int b = 0; b < B; ++b) {
        const double2 pr = cconjmul(q[b][j], v[b]);
        d.x += pr.x;
        d.y += pr.y;
      }
      r[j][u] = d;
      for (int b = 0; b < B; ++b) {
        const double2 pr = cmul(d, q[b][j]);
        v[b].x -= pr.x;
        v[b].y -= pr.y;
      }
    }
    double nrm = 0.0;
    for (int b = 0; b < B; ++b) nrm += v[b].x * v[b].x + v[b].y * v[b].y;
    nrm = sqrt(nrm);
    r[u][u] = make_double2(nrm, 0.0);
    for (int j = u + 1; j < U; ++j) r[j][u] = make_double2(0.0, 0.0);
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int b = 0; b < B; ++b) q[b][u] = make_double2(v[b].x * inv, v[b].y * inv);
  }
  for (int u = 0; u < U; ++u) {
    double2 acc = make_double2(0.0, 0.0);
    for (int b = 0; b < B; ++b) {
      const double2 pr = cconjmul(q[b][u], ldc(p.y, (((size_t)n * p.S + s) * p.T + t) * B + b, p.y_c128));
      acc.x += pr.x;
      acc.y += pr.y;
    }
    yt[u] = acc;
  }

  // breadth-first K-Best: paths hold the symbol index of every decided stream
  uint8_t sym[NRX_CL_MAX_K][NRX_CL_MAX_UES], nsym[NRX_CL_MAX_K][NRX_CL_MAX_UES];
  double met[NRX_CL_MAX_K], nmet[NRX_CL_MAX_K];
  int npath = 1;
  met[0] = 0.0;
  for (int level = U - 1; level >= 0; --level) {
    const int m = p.mod[n * U + level];
    const int cnt = 1 << m;
    const double2* pts = p.qam + qam_offset(m);
    int nn = 0, worst = 0;
    for (int a = 0; a < npath; ++a) {
      double2 intf = make_double2(0.0, 0.0);   // already-decided (higher) streams on this row
      for (int j = level + 1; j < U; ++j) {
        // reference pairing: R[level, level+1+i] times the i-th decided symbol,
        // i.e. stream U-1-i (classical.py:220-221); else R[level, j] * x_j
        const int js = p.ref_pairing ? U - 1 - (j - level - 1) : j;
        const int mj = p.mod[n * U + js];
        const double2 pr = cmul(r[level][j], p.qam[qam_offset(mj) + sym[a][js]]);
        intf.x += pr.x;
        intf.y += pr.y;
      }
      for (int c = 0; c < cnt; ++c) {
        const double2 rx = cmul(r[level][level], pts[c]);
        const double dx = yt[level].x - intf.x - rx.x, dy = yt[level].y - intf.y - rx.y;
        const double hh = hypot(dx, dy);
        const double mm = met[a] + hh * hh;
        int slot = -1;
        if (nn < p.K) {
          slot = nn++;
        } else if (mm < nmet[worst]) {
          slot = worst;
        }
        if (slot < 0) continue;
        nmet[slot] = mm;
        for (int j = level + 1; j < U; ++j) nsym[slot][j] = sym[a][j];
        nsym[slot][level] = static_cast<uint8_t>(c);
        if (nn == p.K) {   // keep track of the largest kept metric
          worst = 0;
          for (int i = 1; i < nn; ++i)
            if (nmet[i] > nmet[worst]) worst = i;
        }
      }
    }
    npath = nn;
    for (int a = 0; a < npath; ++a) {
      met[a] = nmet[a];
      for (int j = level; j < U; ++j) sym[a][j] = nsym[a][j];
    }
  }

  const double n0e = fmax(p.n0[n], kVarFloor);
  for (int u = 0; u < U; ++u) {
    const int m = p.mod[n * U + u];
    float* out = p.llr + ((((size_t)n * U + u) * p.S + s) * p.T + t) * p.W;
    for (int j = 0; j < m; ++j) {
      double m1 = INFINITY, m0 = INFINITY;
      for (int a = 0; a < npath; ++a) {
        if ((sym[a][u] >> (m - 1 - j)) & 1) m1 = fmin(m1, met[a]);
        else m0 = fmin(m0, met[a]);
      }
      double v = (m0 - m1) / n0e;
      if (isinf(m0)) v = p.clip;
      if (isinf(m1)) v = -p.clip;
      out[j] = static_cast<float>(fmin(fmax(v, -(double)p.clip), (double)p.clip));
    }
    for (int j = m; j < p.W; ++j) out[j] = 0.f;
  }
}

void builtin_qam(double2* out) {
  for (int m = 2; m <= 8; m += 2) {
    const int cnt = 1 << m;
    double2* pts = out + qam_offset(m);
    double e = 0.0;
    for (int i = 0; i < cnt; ++i) {
      double ax[2];
      for (int a = 0; a < 2; ++a) {
        const int nb = m / 2;
        int bits[4];
        for (int j = 0; j < nb; ++j) bits[j] = (i >> (m - 1 - (2 * j + a))) & 1;
        double amp = 1.0 - 2.0 * bits[nb - 1];
        for (int level = 1; level < nb; ++level)
          amp = (1.0 - 2.0 * bits[nb - 1 - level]) * (std::ldexp(1.0, level) - amp);
        ax[a] = amp;
      }
      pts[i] = make_double2(ax[0], ax[1]);
      const double hh = std::hypot(ax[0], ax[1]);
      e += hh * hh;
    }
    const double nrm = std::sqrt(e / cnt);
    for (int i = 0; i < cnt; ++i) pts[i] = make_double2(pts[i].x / nrm, pts[i].y / nrm);
  }
}

}  // namespace nrx_cl

using namespace nrx_cl;

extern "C" int nrx_ls_lmmse(const nrx_slot_desc* slot, int bs_antennas, int n_slots, const void* y, int y_c128,
                            const void* pilots, int pilots_c128, int n_pilot_sets, const double* n0,
                            const int32_t* mod_order, const double* qam_points, float clip, float* llr_out,
                            int llr_width, void* stream) {
  if (!slot || n_slots < 0 || !y || !pilots || !n0 || !mod_order || !llr_out || !(clip > 0.f)) return NRX_ERR_INVALID;
  if (slot->num_subcarriers < 1 || slot->num_symbols < 1 || slot->num_ues < 1 || slot->comb_size < 1 ||
      slot->num_ues > slot->comb_size || slot->num_pilot_symbols < 1 ||
      slot->num_pilot_symbols > NRX_MAX_PILOT_SYMBOLS || bs_antennas < 1)
    return NRX_ERR_INVALID;
  if (slot->num_symbols > 32 || slot->num_ues > NRX_CL_MAX_UES || bs_antennas > NRX_CL_MAX_RX_ANT ||
      llr_width < 1 || llr_width > 8)
    return NRX_ERR_UNSUPPORTED;
  if (n_pilot_sets != 1 && n_pilot_sets != n_slots) return NRX_ERR_INVALID;
  if (n_slots == 0) return NRX_OK;
  if (n_slots > 65535) return NRX_ERR_UNSUPPORTED;
  ClParams p;
  std::memset(&p, 0, sizeof(p));
  p.S = slot->num_subcarriers;
  p.T = slot->num_symbols;
  p.U = slot->num_ues;
  p.B = bs_antennas;
  p.comb = slot->comb_size;
  p.K = slot->num_pilot_symbols;
  p.F = (p.S + p.comb - 1) / p.comb;
  p.n_pilot_sets = n_pilot_sets;
  p.W = llr_width;
  for (int k = 0; k < p.K; ++k) {
    if (slot->pilot_symbols[k] < 0 || slot->pilot_symbols[k] >= p.T) return NRX_ERR_INVALID;
    p.ps[k] = slot->pilot_symbols[k];
  }
  for (int t = 0; t < p.T; ++t) {   // nearest pilot symbol, ties -> earlier (classical.py:71)
    int best = 0;
    for (int k = 1; k < p.K; ++k)
      if (std::abs(t - p.ps[k]) < std::abs(t - p.ps[best])) best = k;
    p.nearest[t] = best;
  }
  p.clip = clip;
  if (qam_points)
    std::memcpy(p.qam, qam_points, sizeof(p.qam));
  else
    builtin_qam(p.qam);
  p.y = y;
  p.y_c128 = y_c128;
  p.pilots = pilots;
  p.p_c128 = pilots_c128;
  p.n0 = n0;
  p.mod = mod_order;
  p.llr = llr_out;
  const dim3 grid((p.S * p.T + 127) / 128, n_slots);
  k_ls_lmmse<<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(p);
  const cudaError_t e = cudaPeekAtLastError();
  if (e == cudaErrorNoKernelImageForDevice || e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
    return NRX_ERR_NO_DEVICE;
  return e == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

extern "C" int nrx_kbest(const nrx_slot_desc* slot, int bs_antennas, int n_slots, const void* y, int y_c128,
                         const void* h, int h_c128, const double* n0, const int32_t* mod_order,
                         const double* qam_points, int k, int reference_pairing, float clip, float* llr_out,
                         int llr_width, void* stream) {
  if (!slot || n_slots < 0 || !y || !h || !n0 || !mod_order || !llr_out || !(clip > 0.f) || k < 1 ||
      bs_antennas < 1)
    return NRX_ERR_INVALID;
  if (slot->num_subcarriers < 1 || slot->num_symbols < 1 || slot->num_ues < 1 || slot->num_pilot_symbols < 0 ||
      slot->num_pilot_symbols > NRX_MAX_PILOT_SYMBOLS)
    return NRX_ERR_INVALID;
  if (slot->num_symbols > 32 || slot->num_ues > NRX_CL_MAX_UES || bs_antennas > NRX_CL_MAX_RX_ANT ||
      k > NRX_CL_MAX_K || llr_width < 1 || llr_width > 8)
    return NRX_ERR_UNSUPPORTED;
  if (n_slots == 0) return NRX_OK;
  if (n_slots > 65535) return NRX_ERR_UNSUPPORTED;
  KbParams p;
  std::memset(&p, 0, sizeof(p));
  p.S = slot->num_subcarriers;
  p.T = slot->num_symbols;
  p.U = slot->num_ues;
  p.B = bs_antennas;
  p.W = llr_width;
  p.K = k;
  p.ref_pairing = reference_pairing ? 1 : 0;
  for (int i = 0; i < slot->num_pilot_symbols; ++i) {
    if (slot->pilot_symbols[i] < 0 || slot->pilot_symbols[i] >= p.T) return NRX_ERR_INVALID;
    p.is_pilot[slot->pilot_symbols[i]] = 1;
  }
  p.clip = clip;
  if (qam_points)
    std::memcpy(p.qam, qam_points, sizeof(p.qam));
  else
    builtin_qam(p.qam);
  p.y = y;
  p.y_c128 = y_c128;
  p.h = h;
  p.h_c128 = h_c128;
  p.n0 = n0;
  p.mod = mod_order;
  p.llr = llr_out;
  const dim3 grid((p.S * p.T + 127) / 128, n_slots);
  k_kbest<<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(p);
  const cudaError_t e = cudaPeekAtLastError();
  if (e == cudaErrorNoKernelImageForDevice || e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
    return NRX_ERR_NO_DEVICE;
  return e == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}
