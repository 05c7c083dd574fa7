// k_slotgen.cu — GPU synthetic uplink slots (pilots, Gray QAM on the data
// REs, per-UE TDL sum-of-sinusoids channels, beamforming, AWGN) and the
// uncoded bit-error counter.  C ABI in include/nrx_slotgen.h.
//
// Reference behaviour restated here (file:line under /root/reference/pkg/src/nrxsim):
//   sample_tdl        channel.py:127-150  Jakes gains per (rx b, tx n, tap, symbol)
//   cir_to_freq       channel.py:113-124  H[s] = sum_l g_l exp(-j 2 pi s df tau_l)
//   apply_channel     channel.py:153-167  y = sum_u H_u (x_u v_u) + sqrt(n0/2)(N1 + j N2)
//   effective         channel.py:101-104  h_eff[u,b] = sum_n H[u,b,n] v[u,n]
//   generate_pilots   slot.py:130-139     QPSK on UE u's comb at the pilot symbols
//   map_bits          constellation.py:44-50, data REs subcarrier-major (slot.py:106-109)
//
// Layout and work split (one slot = S*T resource elements, "REs"):
//   k_sg_gains   grid (N*U*B), block 128: the sinusoid variates of one
//                (slot, UE, rx antenna) into shared memory, then the Jakes
//                tap gains per (tap, symbol) for every tx antenna, already
//                beamformed: G[n][u][t][b][l] (C2: 11 KB per slot, float32),
//                plus the UE's comb pilots in the nrx_forward (N,U,F,K) layout.
//   k_sg_grid    grid (ceil(S/32), N), block 4 warps: lane = subcarrier,
//                warps stride over the symbols, so G loads are warp-uniform
//                and the delay phasors of the block's 32 subcarriers are
//                built once in shared memory; per RE the transmit symbols,
//                h_eff = sum_l G E, y = sum_u h_eff x_u + noise.
//   k_sg_count   grid (ceil(S*T/256), N*U): popcount of (hard bits ^ label)
//                per data RE, warp-reduced, one atomic per warp.
// Arithmetic is float64 like the reference; where the reference's numpy
// expression fixes the operation order (Jakes argument, delay phase) the
// same order is kept with explicit round-to-nearest intrinsics (no FMA
// contraction), so a slot built from the reference's own variates matches it
// to float64 rounding of the summations.

#include <cuda_runtime.h>

#include <cmath>
#include <cstring>

#include "../../include/nrx_slotgen.h"

namespace nrx_sg {

constexpr int kMaxT = 32;
constexpr int kGridSc = 32;       // subcarriers per grid block (one per lane)
constexpr int kGridWarps = 4;     // warps per grid block, striding over the symbols
constexpr int kGainThreads = 128;
constexpr int kCountRows = 256;
constexpr int kCountPer = 4;
constexpr uint32_t kPurposeSinus = 1, kPurposeLabel = 2, kPurposeNoise = 3, kPurposePilot = 4;

__host__ __device__ inline int qam_offset(int m) {
  return m == 2 ? 0 : m == 4 ? 4 : m == 6 ? 20 : 84;
}

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11): counter-based, so every variate is a
// pure function of (seed, global slot, purpose, UE, element index).
// ---------------------------------------------------------------------------
struct U4 {
  uint32_t x, y, z, w;
};

__host__ __device__ inline uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return static_cast<uint32_t>((static_cast<uint64_t>(a) * b) >> 32);
#endif
}

__host__ __device__ inline U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = mulhi32(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = mulhi32(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// 53-bit uniform in [0, 1) from two words (the same resolution as numpy's
// random_standard_uniform).
__device__ inline double u53(uint32_t hi, uint32_t lo) {
  const uint64_t v = ((static_cast<uint64_t>(hi) << 32) | lo) >> 11;
  return static_cast<double>(v) * (1.0 / 9007199254740992.0);
}

struct SgParams {
  int S, T, U, B, NU, L, NS, K, comb, F;
  int sym_k[kMaxT];           // pilot-symbol index k of symbol t, or -1
  int taps[NRX_SG_MAX_UES];
  double tsym;                // OFDM symbol duration (1 + cp) / scs
  double two_pi_fd[NRX_SG_MAX_UES];
  double sqrt_ns;
  double sqrt_pw[NRX_SG_MAX_UES][NRX_SG_MAX_TAPS];
  double delays[NRX_SG_MAX_UES][NRX_SG_MAX_TAPS];
  double neg_two_pi_scs;
  double2 beams[NRX_SG_MAX_UES][NRX_SG_MAX_UE_ANT];
  double2 qam[NRX_SG_QAM_POINTS];
  uint32_t key0, key1;
  unsigned long long first_slot;
  // variates (NULL -> Philox)
  const double* v_angles;
  const double* v_phases;
  const uint8_t* v_labels;
  const double2* v_noise;
  const double2* v_pilots;
  // inputs
  const int32_t* mod_order;
  const double* n0;
  // outputs / workspace
  void* gains;                // (N, U, T, B, L) beamformed tap gains, synthesis type
  void* y;
  int y_c128;
  void* pilots;
  int pilots_c128;
  uint8_t* labels;
  void* h_eff;
  int h_c128;
};

__device__ inline U4 draw(const SgParams& p, unsigned long long slot, uint32_t purpose, int u, uint32_t idx) {
  return philox(U4{idx, static_cast<uint32_t>(slot), static_cast<uint32_t>(slot >> 32),
                   (purpose << 8) | static_cast<uint32_t>(u)},
                p.key0, p.key1);
}

// Arithmetic type of the synthesis: float64 for the reference-stream mode and
// complex128 outputs, float32 for device-drawn slots with complex64 outputs
// (same Philox variates; the float32 slot is the float64 one to rounding).
template <typename R> struct Cx;
template <> struct Cx<double> {
  using T = double2;
  static __device__ T make(double a, double b) { return make_double2(a, b); }
};
template <> struct Cx<float> {
  using T = float2;
  static __device__ T make(double a, double b) { return make_float2(static_cast<float>(a), static_cast<float>(b)); }
};

template <typename C>
__device__ inline C cmul(C a, C b) {
  C r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}

template <typename C>
__device__ inline void store_c(void* base, size_t i, C v, int c128) {
  if (c128)
    static_cast<double2*>(base)[i] = make_double2(v.x, v.y);
  else
    static_cast<float2*>(base)[i] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
}

__device__ inline double2 pilot_value(const SgParams& p, int n, unsigned long long slot, int u, int f, int k) {
  if (p.v_pilots) return p.v_pilots[((static_cast<size_t>(n) * p.U + u) * p.F + f) * p.K + k];
  const U4 r = draw(p, slot, kPurposePilot, u, static_cast<uint32_t>(f * p.K + k));
  return p.qam[r.x >> 30];   // QPSK points sit at offset 0 of the table
}

// The (angle, phase) variates of sinusoid k of (rx b, tx nu, tap l).
__device__ inline void sinusoid_variates(const SgParams& p, unsigned long long slot, int u, size_t vbase,
                                         uint32_t vidx, int k, double* ang, double* ph) {
  if (p.v_angles) {
    *ang = p.v_angles[vbase + k];
    *ph = p.v_phases[vbase + k];
  } else {
    const U4 r = draw(p, slot, kPurposeSinus, u, vidx + k);
    *ang = __dmul_rn(6.283185307179586, u53(r.x, r.y));
    *ph = __dmul_rn(6.283185307179586, u53(r.z, r.w));
  }
}

// One block per (slot, UE, rx antenna b).
//   phase 1: the N_u*L*NS sinusoid (omega = 2 pi fD cos(angle), phase) pairs
//            into shared memory (each drawn once);
//   phase 2: one thread per (tap l, symbol t): the Jakes gain of every tx
//            antenna, g = sum_k exp(j(omega_k t Tsym + phase_k)) / sqrt(NS)
//            * sqrt(p_l) (channel.py:139-145), beamformed on the spot:
//            G[n][u][t][b][l] = sum_nu v[u][nu] g_nu, so the per-RE work is
//            h_eff[u][b](s,t) = sum_l G[u][t][b][l] exp(-j 2 pi s df tau_l).
template <typename R>
__global__ void __launch_bounds__(kGainThreads) k_sg_gains(SgParams p) {
  using C = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  const int blk = blockIdx.x;                  // (n * U + u) * B + b
  const int b = blk % p.B, nu_idx = blk / p.B;
  const int n = nu_idx / p.U, u = nu_idx % p.U;
  const unsigned long long slot = p.first_slot + static_cast<unsigned long long>(n);
  const int L = p.taps[u], NS = p.NS;
  R* om = reinterpret_cast<R*>(sm_raw);        // [NU][L][NS]
  R* ph = om + p.NU * L * NS;
  for (int i = threadIdx.x; i < p.NU * L * NS; i += blockDim.x) {
    const int k = i % NS, l = (i / NS) % L, nu = i / (NS * L);
    const int bn = b * p.NU + nu;
    const size_t vbase = ((static_cast<size_t>(nu_idx) * p.B * p.NU + bn) * p.L + l) * NS;
    double ang, phs;
    sinusoid_variates(p, slot, u, vbase, static_cast<uint32_t>((bn * p.L + l) * NS), k, &ang, &phs);
    if (sizeof(R) == 8) {
      om[i] = static_cast<R>(__dmul_rn(p.two_pi_fd[u], cos(ang)));
    } else {
      om[i] = static_cast<R>(p.two_pi_fd[u]) * cosf(static_cast<float>(ang));
    }
    ph[i] = static_cast<R>(phs);
  }
  __syncthreads();
  C* G = reinterpret_cast<C*>(p.gains);
  for (int it = threadIdx.x; it < L * p.T; it += blockDim.x) {
    const int l = it / p.T, t = it % p.T;
    const double tt = __dmul_rn(static_cast<double>(t), p.tsym);
    C acc = Cx<R>::make(0.0, 0.0);
    for (int nu = 0; nu < p.NU; ++nu) {
      const R* o = om + (nu * L + l) * NS;
      const R* q = ph + (nu * L + l) * NS;
      C g;
      if (sizeof(R) == 8) {
        // arg = omega * t Tsym + phase, summed over k in order (channel.py:144-145)
        double re = 0.0, im = 0.0;
        for (int k = 0; k < NS; ++k) {
          double sn, cs;
          sincos(__dadd_rn(__dmul_rn(static_cast<double>(o[k]), tt), static_cast<double>(q[k])), &sn, &cs);
          re = __dadd_rn(re, cs);
          im = __dadd_rn(im, sn);
        }
        const double sp = p.sqrt_pw[u][l];
        g = Cx<R>::make(__dmul_rn(__ddiv_rn(re, p.sqrt_ns), sp), __dmul_rn(__ddiv_rn(im, p.sqrt_ns), sp));
      } else {
        const float ttf = static_cast<float>(tt);
        float re = 0.f, im = 0.f;
        for (int k = 0; k < NS; ++k) {
          float sn, cs;
          sincosf(fmaf(static_cast<float>(o[k]), ttf, static_cast<float>(q[k])), &sn, &cs);
          re += cs;
          im += sn;
        }
        const float sc = static_cast<float>(p.sqrt_pw[u][l] / p.sqrt_ns);
        g = Cx<R>::make(re * sc, im * sc);
      }
      const C v = Cx<R>::make(p.beams[u][nu].x, p.beams[u][nu].y);
      const C gv = cmul(g, v);
      acc.x += gv.x;
      acc.y += gv.y;
    }
    G[((static_cast<size_t>(nu_idx) * p.T + t) * p.B + b) * p.L + l] = acc;
  }
  if (p.pilots && b == 0) {
    const int o = u % p.comb;
    for (int it = threadIdx.x; it < p.F * p.K; it += blockDim.x) {
      const int f = it / p.K, k = it % p.K;
      const double2 v = (o + f * p.comb < p.S) ? pilot_value(p, n, slot, u, f, k) : make_double2(0.0, 0.0);
      store_c(p.pilots, static_cast<size_t>(nu_idx) * p.F * p.K + it, v, p.pilots_c128);
    }
  }
}

// Complex unit normals (re, im) of rx antennas b0 and b0 + 1 of one RE by
// Box-Muller.  Two Philox blocks A, B per antenna pair: the float64 variates
// of antenna b0 are u53(A.x, B.x), u53(A.y, B.y) and of b0 + 1
// u53(A.z, B.z), u53(A.w, B.w); the float32 path uses their leading words
// (A only), so a float32 slot is the float64 slot to rounding.
template <typename R>
__device__ inline void unit_normal_pair(const SgParams& p, unsigned long long slot, int r, int b0,
                                        typename Cx<R>::T* z);
template <>
__device__ inline void unit_normal_pair<double>(const SgParams& p, unsigned long long slot, int r, int b0,
                                                double2* z) {
  const uint32_t idx = static_cast<uint32_t>((r * ((p.B + 1) >> 1) + (b0 >> 1)) * 2);
  const U4 a = draw(p, slot, kPurposeNoise, 0, idx), c = draw(p, slot, kPurposeNoise, 0, idx + 1);
  const uint32_t w1[2] = {a.x, a.z}, w1l[2] = {c.x, c.z}, w2[2] = {a.y, a.w}, w2l[2] = {c.y, c.w};
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double rad = sqrt(-2.0 * log(1.0 - u53(w1[j], w1l[j])));   // 1 - u in (0, 1]
    double sn, cs;
    sincospi(2.0 * u53(w2[j], w2l[j]), &sn, &cs);
    z[j] = make_double2(rad * cs, rad * sn);
  }
}
template <>
__device__ inline void unit_normal_pair<float>(const SgParams& p, unsigned long long slot, int r, int b0,
                                               float2* z) {
  const uint32_t idx = static_cast<uint32_t>((r * ((p.B + 1) >> 1) + (b0 >> 1)) * 2);
  const U4 a = draw(p, slot, kPurposeNoise, 0, idx);
  const uint32_t w1[2] = {a.x, a.z}, w2[2] = {a.y, a.w};
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    // leading 24 bits of the float64 variates: u1 = 1 - u in (0, 1]
    const float u1 = static_cast<float>(16777216u - (w1[j] >> 8)) * 5.9604644775390625e-8f;
    const float rad = sqrtf(-2.f * __logf(u1));
    // cis(2 pi u2) = -cis(2 pi (u2 - 1/2)), argument inside [-pi, pi)
    const float u2 = static_cast<float>(w2[j] >> 8) * 5.9604644775390625e-8f - 0.5f;
    float sn, cs;
    __sincosf(6.283185307179586f * u2, &sn, &cs);
    z[j] = make_float2(-rad * cs, -rad * sn);
  }
}

// Grid block = 32 subcarriers (one per lane) x all symbols (warps stride
// over t), one slot.  The delay phasors E[u][l](s) of the block's
// subcarriers and the slot's beamformed tap gains G[u][t][b][l] are staged
// in shared memory (G reads are warp-uniform: every lane of a warp has the
// same t); per (s, t) a thread forms the UEs' symbols, then per rx antenna
// h_eff = sum_l G E, y = sum_u h_eff x_u + noise.
template <typename R, int LMAX>
__global__ void __launch_bounds__(kGridWarps * 32, sizeof(R) == 4 ? 8 : 4) k_sg_grid(SgParams p) {
  using C = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char sm_raw[];
  C* E = reinterpret_cast<C*>(sm_raw);                   // [U][L][32]
  C* Gs = E + p.U * p.L * kGridSc;                       // [U][T][B][L]
  const int n = blockIdx.y;
  const unsigned long long slot = p.first_slot + static_cast<unsigned long long>(n);
  const int s0 = blockIdx.x * kGridSc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ng = p.U * p.T * p.B * p.L;
  const C* G = reinterpret_cast<const C*>(p.gains) + static_cast<size_t>(n) * ng;
  for (int i = threadIdx.x; i < ng; i += blockDim.x) Gs[i] = G[i];
  for (int i = threadIdx.x; i < p.U * p.L * kGridSc; i += blockDim.x) {
    const int sc = i % kGridSc, l = (i / kGridSc) % p.L, u = i / (kGridSc * p.L);
    double2 e = make_double2(0.0, 0.0);
    if (l < p.taps[u] && s0 + sc < p.S) {
      // phase = -2j*pi*scs * outer(delays, s): theta = (-2 pi scs) * (tau * s)  (channel.py:121)
      const double th = __dmul_rn(p.neg_two_pi_scs, __dmul_rn(p.delays[u][l], static_cast<double>(s0 + sc)));
      sincos(th, &e.y, &e.x);
    }
    E[i] = Cx<R>::make(e.x, e.y);
  }
  __syncthreads();
  const int s = s0 + lane;
  if (s >= p.S) return;
  const int ST = p.S * p.T;
  const double n0 = p.n0 ? p.n0[n] : 0.0;
  const R scale = static_cast<R>(n0 > 0.0 ? sqrt(n0 / 2.0) : 0.0);
  int mods[NRX_SG_MAX_UES], taps[NRX_SG_MAX_UES];
#pragma unroll
  for (int u = 0; u < NRX_SG_MAX_UES; ++u) {
    mods[u] = u < p.U ? p.mod_order[n * p.U + u] : 2;
    taps[u] = u < p.U ? p.taps[u] : 0;
  }

  for (int t = warp; t < p.T; t += kGridWarps) {
    const int r = s * p.T + t;
    const int k_sym = p.sym_k[t];
    const size_t re_global = static_cast<size_t>(n) * ST + r;
    U4 lq{0u, 0u, 0u, 0u};
    if (k_sym < 0 && !p.v_labels) lq = draw(p, slot, kPurposeLabel, 0, static_cast<uint32_t>(r));
    C x[NRX_SG_MAX_UES];
#pragma unroll
    for (int u = 0; u < NRX_SG_MAX_UES; ++u) {
      x[u] = Cx<R>::make(0.0, 0.0);
      if (u >= p.U) continue;
      uint8_t lab = 0;
      if (k_sym < 0) {                                   // data RE
        const int m = mods[u];
        if (p.v_labels) {
          lab = p.v_labels[(static_cast<size_t>(n) * p.U + u) * ST + r];
        } else {
          const uint32_t w = u == 0 ? lq.x : u == 1 ? lq.y : u == 2 ? lq.z : lq.w;
          lab = static_cast<uint8_t>(w >> (32 - m));
        }
        const double2 q = p.qam[qam_offset(m) + lab];
        x[u] = Cx<R>::make(q.x, q.y);
      } else if (s % p.comb == u % p.comb) {             // UE u's pilot RE
        const double2 q = pilot_value(p, n, slot, u, s / p.comb, k_sym);
        x[u] = Cx<R>::make(q.x, q.y);
      }
      if (p.labels) p.labels[(static_cast<size_t>(n) * p.U + u) * ST + r] = lab;
    }
    for (int b0 = 0; b0 < p.B; b0 += 2) {
      C z[2] = {Cx<R>::make(0.0, 0.0), Cx<R>::make(0.0, 0.0)};
      if (scale > R(0)) {
        if (p.v_noise) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (b0 + j < p.B) {
              const double2 zz = p.v_noise[re_global * p.B + b0 + j];
              z[j] = Cx<R>::make(zz.x, zz.y);
            }
          }
        } else {
          unit_normal_pair<R>(p, slot, r, b0, z);
        }
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int b = b0 + j;
        if (b >= p.B) break;
        C acc = Cx<R>::make(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < NRX_SG_MAX_UES; ++u) {
          if (u >= p.U) continue;
          const C* g = Gs + ((u * p.T + t) * p.B + b) * p.L;
          const C* e = E + u * p.L * kGridSc + lane;
          C h = Cx<R>::make(0.0, 0.0);
#pragma unroll
          for (int l = 0; l < LMAX; ++l) {
            if (l < taps[u]) {
              const C pr = cmul(g[l], e[l * kGridSc]);
              h.x += pr.x;
              h.y += pr.y;
            }
          }
          const C hx = cmul(h, x[u]);
          acc.x += hx.x;
          acc.y += hx.y;
          if (p.h_eff) store_c(p.h_eff, ((static_cast<size_t>(n) * p.U + u) * ST + r) * p.B + b, h, p.h_c128);
        }
        if (sizeof(R) == 8) {
          acc.x = __dadd_rn(acc.x, __dmul_rn(scale, z[j].x));
          acc.y = __dadd_rn(acc.y, __dmul_rn(scale, z[j].y));
        } else {
          acc.x += scale * z[j].x;
          acc.y += scale * z[j].y;
        }
        store_c(p.y, re_global * p.B + b, acc, p.y_c128);
      }
    }
  }
}

struct CountParams {
  int S, T, U, W;
  int sym_k[kMaxT];
  const float* llr;
  const uint8_t* labels;
  const int32_t* mod_order;
  unsigned long long* errs;
};

// Hard bits of one LLR row (LLR > 0 -> 1, label position j = bit m-1-j).
template <int W>
__device__ inline uint32_t hard_bits(const float* row, int m) {
  float v[W > 0 ? W : 8];
  if (W == 4 || W == 8) {
#pragma unroll
    for (int i = 0; i < (W > 0 ? W : 8); i += 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(row) + i / 4);
      v[i] = q.x; v[i + 1] = q.y; v[i + 2] = q.z; v[i + 3] = q.w;
    }
  } else if (W == 2 || W == 6) {
#pragma unroll
    for (int i = 0; i < W; i += 2) {
      const float2 q = __ldg(reinterpret_cast<const float2*>(row) + i / 2);
      v[i] = q.x; v[i + 1] = q.y;
    }
  } else {
    for (int i = 0; i < m; ++i) v[i] = __ldg(row + i);
  }
  uint32_t hard = 0;
#pragma unroll
  for (int j = 0; j < (W > 0 ? W : 8); ++j)
    if (j < m) hard = (hard << 1) | (v[j] > 0.f ? 1u : 0u);
  return hard;
}

// Each thread scores kCountPer REs of one (slot, UE) stream (independent
// loads in flight), warp-reduces, one atomic per warp.
template <int W>
__global__ void __launch_bounds__(kCountRows) k_sg_count(CountParams p) {
  const int slab = blockIdx.y;
  const int ST = p.S * p.T;
  const int m = p.mod_order[slab];
  const int width = W > 0 ? W : p.W;
  uint32_t e = 0;
#pragma unroll
  for (int k = 0; k < kCountPer; ++k) {
    const int r = (blockIdx.x * kCountPer + k) * kCountRows + threadIdx.x;
    if (r < ST && p.sym_k[r % p.T] < 0) {
      const uint32_t hard = hard_bits<W>(p.llr + (static_cast<size_t>(slab) * ST + r) * width, m);
      e += __popc((hard ^ p.labels[static_cast<size_t>(slab) * ST + r]) & ((1u << m) - 1u));
    }
  }
  const uint32_t tot = __reduce_add_sync(0xffffffffu, e);
  if ((threadIdx.x & 31) == 0 && tot) atomicAdd(p.errs + slab, static_cast<unsigned long long>(tot));
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

int max_taps(const nrx_slot_desc* s, const nrx_channel_desc* c) {
  int L = 1;
  for (int u = 0; u < s->num_ues; ++u) L = c->profiles[u].num_taps > L ? c->profiles[u].num_taps : L;
  return L;
}

int validate(const nrx_slot_desc* s, const nrx_channel_desc* c) {
  if (!s || !c) return NRX_ERR_INVALID;
  if (s->num_subcarriers < 1 || s->num_symbols < 1 || s->num_ues < 1 || s->comb_size < 1) return NRX_ERR_INVALID;
  if (s->num_ues > s->comb_size) return NRX_ERR_INVALID;               // slot.py:65-66
  if (s->num_pilot_symbols < 1 || s->num_pilot_symbols > NRX_MAX_PILOT_SYMBOLS) return NRX_ERR_INVALID;
  for (int k = 0; k < s->num_pilot_symbols; ++k)
    if (s->pilot_symbols[k] < 0 || s->pilot_symbols[k] >= s->num_symbols) return NRX_ERR_INVALID;
  if (s->num_symbols > kMaxT || s->num_ues > NRX_SG_MAX_UES) return NRX_ERR_UNSUPPORTED;
  if (static_cast<long long>(s->num_subcarriers) * s->num_symbols * NRX_SG_MAX_RX_ANT >= (1ll << 31))
    return NRX_ERR_UNSUPPORTED;
  if (c->bs_antennas < 1 || c->ue_antennas < 1 || c->num_sinusoids < 1) return NRX_ERR_INVALID;
  if (c->bs_antennas > NRX_SG_MAX_RX_ANT || c->ue_antennas > NRX_SG_MAX_UE_ANT || c->num_sinusoids > 4096)
    return NRX_ERR_UNSUPPORTED;
  if (!(c->subcarrier_spacing_hz > 0.0) || !(c->cp_fraction >= 0.0)) return NRX_ERR_INVALID;
  const double cp_s = c->cp_fraction / c->subcarrier_spacing_hz;
  for (int u = 0; u < s->num_ues; ++u) {
    const nrx_tdl_profile& pr = c->profiles[u];
    if (pr.num_taps < 1) return NRX_ERR_INVALID;
    if (pr.num_taps > NRX_SG_MAX_TAPS) return NRX_ERR_UNSUPPORTED;
    double sum = 0.0;
    for (int l = 0; l < pr.num_taps; ++l) {
      if (!(pr.delays_s[l] >= 0.0) || (l && pr.delays_s[l] < pr.delays_s[l - 1])) return NRX_ERR_INVALID;
      if (!(pr.powers[l] >= 0.0)) return NRX_ERR_INVALID;
      sum += pr.powers[l];
    }
    if (std::fabs(sum - 1.0) > 1e-9) return NRX_ERR_INVALID;           // channel.py:47-48
    if (pr.delays_s[pr.num_taps - 1] > cp_s) return NRX_ERR_INVALID;    // channel.py:135-138
    if (!std::isfinite(pr.doppler_hz)) return NRX_ERR_INVALID;
  }
  return NRX_OK;
}

// Built-in Gray QAM table (constellation.py:58-82): point i carries the
// big-endian label of i, even label positions steer the real axis.
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
      const double h = std::hypot(ax[0], ax[1]);
      e += h * h;
    }
    const double nrm = std::sqrt(e / cnt);
    for (int i = 0; i < cnt; ++i) pts[i] = make_double2(pts[i].x / nrm, pts[i].y / nrm);
  }
}

int fill_params(const nrx_slot_desc* s, const nrx_channel_desc* c, SgParams* p) {
  std::memset(p, 0, sizeof(*p));
  p->S = s->num_subcarriers;
  p->T = s->num_symbols;
  p->U = s->num_ues;
  p->B = c->bs_antennas;
  p->NU = c->ue_antennas;
  p->L = max_taps(s, c);
  p->NS = c->num_sinusoids;
  p->K = s->num_pilot_symbols;
  p->comb = s->comb_size;
  p->F = (p->S + p->comb - 1) / p->comb;
  for (int t = 0; t < kMaxT; ++t) p->sym_k[t] = -1;
  // a symbol listed twice keeps its last index k (numpy fancy assignment)
  for (int k = 0; k < s->num_pilot_symbols; ++k) p->sym_k[s->pilot_symbols[k]] = k;
  const double two_pi = 2.0 * 3.141592653589793;
  p->tsym = (1.0 + c->cp_fraction) / c->subcarrier_spacing_hz;        // slot.py:85-87
  p->sqrt_ns = std::sqrt(static_cast<double>(c->num_sinusoids));
  p->neg_two_pi_scs = (-two_pi) * c->subcarrier_spacing_hz;
  for (int u = 0; u < p->U; ++u) {
    const nrx_tdl_profile& pr = c->profiles[u];
    p->taps[u] = pr.num_taps;
    p->two_pi_fd[u] = two_pi * pr.doppler_hz;
    for (int l = 0; l < pr.num_taps; ++l) {
      p->sqrt_pw[u][l] = std::sqrt(pr.powers[l]);
      p->delays[u][l] = pr.delays_s[l];
    }
    for (int a = 0; a < p->NU; ++a) p->beams[u][a] = make_double2(c->beams[u][a][0], c->beams[u][a][1]);
  }
  return NRX_OK;
}

size_t gains_bytes(const SgParams& p, int n_slots) {
  return static_cast<size_t>(n_slots) * p.U * p.T * p.B * p.L * sizeof(double2);
}

template <typename R>
int launch_synth(const SgParams& q, int n_slots, cudaStream_t st) {
  using C = typename Cx<R>::T;
  const size_t gsm = 2 * static_cast<size_t>(q.NU) * q.L * q.NS * sizeof(R);
  const size_t esm = (static_cast<size_t>(q.U) * q.L * kGridSc + static_cast<size_t>(q.U) * q.T * q.B * q.L) *
                     sizeof(C);
  if (gsm > 200 * 1024 || esm > 200 * 1024) return NRX_ERR_UNSUPPORTED;
  auto gain_fn = k_sg_gains<R>;
  auto grid_fn = q.L <= 8 ? k_sg_grid<R, 8> : k_sg_grid<R, NRX_SG_MAX_TAPS>;
  if (gsm > 48 * 1024 &&
      cudaFuncSetAttribute(gain_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(gsm)) != cudaSuccess)
    return NRX_ERR_CUDA;
  if (esm > 48 * 1024 &&
      cudaFuncSetAttribute(grid_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(esm)) != cudaSuccess)
    return NRX_ERR_CUDA;
  gain_fn<<<n_slots * q.U * q.B, kGainThreads, gsm, st>>>(q);
  grid_fn<<<dim3((q.S + kGridSc - 1) / kGridSc, n_slots), kGridWarps * 32, esm, st>>>(q);
  return NRX_OK;
}

}  // namespace nrx_sg

using namespace nrx_sg;

extern "C" int nrx_synth_validate(const nrx_slot_desc* slot, const nrx_channel_desc* chan) {
  return validate(slot, chan);
}

extern "C" size_t nrx_synth_workspace_bytes(const nrx_slot_desc* slot, const nrx_channel_desc* chan, int n_slots) {
  if (validate(slot, chan) != NRX_OK || n_slots < 0) return 0;
  SgParams p;
  fill_params(slot, chan, &p);
  const size_t b = gains_bytes(p, n_slots);
  return b ? b : 16;
}

extern "C" int nrx_synth_slots(const nrx_slot_desc* slot, const nrx_channel_desc* chan, int n_slots,
                               uint64_t seed, uint64_t first_slot, const int32_t* mod_order, const double* n0,
                               const nrx_slot_variates* variates, const double* qam_points, void* y, int y_c128,
                               void* pilots, int pilots_c128, uint8_t* labels, void* h_eff, int h_eff_c128,
                               void* workspace, size_t workspace_bytes, void* stream) {
  const int v = validate(slot, chan);
  if (v != NRX_OK) return v;
  if (n_slots < 0 || !mod_order || !y) return NRX_ERR_INVALID;
  if (n_slots == 0) return NRX_OK;
  SgParams q;   // ~7 KB, passed by value as the kernel parameter block
  fill_params(slot, chan, &q);
  if (workspace_bytes < gains_bytes(q, n_slots) || !workspace) return NRX_ERR_WORKSPACE;
  if (qam_points) {
    std::memcpy(q.qam, qam_points, sizeof(q.qam));
  } else {
    builtin_qam(q.qam);
  }
  q.key0 = static_cast<uint32_t>(seed);
  q.key1 = static_cast<uint32_t>(seed >> 32);
  q.first_slot = first_slot;
  if (variates) {
    q.v_angles = variates->angles;
    q.v_phases = variates->phases;
    if ((q.v_angles == nullptr) != (q.v_phases == nullptr)) return NRX_ERR_INVALID;
    q.v_labels = variates->labels;
    q.v_noise = reinterpret_cast<const double2*>(variates->noise);
    q.v_pilots = reinterpret_cast<const double2*>(variates->pilots);
  }
  q.mod_order = mod_order;
  q.n0 = n0;
  q.gains = workspace;
  q.y = y;
  q.y_c128 = y_c128;
  q.pilots = pilots;
  q.pilots_c128 = pilots_c128;
  q.labels = labels;
  q.h_eff = h_eff;
  q.h_c128 = h_eff_c128;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // float64 when continuous variates come from the caller (reference stream) or a
  // complex128 output is asked for; supplied labels / pilots alone keep float32
  const bool exact = (variates && (variates->angles || variates->noise)) || y_c128 || (h_eff && h_eff_c128);
  const int rc = exact ? launch_synth<double>(q, n_slots, st) : launch_synth<float>(q, n_slots, st);
  if (rc != NRX_OK) return rc;
  const cudaError_t e = cudaPeekAtLastError();
  if (e == cudaErrorNoKernelImageForDevice || e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
    return NRX_ERR_NO_DEVICE;
  return e == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

extern "C" int nrx_count_bit_errors(const nrx_slot_desc* slot, int n_slots, const float* llr, int llr_width,
                                    const uint8_t* labels, const int32_t* mod_order, unsigned long long* bit_errors,
                                    void* stream) {
  if (!slot || n_slots < 0 || !llr || !labels || !mod_order || !bit_errors) return NRX_ERR_INVALID;
  if (slot->num_subcarriers < 1 || slot->num_symbols < 1 || slot->num_ues < 1) return NRX_ERR_INVALID;
  if (slot->num_symbols > kMaxT || llr_width < 1 || llr_width > 8) return NRX_ERR_UNSUPPORTED;
  if (slot->num_pilot_symbols < 0 || slot->num_pilot_symbols > NRX_MAX_PILOT_SYMBOLS) return NRX_ERR_INVALID;
  if (n_slots == 0) return NRX_OK;
  CountParams p;
  p.S = slot->num_subcarriers;
  p.T = slot->num_symbols;
  p.U = slot->num_ues;
  p.W = llr_width;
  for (int t = 0; t < kMaxT; ++t) p.sym_k[t] = -1;
  for (int k = 0; k < slot->num_pilot_symbols; ++k) {
    if (slot->pilot_symbols[k] < 0 || slot->pilot_symbols[k] >= p.T) return NRX_ERR_INVALID;
    p.sym_k[slot->pilot_symbols[k]] = k;
  }
  p.llr = llr;
  p.labels = labels;
  p.mod_order = mod_order;
  p.errs = bit_errors;
  const dim3 grid((p.S * p.T + kCountRows * kCountPer - 1) / (kCountRows * kCountPer), n_slots * p.U);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (llr_width) {
    case 2: k_sg_count<2><<<grid, kCountRows, 0, st>>>(p); break;
    case 4: k_sg_count<4><<<grid, kCountRows, 0, st>>>(p); break;
    case 6: k_sg_count<6><<<grid, kCountRows, 0, st>>>(p); break;
    case 8: k_sg_count<8><<<grid, kCountRows, 0, st>>>(p); break;
    default: k_sg_count<0><<<grid, kCountRows, 0, st>>>(p); break;
  }
  const cudaError_t e = cudaPeekAtLastError();
  if (e == cudaErrorNoKernelImageForDevice || e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
    return NRX_ERR_NO_DEVICE;
  return e == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

extern "C" void nrx_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  const U4 r = philox(U4{ctr[0], ctr[1], ctr[2], ctr[3]}, key[0], key[1]);
  out[0] = r.x;
  out[1] = r.y;
  out[2] = r.z;
  out[3] = r.w;
}
