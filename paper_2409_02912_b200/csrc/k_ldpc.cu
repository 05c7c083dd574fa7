// k_ldpc.cu — GPU LDPC decoding (flooding min-sum, early exit on parity) and
// staircase (IRA) encoding.  C ABI in include/nrx_ldpc.h.
//
// Reference (/root/reference/pkg/src/nrxsim/ldpc.py): LdpcCode.decode
// ldpc.py:99-178, check_parity :91-97, encode :88-90, rate matching
// :303-330.  The decoder keeps the reference's float32 operation order, so
// the decoded bits and success flags are bit-identical
// (tests/test_gpu_ldpc.py against tests/golden/ldpc_*.npz):
//   total_j = chan_j + ((c2v_0 + c2v_1) + c2v_2)      variable update
//   v2c     = total_col - c2v                          check update
//   c2v     = (row_sign * sgn) * (s == argmin ? min2 : min1)
//
// Codewords are decoded 32 at a time, interleaved: lane l of every warp
// works on codeword l of its group, so the random gathers of the Tanner
// graph move 128 contiguous bytes (one value per codeword) instead of a
// 32-byte sector per 4-byte value.  Per iteration two launches (grid.y =
// group): k_ldpc_var (four variables per warp: totals + hard bits) and
// k_ldpc_check_rows / k_ldpc_check (two rows per warp for row widths 5 and 6,
// else one: syndrome, then min-sum messages; the lanes with an unsatisfied
// check OR-ed into a per-group mask).  The next variable pass marks the
// codewords whose checks were all satisfied as done: a done lane is skipped
// from then on, exactly the reference's per-codeword early exit, and a group
// with all lanes done returns at once.  A final variable pass gives the hard
// bits of codewords that never converged (the reference's for-else branch).
//
// Encoder (codes with a staircase parity part): information bits placed,
// per-check information syndromes s_i, then the Z interleaved accumulator
// chains p_i = s_i ^ p_{i-Z} (one thread per chain), and the transmitted
// positions gathered.

#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <algorithm>
#include <vector>

#include "../../include/nrx_ldpc.h"

struct nrx_ldpc_code {
  int n, m, k, dmax, cdeg, k_eff, ntx, has_chain, chain_step;
  int32_t* row_cols;   // (m, dmax)
  int32_t* col_rows;   // (n, cdeg)
  int32_t* col_slots;  // (n, cdeg)
  int32_t* chan_src;   // (n): transmitted index, -1 punctured, -2 shortened
  int32_t* keep_pos;   // (k_eff): mother positions of the kept info bits
  int32_t* tx_pos;     // (ntx)
  int32_t* skip_pos;   // (n_skip): punctured and shortened positions, or null
  int n_skip;
  int32_t* info_slot;  // (n): payload index of an info position, -1 shortened, -2 parity
  int32_t* chain_cols; // (m) or null
  int4* edges;         // (n): the column's messages as row * dmax + slot, -1 padded
};

namespace nrx_ldpc {

constexpr float kShortenedLlr = 60.0f;   // ldpc.py:25
constexpr int kThreads = 256;

constexpr int kLanes = 32;           // codewords interleaved per group, one per lane
constexpr int kWarps = 8;            // warps per block
constexpr int kVarsPerWarp = 4;      // variables per warp in the variable update

// Decoder state, codeword-interleaved: element e of group g for lane l lives
// at [(g * count + e) * 32 + l], so a warp working on one variable / check
// moves 128 contiguous bytes for 32 codewords at once.
struct DecWs {
  float* chan;      // [G][n][32]
  float* total;     // [G][n][32]
  float* c2v;       // [G][m][dmax][32]
  uint32_t* done;   // [G] lane mask of finished codewords
  uint32_t* unsat;  // [2][G][32] lanes with an unsatisfied check, by iteration parity,
                    // OR-ed by the check blocks into 32 slots (blockIdx.x % 32)
};

constexpr int kUnsatSlots = 32;     // spread of the check blocks' unsatisfied-lane atomics

size_t align256(size_t v) { return (v + 255) / 256 * 256; }

DecWs dec_layout(const nrx_ldpc_code& c, int n_cw, uint8_t* base, size_t* total_bytes) {
  DecWs w{};
  const size_t G = (size_t)(n_cw + kLanes - 1) / kLanes;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align256(off + bytes);
    return o;
  };
  const size_t o_chan = take(sizeof(float) * c.n * kLanes * G);
  const size_t o_total = take(sizeof(float) * c.n * kLanes * G);
  const size_t o_c2v = take(sizeof(float) * (size_t)c.m * c.dmax * kLanes * G);
  const size_t o_done = take(sizeof(uint32_t) * G);
  const size_t o_unsat = take(sizeof(uint32_t) * 2 * G * kUnsatSlots);
  if (total_bytes) *total_bytes = off;
  if (base) {
    w.chan = reinterpret_cast<float*>(base + o_chan);
    w.total = reinterpret_cast<float*>(base + o_total);
    w.c2v = reinterpret_cast<float*>(base + o_c2v);
    w.done = reinterpret_cast<uint32_t*>(base + o_done);
    w.unsat = reinterpret_cast<uint32_t*>(base + o_unsat);
  }
  return w;
}

struct EncWs {
  uint8_t* cw;
  uint8_t* syn;
};

EncWs enc_layout(const nrx_ldpc_code& c, int n_cw, uint8_t* base, size_t* total_bytes) {
  EncWs w{};
  const size_t o_cw = 0;
  const size_t o_syn = align256((size_t)c.n * n_cw);
  const size_t end = align256(o_syn + (size_t)c.m * n_cw);
  if (total_bytes) *total_bytes = end;
  if (base) {
    w.cw = base + o_cw;
    w.syn = base + o_syn;
  }
  return w;
}

// ---------------------------------------------------------------------------
// decoder kernels (grid.y = group of 32 codewords)
// ---------------------------------------------------------------------------

// Channel values only: the zero initial messages are never stored, the
// first iteration's kernels take them as zero (template flag FIRST).  The received
// LLRs are transposed through shared memory: read codeword-major (coalesced
// along the transmitted index), written lane-per-codeword at their mother
// positions (128 B per position).
constexpr int kInitTile = 256;

__global__ void __launch_bounds__(kWarps * 32) k_ldpc_init_tx(nrx_ldpc_code c, const float* llr, int n_cw, DecWs w) {
  __shared__ float tile[kLanes][kInitTile + 1];
  const int g = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int base = blockIdx.x * kInitTile;
  for (int l = warp; l < kLanes; l += kWarps) {
    const int cw = g * kLanes + l;
    const float* row = llr + (size_t)cw * c.ntx + base;
#pragma unroll
    for (int i = lane; i < kInitTile; i += 32)
      tile[l][i] = cw < n_cw && base + i < c.ntx ? row[i] : 0.f;
  }
  __syncthreads();
  float* chan = w.chan + (size_t)g * c.n * kLanes + lane;
  for (int i = warp; i < kInitTile && base + i < c.ntx; i += kWarps)   // ln(p0/p1): the negated logit LLR
    chan[(size_t)__ldg(c.tx_pos + base + i) * kLanes] = g * kLanes + lane < n_cw ? -tile[lane][i] : 0.f;
}

// Positions that are not transmitted (punctured: erased, shortened: known
// zero) and the group's early-exit state.
__global__ void k_ldpc_init_state(nrx_ldpc_code c, int n_cw, DecWs w) {
  const int g = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const bool live = g * kLanes + lane < n_cw;
  float* chan = w.chan + (size_t)g * c.n * kLanes + lane;
  for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < c.n_skip; i += (gridDim.x * blockDim.x) >> 5) {
    const int j = __ldg(c.skip_pos + i);
    chan[(size_t)j * kLanes] = live && __ldg(c.chan_src + j) == -2 ? kShortenedLlr : 0.f;
  }
  if (blockIdx.x == 0 && threadIdx.x < kUnsatSlots)   // "iteration -1": no lane newly satisfied
    w.unsat[((size_t)gridDim.y + g) * kUnsatSlots + threadIdx.x] = 0xffffffffu;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int valid = min(kLanes, n_cw - g * kLanes);
    w.done[g] = valid >= kLanes ? 0u : ~((1u << valid) - 1u);   // absent codewords count as done
  }
}

// Variable update, warp per kVarsPerWarp variables (their edge records and
// message gathers all issued before use): total = chan + ((c2v_0 + c2v_1) + c2v_2).
// The hard bits are the signs of the totals; a converged lane's totals stay
// frozen, so they are its decision.
//
// Early exit: a codeword whose checks were all satisfied by the previous
// check pass's hard bits (parity `1 - par` of w.unsat) is done from now on;
// block 0 records the new mask and clears parity `par` for this iteration's
// check pass.  FIRST: the messages are still all zero (not read).
template <bool FIRST>
__global__ void __launch_bounds__(kWarps * 32) k_ldpc_var(nrx_ldpc_code c, DecWs w, int par) {
  const int g = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const uint32_t unsat =
      __reduce_or_sync(0xffffffffu, w.unsat[((size_t)(par ^ 1) * gridDim.y + g) * kUnsatSlots + lane]);
  const uint32_t done = w.done[g] | ~unsat;
  if (blockIdx.x == 0 && threadIdx.x < kUnsatSlots) {
    w.unsat[((size_t)par * gridDim.y + g) * kUnsatSlots + lane] = 0u;
    if (lane == 0) w.done[g] = done;
  }
  if (done == 0xffffffffu) return;
  if ((done >> lane) & 1u) return;
  const int j0 = (blockIdx.x * kWarps + (threadIdx.x >> 5)) * kVarsPerWarp;
  const float* c2v = w.c2v + (size_t)g * c.m * c.dmax * kLanes + lane;
  int4 ed[kVarsPerWarp];
#pragma unroll
  for (int q = 0; q < kVarsPerWarp; ++q)
    ed[q] = j0 + q < c.n ? __ldg(c.edges + j0 + q) : make_int4(-1, -1, -1, -1);
  float v[kVarsPerWarp][3], ch[kVarsPerWarp];
#pragma unroll
  for (int q = 0; q < kVarsPerWarp; ++q) {
    const int e3[3] = {ed[q].x, ed[q].y, ed[q].z};
#pragma unroll
    for (int t = 0; t < 3; ++t)
      v[q][t] = !FIRST && e3[t] >= 0 ? c2v[(size_t)e3[t] * kLanes] : 0.f;
    ch[q] = j0 + q < c.n ? w.chan[((size_t)g * c.n + j0 + q) * kLanes + lane] : 0.f;
  }
#pragma unroll
  for (int q = 0; q < kVarsPerWarp; ++q) {
    if (j0 + q >= c.n) break;
    float s = v[q][0];
    if (ed[q].y >= 0) s = __fadd_rn(s, v[q][1]);
    if (ed[q].z >= 0) s = __fadd_rn(s, v[q][2]);
    if (ed[q].x < 0) s = 0.f;
    w.total[((size_t)g * c.n + j0 + q) * kLanes + lane] = __fadd_rn(ch[q], s);
  }
}

// Check update, warp per check: v2c of every slot kept in registers between
// the min-sum pass and the message write; plus the lanes whose hard bits
// violate this check.  DMAX > 0: row width fixed at compile time.
template <int DMAX, bool FIRST>
__global__ void __launch_bounds__(kWarps * 32) k_ldpc_check(nrx_ldpc_code c, DecWs w, int par) {
  __shared__ uint32_t block_unsat;
  const int g = blockIdx.y;
  const uint32_t done = w.done[g];
  if (done == 0xffffffffu) return;   // uniform over the block
  if (threadIdx.x == 0) block_unsat = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int dmax = DMAX > 0 ? DMAX : c.dmax;
  int syn = 0;
  if (r < c.m && !((done >> lane) & 1u)) {
    const int32_t* cols = c.row_cols + (size_t)r * dmax;
    float* msg = w.c2v + (((size_t)g * c.m + r) * dmax) * kLanes + lane;
    const float* tot = w.total + (size_t)g * c.n * kLanes + lane;
    constexpr int RD = DMAX > 0 ? DMAX : 1;
    float xs[RD];
    int cl[RD];
    float min1 = INFINITY, min2 = INFINITY;
    int amin = 0, neg = 0;
    bool first = true;
#pragma unroll
    for (int s = 0; s < (DMAX > 0 ? DMAX : NRX_LDPC_MAX_ROW_DEG); ++s) {
      if (s >= dmax) break;
      const int col = __ldg(cols + s);
      float mag = INFINITY, x = 0.f;
      if (col >= 0) {
        const float v = tot[(size_t)col * kLanes];
        syn ^= v < 0.f ? 1 : 0;
        x = FIRST ? v : __fsub_rn(v, msg[s * kLanes]);
        mag = fabsf(x);
        neg ^= x < 0.f ? 1 : 0;
      }
      if (DMAX > 0) {
        xs[s] = x;
        cl[s] = col;
      }
      // np.argmin: first index of the smallest magnitude (invalid slots are +inf)
      if (first || mag < min1) {
        if (!first) min2 = min1;
        min1 = mag;
        amin = s;
        first = false;
      } else if (mag < min2) {
        min2 = mag;
      }
    }
    const float rs = neg ? -1.f : 1.f;
#pragma unroll
    for (int s = 0; s < (DMAX > 0 ? DMAX : NRX_LDPC_MAX_ROW_DEG); ++s) {
      if (s >= dmax) break;
      const int col = DMAX > 0 ? cl[s] : __ldg(cols + s);
      if (col < 0) {
        msg[s * kLanes] = 0.f;
        continue;
      }
      const float x = DMAX > 0 ? xs[s] : FIRST ? tot[(size_t)col * kLanes]
                                                : __fsub_rn(tot[(size_t)col * kLanes], msg[s * kLanes]);
      const float sg = x < 0.f ? -1.f : 1.f;
      msg[s * kLanes] = __fmul_rn(rs * sg, s == amin ? min2 : min1);
    }
  }
  const uint32_t bal = __ballot_sync(0xffffffffu, syn);
  if (lane == 0 && bal) atomicOr(&block_unsat, bal);
  __syncthreads();
  if (threadIdx.x == 0 && block_unsat)
    atomicOr(w.unsat + ((size_t)par * gridDim.y + g) * kUnsatSlots + blockIdx.x % kUnsatSlots, block_unsat);
}

// Check update for a fixed row width, KC checks per warp: every column
// index, total and previous message of the KC rows is loaded before any is
// used (KC x DMAX gathers in flight per warp), then each row runs the same
// min-sum arithmetic as k_ldpc_check.
template <int DMAX, bool FIRST, int KC>
__global__ void __launch_bounds__(kWarps * 32) k_ldpc_check_rows(nrx_ldpc_code c, DecWs w, int par) {
  __shared__ uint32_t block_unsat;
  const int g = blockIdx.y;
  const uint32_t done = w.done[g];
  if (done == 0xffffffffu) return;   // uniform over the block
  if (threadIdx.x == 0) block_unsat = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int r0 = (blockIdx.x * kWarps + (threadIdx.x >> 5)) * KC;
  int syn = 0;
  if (r0 < c.m && !((done >> lane) & 1u)) {
    float* msg0 = w.c2v + (((size_t)g * c.m + r0) * DMAX) * kLanes + lane;
    const float* tot = w.total + (size_t)g * c.n * kLanes + lane;
    int cl[KC][DMAX];
    float tv[KC][DMAX], mo[KC][DMAX];
#pragma unroll
    for (int q = 0; q < KC; ++q)
#pragma unroll
      for (int s = 0; s < DMAX; ++s) cl[q][s] = r0 + q < c.m ? __ldg(c.row_cols + (size_t)(r0 + q) * DMAX + s) : -1;
#pragma unroll
    for (int q = 0; q < KC; ++q)
#pragma unroll
      for (int s = 0; s < DMAX; ++s) {
        tv[q][s] = cl[q][s] >= 0 ? tot[(size_t)cl[q][s] * kLanes] : 0.f;
        mo[q][s] = !FIRST && cl[q][s] >= 0 ? msg0[(q * DMAX + s) * kLanes] : 0.f;
      }
#pragma unroll
    for (int q = 0; q < KC; ++q) {
      if (r0 + q >= c.m) break;
      float xs[DMAX];
      float min1 = INFINITY, min2 = INFINITY;
      int amin = 0, neg = 0;
#pragma unroll
      for (int s = 0; s < DMAX; ++s) {
        float mag = INFINITY, x = 0.f;
        if (cl[q][s] >= 0) {
          syn ^= tv[q][s] < 0.f ? 1 : 0;
          x = FIRST ? tv[q][s] : __fsub_rn(tv[q][s], mo[q][s]);
          mag = fabsf(x);
          neg ^= x < 0.f ? 1 : 0;
        }
        xs[s] = x;
        // np.argmin: first index of the smallest magnitude (invalid slots are +inf)
        if (s == 0 || mag < min1) {
          if (s != 0) min2 = min1;
          min1 = mag;
          amin = s;
        } else if (mag < min2) {
          min2 = mag;
        }
      }
      const float rs = neg ? -1.f : 1.f;
      float* msg = msg0 + (size_t)q * DMAX * kLanes;
#pragma unroll
      for (int s = 0; s < DMAX; ++s) {
        const float sg = xs[s] < 0.f ? -1.f : 1.f;
        msg[s * kLanes] = cl[q][s] < 0 ? 0.f : __fmul_rn(rs * sg, s == amin ? min2 : min1);
      }
    }
  }
  const uint32_t bal = __ballot_sync(0xffffffffu, syn);
  if (lane == 0 && bal) atomicOr(&block_unsat, bal);
  __syncthreads();
  if (threadIdx.x == 0 && block_unsat)
    atomicOr(w.unsat + ((size_t)par * gridDim.y + g) * kUnsatSlots + blockIdx.x % kUnsatSlots, block_unsat);
}

// Hard decisions of the kept information bits, transposed through shared
// memory: gathered lane-per-codeword (128 B per position), written
// codeword-major with consecutive threads on consecutive bytes.
constexpr int kExtractTile = 256;

__global__ void __launch_bounds__(kWarps * 32) k_ldpc_extract(nrx_ldpc_code c, DecWs w, uint8_t* info,
                                                            uint8_t* success, int n_cw) {
  __shared__ uint8_t bits[kLanes][kExtractTile + 4];
  const int g = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int base = blockIdx.x * kExtractTile;
  const float* tot = w.total + (size_t)g * c.n * kLanes + lane;
  for (int i = warp; i < kExtractTile; i += kWarps)
    if (base + i < c.k_eff) bits[lane][i] = tot[(size_t)__ldg(c.keep_pos + base + i) * kLanes] < 0.f ? 1 : 0;
  __syncthreads();
  for (int idx = threadIdx.x; idx < kLanes * kExtractTile; idx += kWarps * 32) {
    const int l = idx / kExtractTile, i = idx % kExtractTile, cw = g * kLanes + l;
    if (cw < n_cw && base + i < c.k_eff) info[(size_t)cw * c.k_eff + base + i] = bits[l][i];
  }
  const int cw = g * kLanes + lane;
  if (blockIdx.x == 0 && threadIdx.x < 32 && cw < n_cw) success[cw] = static_cast<uint8_t>((w.done[g] >> lane) & 1u);
}

// ---------------------------------------------------------------------------
// staircase encoder kernels
// ---------------------------------------------------------------------------

__global__ void k_enc_place(nrx_ldpc_code c, const uint8_t* info, EncWs w) {
  const int cw = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= c.n) return;
  const int slot = c.info_slot[j];
  w.cw[(size_t)cw * c.n + j] = slot >= 0 ? (info[(size_t)cw * c.k_eff + slot] & 1) : 0;
}

__global__ void k_enc_syn(nrx_ldpc_code c, EncWs w) {
  const int cw = blockIdx.y;
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= c.m) return;
  const uint8_t* bits = w.cw + (size_t)cw * c.n;
  int s = 0;
  for (int k = 0; k < c.dmax; ++k) {
    const int col = c.row_cols[(size_t)r * c.dmax + k];
    if (col >= 0 && c.info_slot[col] != -2) s ^= bits[col];
  }
  w.syn[(size_t)cw * c.m + r] = static_cast<uint8_t>(s);
}

// Accumulator chains: p_i = s_i ^ p_{i-Z}, one thread per chain z < Z.
__global__ void k_enc_chain(nrx_ldpc_code c, EncWs w) {
  const int cw = blockIdx.y;
  const int z = blockIdx.x * blockDim.x + threadIdx.x;
  if (z >= c.chain_step) return;
  const uint8_t* syn = w.syn + (size_t)cw * c.m;
  uint8_t* bits = w.cw + (size_t)cw * c.n;
  uint8_t acc = 0;
  for (int i = z; i < c.m; i += c.chain_step) {
    acc ^= syn[i];
    bits[c.chain_cols[i]] = acc;
  }
}

__global__ void k_enc_tx(nrx_ldpc_code c, EncWs w, uint8_t* tx) {
  const int cw = blockIdx.y;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= c.ntx) return;
  tx[(size_t)cw * c.ntx + e] = w.cw[(size_t)cw * c.n + c.tx_pos[e]];
}

// ---------------------------------------------------------------------------
// coded Monte-Carlo glue
// ---------------------------------------------------------------------------

__device__ inline uint4 philox10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// one Philox block -> 128 bits of one row
__global__ void k_random_bits(uint32_t k0, uint32_t k1, unsigned long long first, int cols, uint8_t* out) {
  const int row = blockIdx.y;
  const int blk = blockIdx.x * blockDim.x + threadIdx.x;   // 128-bit block of the row
  if (blk * 128 >= cols) return;
  const unsigned long long g = first + (unsigned long long)row;
  const uint4 r = philox10(make_uint4((uint32_t)blk, (uint32_t)g, (uint32_t)(g >> 32), 0x5A17u), k0, k1);
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
  uint8_t* o = out + (size_t)row * cols + (size_t)blk * 128;
  const int nb = min(128, cols - blk * 128);
  for (int i = 0; i < nb; ++i) o[i] = (w[i >> 5] >> (i & 31)) & 1u;
}

struct SlotGeo {
  int S, T, U, nsym;      // nsym: data symbols per subcarrier
  int data_t[32];         // the data symbols, ascending
};

__global__ void k_bits_to_labels(SlotGeo g, int ue, int m, const uint8_t* bits, uint8_t* labels) {
  const int n = blockIdx.y;
  const int d = blockIdx.x * blockDim.x + threadIdx.x;     // data RE, subcarrier-major
  const int nd = g.S * g.nsym;
  if (d >= nd) return;
  const int s = d / g.nsym, t = g.data_t[d - s * g.nsym];
  const uint8_t* b = bits + ((size_t)n * nd + d) * m;
  int lab = 0;
  for (int j = 0; j < m; ++j) lab = (lab << 1) | (b[j] & 1);
  labels[(((size_t)n * g.U + ue) * g.S + s) * g.T + t] = static_cast<uint8_t>(lab);
}

__global__ void k_extract_llrs(SlotGeo g, int ue, int m, const float* llr, int W, float clip, float* out) {
  const int n = blockIdx.y;
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  const int nd = g.S * g.nsym;
  if (d >= nd) return;
  const int s = d / g.nsym, t = g.data_t[d - s * g.nsym];
  const float* src = llr + ((((size_t)n * g.U + ue) * g.S + s) * g.T + t) * W;
  float* dst = out + ((size_t)n * nd + d) * m;
  for (int j = 0; j < m; ++j) dst[j] = fminf(fmaxf(src[j], -clip), clip);
}

__global__ void k_mismatches(int cols, const uint8_t* a, const uint8_t* b, unsigned long long* errors) {
  const int row = blockIdx.y;
  int e = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cols; i += gridDim.x * blockDim.x)
    e += (a[(size_t)row * cols + i] & 1) != (b[(size_t)row * cols + i] & 1);
  const int tot = __reduce_add_sync(0xffffffffu, e);
  if ((threadIdx.x & 31) == 0 && tot) atomicAdd(errors + row, (unsigned long long)tot);
}

int slot_geo(const nrx_slot_desc* s, SlotGeo* g) {
  if (!s || s->num_subcarriers < 1 || s->num_symbols < 1 || s->num_symbols > 32 || s->num_ues < 1 ||
      s->num_pilot_symbols < 1 || s->num_pilot_symbols > NRX_MAX_PILOT_SYMBOLS)
    return NRX_ERR_INVALID;
  g->S = s->num_subcarriers;
  g->T = s->num_symbols;
  g->U = s->num_ues;
  bool pilot[32] = {};
  for (int k = 0; k < s->num_pilot_symbols; ++k) {
    if (s->pilot_symbols[k] < 0 || s->pilot_symbols[k] >= g->T) return NRX_ERR_INVALID;
    pilot[s->pilot_symbols[k]] = true;
  }
  g->nsym = 0;
  for (int t = 0; t < g->T; ++t)
    if (!pilot[t]) g->data_t[g->nsym++] = t;
  return g->nsym > 0 ? NRX_OK : NRX_ERR_INVALID;
}

int launch_status() {
  const cudaError_t e = cudaPeekAtLastError();
  if (e == cudaErrorNoKernelImageForDevice || e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
    return NRX_ERR_NO_DEVICE;
  return e == cudaSuccess ? NRX_OK : NRX_ERR_CUDA;
}

template <typename T>
int upload(T** dst, const std::vector<T>& v) {
  *dst = nullptr;
  if (v.empty()) return NRX_OK;
  if (cudaMalloc(reinterpret_cast<void**>(dst), v.size() * sizeof(T)) != cudaSuccess) return NRX_ERR_CUDA;
  return cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) == cudaSuccess ? NRX_OK
                                                                                              : NRX_ERR_CUDA;
}

}  // namespace nrx_ldpc

using namespace nrx_ldpc;

extern "C" int nrx_ldpc_create(const nrx_ldpc_desc* d, nrx_ldpc_code** out) {
  if (!d || !out) return NRX_ERR_INVALID;
  *out = nullptr;
  if (d->n < 2 || d->m < 1 || d->k < 1 || d->k >= d->n || d->dmax < 1 || d->cdeg < 1) return NRX_ERR_INVALID;
  if (d->cdeg > NRX_LDPC_MAX_COL_DEG || d->dmax > NRX_LDPC_MAX_ROW_DEG || (int64_t)d->m * d->dmax >= (int64_t)1 << 31)
    return NRX_ERR_UNSUPPORTED;   // edge records hold the message index in an int32
  if (!d->row_cols || !d->col_rows || !d->col_slots || !d->info_positions) return NRX_ERR_INVALID;
  if (d->n_punctured < 0 || d->n_shortened < 0 || (d->n_punctured && !d->punctured) ||
      (d->n_shortened && !d->shortened))
    return NRX_ERR_INVALID;
  const int n = d->n, m = d->m, k = d->k;
  for (size_t i = 0; i < (size_t)m * d->dmax; ++i)
    if (d->row_cols[i] < -1 || d->row_cols[i] >= n) return NRX_ERR_INVALID;
  for (size_t i = 0; i < (size_t)n * d->cdeg; ++i) {
    if (d->col_rows[i] < -1 || d->col_rows[i] >= m) return NRX_ERR_INVALID;
    if (d->col_rows[i] >= 0 && (d->col_slots[i] < 0 || d->col_slots[i] >= d->dmax)) return NRX_ERR_INVALID;
  }
  std::vector<int32_t> info_slot(n, -2), chan_src(n, 0);
  std::vector<char> skip(n, 0), is_short(n, 0);
  for (int i = 0; i < d->n_punctured; ++i) {
    const int p = d->punctured[i];
    if (p < 0 || p >= n) return NRX_ERR_INVALID;
    skip[p] = 1;
  }
  for (int i = 0; i < d->n_shortened; ++i) {
    const int p = d->shortened[i];
    if (p < 0 || p >= n) return NRX_ERR_INVALID;
    skip[p] = 1;
    is_short[p] = 1;
  }
  std::vector<int32_t> keep_pos;
  for (int i = 0; i < k; ++i) {
    const int p = d->info_positions[i];
    if (p < 0 || p >= n || (i && p <= d->info_positions[i - 1])) return NRX_ERR_INVALID;
    if (is_short[p]) {
      info_slot[p] = -1;
    } else {
      info_slot[p] = static_cast<int32_t>(keep_pos.size());
      keep_pos.push_back(p);
    }
  }
  std::vector<int32_t> tx_pos;
  for (int j = 0; j < n; ++j) {
    if (!skip[j]) {
      chan_src[j] = static_cast<int32_t>(tx_pos.size());
      tx_pos.push_back(j);
    } else {
      chan_src[j] = is_short[j] ? -2 : -1;   // shortened: known zero; punctured: erased
    }
  }
  if (keep_pos.empty() || tx_pos.empty()) return NRX_ERR_INVALID;
  if (d->chain_cols) {
    if (d->chain_step < 1 || d->chain_step > m) return NRX_ERR_INVALID;
    for (int i = 0; i < m; ++i)
      if (d->chain_cols[i] < 0 || d->chain_cols[i] >= n || info_slot[d->chain_cols[i]] != -2) return NRX_ERR_INVALID;
  }
  nrx_ldpc_code* c = new nrx_ldpc_code{};
  c->n = n;
  c->m = m;
  c->k = k;
  c->dmax = d->dmax;
  c->cdeg = d->cdeg;
  c->k_eff = static_cast<int>(keep_pos.size());
  c->ntx = static_cast<int>(tx_pos.size());
  c->has_chain = d->chain_cols != nullptr;
  c->chain_step = d->chain_step;
  int rc = NRX_OK;
  rc = rc ? rc : upload(&c->row_cols, std::vector<int32_t>(d->row_cols, d->row_cols + (size_t)m * d->dmax));
  rc = rc ? rc : upload(&c->col_rows, std::vector<int32_t>(d->col_rows, d->col_rows + (size_t)n * d->cdeg));
  rc = rc ? rc : upload(&c->col_slots, std::vector<int32_t>(d->col_slots, d->col_slots + (size_t)n * d->cdeg));
  rc = rc ? rc : upload(&c->chan_src, chan_src);
  rc = rc ? rc : upload(&c->keep_pos, keep_pos);
  rc = rc ? rc : upload(&c->tx_pos, tx_pos);
  std::vector<int32_t> skip_pos;
  for (int j = 0; j < n; ++j)
    if (skip[j]) skip_pos.push_back(j);
  c->n_skip = static_cast<int>(skip_pos.size());
  rc = rc ? rc : upload(&c->skip_pos, skip_pos);
  rc = rc ? rc : upload(&c->info_slot, info_slot);
  if (!rc && d->chain_cols) rc = upload(&c->chain_cols, std::vector<int32_t>(d->chain_cols, d->chain_cols + m));
  if (!rc) {
    std::vector<int4> edges(n, make_int4(-1, -1, -1, -1));
    for (int j = 0; j < n; ++j) {
      int e[3] = {-1, -1, -1};
      for (int t = 0; t < d->cdeg && t < 3; ++t) {
        const int r = d->col_rows[(size_t)j * d->cdeg + t];
        if (r < 0) break;
        e[t] = r * d->dmax + d->col_slots[(size_t)j * d->cdeg + t];
      }
      edges[j] = make_int4(e[0], e[1], e[2], -1);
    }
    rc = upload(&c->edges, edges);
  }
  if (rc) {
    nrx_ldpc_destroy(c);
    return rc == NRX_ERR_CUDA && cudaGetLastError() == cudaErrorNoDevice ? NRX_ERR_NO_DEVICE : rc;
  }
  *out = c;
  return NRX_OK;
}

extern "C" void nrx_ldpc_destroy(nrx_ldpc_code* c) {
  if (!c) return;
  int32_t* ptrs[] = {c->row_cols, c->col_rows, c->col_slots, c->chan_src, c->keep_pos, c->tx_pos, c->skip_pos,
                     c->info_slot, c->chain_cols};
  for (int32_t* p : ptrs)
    if (p) cudaFree(p);
  if (c->edges) cudaFree(c->edges);
  delete c;
}

extern "C" int nrx_ldpc_dims(const nrx_ldpc_code* c, int32_t* out4) {
  if (!c || !out4) return NRX_ERR_INVALID;
  out4[0] = c->n;
  out4[1] = c->k_eff;
  out4[2] = c->ntx;
  out4[3] = c->m;
  return NRX_OK;
}

extern "C" size_t nrx_ldpc_workspace_bytes(const nrx_ldpc_code* c, int n_cw) {
  if (!c || n_cw < 1) return 0;
  size_t a = 0, b = 0;
  dec_layout(*c, n_cw, nullptr, &a);
  enc_layout(*c, n_cw, nullptr, &b);
  return a > b ? a : b;
}

extern "C" int nrx_ldpc_decode(const nrx_ldpc_code* c, int n_cw, const float* llr, int iterations,
                               uint8_t* info_out, uint8_t* success, void* ws, size_t ws_bytes, void* stream) {
  if (!c || n_cw < 0 || iterations < 0 || !llr || !info_out || !success) return NRX_ERR_INVALID;
  if (n_cw == 0) return NRX_OK;
  const int G = (n_cw + kLanes - 1) / kLanes;
  if (G > 65535) return NRX_ERR_UNSUPPORTED;
  size_t need = 0;
  dec_layout(*c, n_cw, nullptr, &need);
  if (!ws || ws_bytes < need) return NRX_ERR_WORKSPACE;
  const DecWs w = dec_layout(*c, n_cw, static_cast<uint8_t*>(ws), nullptr);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int vb = (c->n + kWarps * kVarsPerWarp - 1) / (kWarps * kVarsPerWarp);
  // fixed row widths 5 / 6 (the IRA codes and the reference's codes): two checks per warp
  // (2 % faster than one at the C2 codeword; four is 5 % slower: 78 registers)
  const int kc = c->dmax == 5 || c->dmax == 6 ? 2 : 1;
  auto check_fn = [&](bool first) {
    if (c->dmax == 5) return first ? k_ldpc_check_rows<5, true, 2> : k_ldpc_check_rows<5, false, 2>;
    if (c->dmax == 6) return first ? k_ldpc_check_rows<6, true, 2> : k_ldpc_check_rows<6, false, 2>;
    return first ? (c->dmax == 7 ? k_ldpc_check<7, true> : c->dmax == 8 ? k_ldpc_check<8, true> : k_ldpc_check<0, true>)
                 : (c->dmax == 7 ? k_ldpc_check<7, false> : c->dmax == 8 ? k_ldpc_check<8, false> : k_ldpc_check<0, false>);
  };
  const int cb = (c->m + kWarps * kc - 1) / (kWarps * kc);
  k_ldpc_init_tx<<<dim3((c->ntx + kInitTile - 1) / kInitTile, G), kWarps * 32, 0, st>>>(*c, llr, n_cw, w);
  k_ldpc_init_state<<<dim3(std::max(1, std::min(256, (c->n_skip + kWarps - 1) / kWarps)), G), kWarps * 32, 0, st>>>(
      *c, n_cw, w);
  for (int it = 0; it < iterations; ++it) {
    (it == 0 ? k_ldpc_var<true> : k_ldpc_var<false>)<<<dim3(vb, G), kWarps * 32, 0, st>>>(*c, w, it & 1);
    check_fn(it == 0)<<<dim3(cb, G), kWarps * 32, 0, st>>>(*c, w, it & 1);
  }
  // codewords that never satisfied every check: totals of the final messages
  (iterations == 0 ? k_ldpc_var<true> : k_ldpc_var<false>)<<<dim3(vb, G), kWarps * 32, 0, st>>>(*c, w,
                                                                                               iterations & 1);
  k_ldpc_extract<<<dim3((c->k_eff + kExtractTile - 1) / kExtractTile, G), kWarps * 32, 0, st>>>(
      *c, w, info_out, success, n_cw);
  return launch_status();
}

extern "C" int nrx_ldpc_encode(const nrx_ldpc_code* c, int n_cw, const uint8_t* info, uint8_t* tx, void* ws,
                               size_t ws_bytes, void* stream) {
  if (!c || n_cw < 0 || !info || !tx) return NRX_ERR_INVALID;
  if (!c->has_chain) return NRX_ERR_UNSUPPORTED;
  if (n_cw == 0) return NRX_OK;
  if (n_cw > 65535) return NRX_ERR_UNSUPPORTED;
  size_t need = 0;
  enc_layout(*c, n_cw, nullptr, &need);
  if (!ws || ws_bytes < need) return NRX_ERR_WORKSPACE;
  const EncWs w = enc_layout(*c, n_cw, static_cast<uint8_t*>(ws), nullptr);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_enc_place<<<dim3((c->n + kThreads - 1) / kThreads, n_cw), kThreads, 0, st>>>(*c, info, w);
  k_enc_syn<<<dim3((c->m + kThreads - 1) / kThreads, n_cw), kThreads, 0, st>>>(*c, w);
  k_enc_chain<<<dim3((c->chain_step + kThreads - 1) / kThreads, n_cw), kThreads, 0, st>>>(*c, w);
  k_enc_tx<<<dim3((c->ntx + kThreads - 1) / kThreads, n_cw), kThreads, 0, st>>>(*c, w, tx);
  return launch_status();
}

extern "C" int nrx_random_bits(uint64_t seed, uint64_t first_row, int rows, int cols, uint8_t* out, void* stream) {
  if (rows < 0 || cols < 0 || (!out && rows && cols)) return NRX_ERR_INVALID;
  if (!rows || !cols) return NRX_OK;
  if (rows > 65535) return NRX_ERR_UNSUPPORTED;
  const int blocks = (cols + 127) / 128;
  k_random_bits<<<dim3((blocks + 127) / 128, rows), 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      (uint32_t)seed, (uint32_t)(seed >> 32), first_row, cols, out);
  return launch_status();
}

extern "C" int nrx_bits_to_labels(const nrx_slot_desc* slot, int n_slots, int ue, int mod_order, const uint8_t* bits,
                                  uint8_t* labels, void* stream) {
  SlotGeo g;
  const int rc = slot_geo(slot, &g);
  if (rc) return rc;
  if (n_slots < 0 || ue < 0 || ue >= g.U || mod_order < 1 || mod_order > 8 || !bits || !labels) return NRX_ERR_INVALID;
  if (!n_slots) return NRX_OK;
  if (n_slots > 65535) return NRX_ERR_UNSUPPORTED;
  const int nd = g.S * g.nsym;
  k_bits_to_labels<<<dim3((nd + 255) / 256, n_slots), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      g, ue, mod_order, bits, labels);
  return launch_status();
}

extern "C" int nrx_extract_llrs(const nrx_slot_desc* slot, int n_slots, int ue, int mod_order, const float* llr,
                                int llr_width, float clip, float* out, void* stream) {
  SlotGeo g;
  const int rc = slot_geo(slot, &g);
  if (rc) return rc;
  if (n_slots < 0 || ue < 0 || ue >= g.U || mod_order < 1 || mod_order > llr_width || llr_width > 8 || !llr ||
      !out || !(clip > 0.f))
    return NRX_ERR_INVALID;
  if (!n_slots) return NRX_OK;
  if (n_slots > 65535) return NRX_ERR_UNSUPPORTED;
  const int nd = g.S * g.nsym;
  k_extract_llrs<<<dim3((nd + 255) / 256, n_slots), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      g, ue, mod_order, llr, llr_width, clip, out);
  return launch_status();
}

extern "C" int nrx_count_mismatches(int rows, int cols, const uint8_t* a, const uint8_t* b, unsigned long long* errors,
                                    void* stream) {
  if (rows < 0 || cols < 0 || ((!a || !b || !errors) && rows && cols)) return NRX_ERR_INVALID;
  if (!rows || !cols) return NRX_OK;
  if (rows > 65535) return NRX_ERR_UNSUPPORTED;
  const int blocks = min(64, (cols + 255) / 256);
  k_mismatches<<<dim3(blocks, rows), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(cols, a, b, errors);
  return launch_status();
}
