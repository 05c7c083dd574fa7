/*
 * nrx_b200.h — C ABI of the B200-native (sm_100a) neural-receiver forward pass.
 *
 * Drop-in boundary for the reference receiver path
 *   nrxsim.nrx.nrx_forward   /root/reference/pkg/src/nrxsim/nrx.py:345-385
 * The reference is pure Python/numpy and has no native FFI of its own; this
 * header is the C surface a ctypes/cffi binding of that Python API binds
 * (see INTEGRATION.md).  Plain pointers and sizes only: no torch or CUDA
 * types appear in the signatures (streams are passed as void*).
 *
 * Entry point -> reference interface it replaces:
 *   nrx_forward          nrx_forward (nrx.py:345-385) minus the numpy-only
 *                        host steps (MCS validation, squeeze, per-UE slicing)
 *                        which the Python wrapper keeps;
 *                        internally: ls_features nrx.py:205-213 +
 *                        classical.ls_estimate classical.py:64-78,
 *                        assemble_features nrx.py:184-202,
 *                        nrx_forward_graph nrx.py:302-342 (training=False),
 *                        readout_llrs/readout_chest nrx.py:266-281,
 *                        planar chest decode nrx.py:382-384.
 *   nrx_weight_count/_name  expected_shapes nrx.py:92-120 (canonical order
 *                        of the tensors nrx_pack_weights consumes).
 *   nrx_pack_weights     the weight dict consumed by nrx_forward_graph
 *                        (init_weights nrx.py:123-133 / checkpoint_load
 *                        nrx.py:420-471 produce it); host-side repack into
 *                        the kernels' device layout.
 *   nrx_validate         NrxConfig.__post_init__ nrx.py:53-67 plus the
 *                        limits of this implementation.
 *
 * Semantics: nrx_forward never allocates, never synchronises the host and
 * never throws; it enqueues kernels on `stream` and returns an nrx_status.
 * All device pointers must stay valid until the stream reaches the end of
 * the enqueued work.  It is reentrant: concurrent calls must use distinct
 * workspaces (and usually distinct streams); the packed weights are
 * read-only and may be shared.
 */
#ifndef NRX_B200_H_
#define NRX_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NRX_ABI_VERSION 1
#define NRX_MAX_PILOT_SYMBOLS 16
#define NRX_MAX_IO 4
/* Byte offset in the workspace of a uint32 the tensor-core modes set to
 * nonzero when a readout produced a non-finite LLR / channel value (fp16
 * operand planes overflow above 65504); nrx_forward zeroes it first.  The
 * drop-in re-runs such a call on the fp32 SIMT kernels. */
#define NRX_WS_FLAG_OFFSET 0

typedef enum nrx_status {
  NRX_OK = 0,
  NRX_ERR_INVALID = 1,      /* malformed descriptor / argument            */
  NRX_ERR_UNSUPPORTED = 2,  /* valid for the reference, beyond our limits */
  NRX_ERR_WORKSPACE = 3,    /* workspace too small                        */
  NRX_ERR_CUDA = 4,         /* a CUDA launch/driver call failed           */
  NRX_ERR_DEPTH = 5,        /* num_iterations outside [1, N_it]           */
  NRX_ERR_NO_DEVICE = 6     /* no sm_100 device / kernel image            */
} nrx_status;

typedef enum nrx_variant { NRX_SINGLE = 0, NRX_MASKING = 1, NRX_VAR_IO = 2 } nrx_variant;

typedef enum nrx_precision {
  NRX_FP32 = 0,  /* fp32 SIMT arithmetic, parity mode (<=1e-5 rel. of ref)   */
  NRX_BF16 = 1,  /* bf16 operands on tcgen05 tensor cores, fp32 accumulate,
                    fp32 residual state stream                               */
  NRX_FP16 = 2,  /* fp16 operands on tcgen05, fp32 accumulate, fp16 state
                    (8x finer operand rounding than bf16, no fp32 stream)    */
  NRX_FP32X3 = 3 /* fp32-grade on tcgen05: every operand split into fp16
                    hi + lo planes (a = hi + lo 2^-11, 22 significant bits),
                    each product as lo*W_hi + hi*W_hi + hi*W_lo (three MMAs,
                    one fp32 TMEM accumulator via scale-input-d), CTA-pair
                    (cta_group::2) convolutions; parity gate <=1e-5 rel.    */
} nrx_precision;

/* NrxConfig (nrx.py:37-89). io_orders: var_io -> io_modulations (sorted);
 * single/masking -> n_io = 1, io_orders[0] = m_max. */
typedef struct nrx_model_desc {
  int32_t d_s;
  int32_t hidden;            /* MLP hidden width (hidden_width or d_s) */
  int32_t num_iterations;    /* N_it, weights shared across iterations */
  int32_t kernel_size;       /* odd */
  int32_t variant;           /* nrx_variant */
  int32_t m_max;
  int32_t n_io;
  int32_t io_orders[NRX_MAX_IO];
  int32_t num_rx_ant;        /* B */
  int32_t include_noise_plane;
  int32_t include_freq_encoding;
} nrx_model_desc;

/* SlotConfig geometry (slot.py:47-116). bs_antennas == model num_rx_ant. */
typedef struct nrx_slot_desc {
  int32_t num_subcarriers;   /* S */
  int32_t num_symbols;       /* T */
  int32_t num_ues;           /* U, UE u uses comb offset u % comb_size */
  int32_t comb_size;
  int32_t num_pilot_symbols; /* K */
  int32_t pilot_symbols[NRX_MAX_PILOT_SYMBOLS];
} nrx_slot_desc;

int nrx_abi_version(void);
const char* nrx_status_string(int status);

/* 0 when (model, slot) is valid and supported. */
int nrx_validate(const nrx_model_desc* model, const nrx_slot_desc* slot);

/* Weights: the tensors of expected_shapes(config) in the canonical order
 * below, each float32 C-contiguous in the reference shape
 * (conv (k,k,Cin,Cout), dense (in,out), bias (out,)):
 *   for each io set i < n_io (tag = ".m{io_orders[i]}" for var_io, "" else):
 *     state_init{tag}.conv0.w, .conv0.b, .conv1.w, .conv1.b,
 *     readout_llr{tag}.fc0.w, .fc0.b, .fc1.w, .fc1.b
 *   iteration.msg.fc0.w, .fc0.b, .fc1.w, .fc1.b,
 *   iteration.update.conv0.w, .conv0.b, .conv1.w, .conv1.b,
 *   readout_chest.fc0.w, .fc0.b, .fc1.w, .fc1.b                         */
int nrx_weight_count(const nrx_model_desc* model);
/* Writes the i-th canonical name (NUL-terminated) into buf; returns its
 * length or -1. */
int nrx_weight_name(const nrx_model_desc* model, int i, char* buf, size_t buf_len);
/* Expected element count of the i-th tensor, or -1. */
int64_t nrx_weight_numel(const nrx_model_desc* model, int i);

size_t nrx_packed_weight_bytes(const nrx_model_desc* model, int precision);
/* Host-side repack (no GPU needed): tensors[i] -> packed_host (size
 * nrx_packed_weight_bytes).  The caller copies packed_host to the device. */
int nrx_pack_weights(const nrx_model_desc* model, int precision,
                     const float* const* tensors, int n_tensors, void* packed_host);

size_t nrx_workspace_bytes(const nrx_model_desc* model, const nrx_slot_desc* slot,
                           int n_slots, int precision);

/*
 * One batched forward pass over n_slots independent slots (device pointers):
 *   y        (n_slots, S, T, B) complex: float2 (y_c128=0) or double2 (=1)
 *   pilots   (n_pilot_sets, U, F, K) complex values of each UE's pilots at
 *            its comb subcarriers f (subcarrier u%comb + f*comb, F =
 *            ceil(S/comb), entries past the UE's comb are ignored) and
 *            pilot symbols k; float2 or double2 (pilots_c128);
 *            n_pilot_sets is 1 (shared book) or n_slots.
 *   noise_feat (n_slots) float: log10(max(float32(n0), 1e-30)) as float32
 *            (nrx.py:199-201); ignored without the noise plane.
 *   mod_order  (n_slots*U) int32 modulation order per slab (var_io selects
 *            the IO weight set by it; must be one of io_orders).
 *   llr_out  (n_slots, U, S, T, llr_width) float32; slab (n,u) writes its
 *            llr_width(m) columns (m_max, or m for var_io) then zeros.
 *   chest_out (n_slots, U, S, T, B) complex64 (float2): readout channel b
 *            is the real part and B+b the imaginary part (planar decode).
 */
int nrx_forward(const nrx_model_desc* model, const nrx_slot_desc* slot, int n_slots,
                int precision, int num_iterations,
                const void* y, int y_c128,
                const void* pilots, int pilots_c128, int n_pilot_sets,
                const float* noise_feat, const int32_t* mod_order,
                const void* packed_weights,
                float* llr_out, int llr_width, void* chest_out,
                void* workspace, size_t workspace_bytes, void* stream);

/* Diagnostics (used by the parity tests).
 * nrx_buffer_geometry writes {rows_slab, Tp, Cf, Cs, Ch, Ca, cw, tiles} of
 * the internal chunk-planar activation layout (see csrc/nrx_internal.h). */
int nrx_buffer_geometry(const nrx_model_desc* model, const nrx_slot_desc* slot, int precision,
                        int32_t* out8);
/* Runs only the LS + feature-assembly kernel; feats_out receives the
 * (n_slots*U, Cf/cw, rows_slab, cw) chunk-planar feature tensor. */
int nrx_ls_features(const nrx_model_desc* model, const nrx_slot_desc* slot, int n_slots,
                    int precision, const void* y, int y_c128, const void* pilots,
                    int pilots_c128, int n_pilot_sets, const float* noise_feat,
                    void* feats_out, void* stream);

/* Optional per-launch device timing (bench.py's roofline measurement).
 * While enabled, nrx_forward brackets every launch whose kernel id bit is
 * set in kernel_mask with CUDA events recorded on the launch stream.
 * Kernel ids: 0 ls_feat, 1 conv state_init.conv0, 2 conv state_init.conv1,
 * 3 msg_agg, 4 conv iteration.update.conv0, 5 conv iteration.update.conv1,
 * 6 readout.  nrx_profile_collect waits for the recorded events, writes up
 * to cap (kernel id, milliseconds) records, clears them and returns the
 * count.  Process-wide; not meant for concurrent use. */
int nrx_profile_enable(uint32_t kernel_mask, int max_records);
int nrx_profile_collect(int32_t* kernel_ids, float* ms, int cap);
void nrx_profile_disable(void);
const char* nrx_kernel_name(int kernel_id);

/* Number of kernel launches one nrx_forward call enqueues. */
int nrx_forward_launch_count(const nrx_model_desc* model, const nrx_slot_desc* slot, int precision,
                             int num_iterations);

#ifdef __cplusplus
}
#endif
#endif /* NRX_B200_H_ */
