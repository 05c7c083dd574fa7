/*
 * nrx_slotgen.h — C ABI of the GPU synthetic uplink-slot generator and the
 * uncoded bit-error counter (the step immediately
 * upstream of the receiver, and its BER read-out).
 *
 * Entry point -> reference interface it replaces:
 *   nrx_synth_slots      one uncoded Monte-Carlo slot batch, i.e. per slot
 *                        generate_pilots            slot.py:130-139
 *                        Constellation.map_bits     constellation.py:44-50
 *                        (data REs subcarrier-major, slot.py:106-109,
 *                         LDPC bypassed: the labels are iid, SURVEY finding 5)
 *                        beamform                   slot.py:231-233
 *                        TdlChannelSource.sample    channel.py:178-190
 *                          -> sample_tdl            channel.py:127-150
 *                          -> cir_to_freq           channel.py:113-124
 *                        apply_channel              channel.py:153-167
 *                        ChannelRealization.effective channel.py:101-104
 *   nrx_count_bit_errors hard decisions (LLR > 0 -> bit 1, test_slot.py:141)
 *                        against the transmitted labels on the data REs;
 *                        the bit/block counters of MetricsRecord
 *                        (evaluation.py:44-72) for the uncoded receiver.
 *
 * Randomness.  Each variate is either supplied by the caller (the
 * reference-stream mode: draw them on the host with numpy exactly as the
 * reference does, and the generated slot equals the reference's to float64
 * rounding) or drawn on the device from a counter-based Philox4x32-10
 * stream keyed by (seed, global slot index), so a slot's content never
 * depends on the batch it was generated in or on the rank that made it.
 *
 * Arithmetic: float64 (like the reference) whenever channel or noise
 * variates are supplied or a complex128 output is requested; otherwise
 * (device variates, possibly caller labels / pilots, complex64 outputs) the
 * slot is synthesised in float32 from the same variates.
 *
 * Like nrx_forward: no allocation, no host synchronisation; work is
 * enqueued on `stream` (void* = cudaStream_t) and an nrx_status returned.
 */
#ifndef NRX_SLOTGEN_H_
#define NRX_SLOTGEN_H_

#include <stddef.h>
#include <stdint.h>

#include "nrx_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define NRX_SG_MAX_UES 4
#define NRX_SG_MAX_TAPS 24
#define NRX_SG_MAX_UE_ANT 4
#define NRX_SG_MAX_RX_ANT 8
/* QAM point table: orders 2, 4, 6, 8 concatenated, complex (re, im). */
#define NRX_SG_QAM_POINTS (4 + 16 + 64 + 256)

/* TdlProfile (channel.py:29-50): ascending delays, linear powers summing
 * to 1, maximum Doppler. */
typedef struct nrx_tdl_profile {
  int32_t num_taps;
  double delays_s[NRX_SG_MAX_TAPS];
  double powers[NRX_SG_MAX_TAPS];
  double doppler_hz;
} nrx_tdl_profile;

/* Antennas, numerology, beams and the per-UE channel profiles
 * (SlotConfig slot.py:47-71, TdlChannelSource channel.py:170-176). */
typedef struct nrx_channel_desc {
  int32_t bs_antennas;              /* B                                  */
  int32_t ue_antennas;              /* N_u                                */
  int32_t num_sinusoids;            /* NUM_SINUSOIDS = 32 (channel.py:22) */
  double subcarrier_spacing_hz;
  double cp_fraction;
  double beams[NRX_SG_MAX_UES][NRX_SG_MAX_UE_ANT][2];  /* unit-norm, complex */
  nrx_tdl_profile profiles[NRX_SG_MAX_UES];            /* UE u -> profiles[u] */
} nrx_channel_desc;

/* Caller-supplied variates (device pointers; any may be NULL, which draws
 * that group on the device).  L = max taps over the UEs, NS = sinusoids.
 *   angles, phases  (N, U, B, N_u, L, NS) float64 in [0, 2 pi): the two
 *                   rng.uniform draws of sample_tdl (channel.py:140-141)
 *   labels          (N, U, S, T) uint8: QAM label index (big-endian bit
 *                   label, constellation.py:26-29) of each data RE
 *   noise           (N, S, T, B) complex128 standard-normal pairs
 *                   (re = first standard_normal draw, im = second,
 *                   channel.py:164-165); scaled by sqrt(n0/2) on device
 *   pilots          (N, U, F, K) complex128 pilot values at UE u's comb
 *                   subcarrier u%comb + f*comb and pilot symbol k        */
typedef struct nrx_slot_variates {
  const double* angles;
  const double* phases;
  const uint8_t* labels;
  const double* noise;
  const double* pilots;
} nrx_slot_variates;

/* 0 when the slot/channel description is valid; NRX_ERR_INVALID for what
 * the reference rejects (e.g. a tap beyond the cyclic prefix,
 * channel.py:135-138; more UEs than the comb), NRX_ERR_UNSUPPORTED beyond
 * the limits above. */
int nrx_synth_validate(const nrx_slot_desc* slot, const nrx_channel_desc* chan);

size_t nrx_synth_workspace_bytes(const nrx_slot_desc* slot, const nrx_channel_desc* chan, int n_slots);

/*
 * Generate n_slots slots (global indices first_slot .. first_slot+n_slots-1).
 *   mod_order  (n_slots*U) int32 device: modulation order per (slot, UE),
 *              one of 2, 4, 6, 8
 *   n0         (n_slots) float64 device: noise power (no noise when <= 0,
 *              exactly like apply_channel)
 *   qam_points host pointer to NRX_SG_QAM_POINTS complex float64 points or
 *              NULL for the built-in table (pass build_constellation(m)
 *              .points for bit-compatibility with the reference)
 * Outputs (device; NULL skips an optional one):
 *   y          (n_slots, S, T, B) complex (y_c128: double2, else float2)
 *   pilots     (n_slots, U, F, K) complex, the nrx_forward pilot layout
 *              (pilots_c128 selects double2); entries past a UE's comb = 0
 *   labels     (n_slots, U, S, T) uint8 label index, 0 off the data REs
 *   h_eff      optional (n_slots, U, S, T, B) effective channel
 *              (h_eff_c128 selects double2)
 */
int nrx_synth_slots(const nrx_slot_desc* slot, const nrx_channel_desc* chan, int n_slots,
                    uint64_t seed, uint64_t first_slot,
                    const int32_t* mod_order, const double* n0,
                    const nrx_slot_variates* variates, const double* qam_points,
                    void* y, int y_c128, void* pilots, int pilots_c128,
                    uint8_t* labels, void* h_eff, int h_eff_c128,
                    void* workspace, size_t workspace_bytes, void* stream);

/*
 * Uncoded bit errors per (slot, UE), ADDED to bit_errors (n_slots*U,
 * device uint64): for every data RE and label position j < m,
 * (llr[j] > 0) != bit j of the label.  llr is nrx_forward's llr_out
 * (n_slots, U, S, T, llr_width) float32.
 */
int nrx_count_bit_errors(const nrx_slot_desc* slot, int n_slots, const float* llr, int llr_width,
                         const uint8_t* labels, const int32_t* mod_order,
                         unsigned long long* bit_errors, void* stream);

/* Philox4x32-10 block (ctr[4], key[2] -> out[4]); the device generator's
 * bijection, exported for known-answer tests. */
void nrx_philox4x32_10(const uint32_t* ctr, const uint32_t* key, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif /* NRX_SLOTGEN_H_ */
