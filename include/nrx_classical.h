/*
 * nrx_classical.h — C ABI of the classical baseline receiver on the GPU
 * (SURVEY.md §8(f) row 4): the "ls_lmmse" receiver of the reference's
 * ReceiverBank (evaluation.py:130-135), the comparison curve of every TBLER
 * sweep.
 *
 * Entry point -> reference interface it replaces (/root/reference/pkg/src/nrxsim):
 *   nrx_ls_lmmse   ls_estimate            classical.py:40-78  (comb LS, linear
 *                                          interpolation in frequency with edge
 *                                          extrapolation, nearest pilot symbol)
 *                  lmmse_equalize         classical.py:113-143 (per-RE LMMSE,
 *                                          unbiased outputs, noise variances)
 *                  app_demap (exact)      classical.py:150-174 (log-sum-exp
 *                                          over the Gray constellation)
 *                  np.clip(llr, -clip, clip)  evaluation.py:79-84
 * float64 arithmetic like the reference; LLRs written as float32.
 */
#ifndef NRX_CLASSICAL_H_
#define NRX_CLASSICAL_H_

#include <stddef.h>
#include <stdint.h>

#include "nrx_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define NRX_CL_MAX_UES 4
#define NRX_CL_MAX_RX_ANT 8

/*
 * y          (n_slots, S, T, B) complex (y_c128: double2, else float2)
 * pilots     (n_pilot_sets, U, F, K) complex comb pilot values (the
 *            nrx_forward layout; pilots_c128 selects double2), n_pilot_sets
 *            1 or n_slots
 * n0         (n_slots) float64 noise power
 * mod_order  (n_slots * U) int32, one of 2, 4, 6, 8
 * qam_points host pointer to NRX_SG_QAM_POINTS complex float64 points
 *            (orders 2, 4, 6, 8 concatenated; nrx_slotgen.h) or NULL for the
 *            built-in Gray table
 * llr_out    (n_slots, U, S, T, llr_width) float32: per RE and UE the m
 *            exact APP LLRs (logit convention), clipped to +-clip, zeros
 *            beyond m
 */
int nrx_ls_lmmse(const nrx_slot_desc* slot, int bs_antennas, int n_slots, const void* y, int y_c128,
                 const void* pilots, int pilots_c128, int n_pilot_sets, const double* n0,
                 const int32_t* mod_order, const double* qam_points, float clip, float* llr_out, int llr_width,
                 void* stream);

/*
 * K-Best detection with max-log LLRs on a given channel (the reference's
 * "perfect_kbest" receiver with the true effective channel:
 * classical.kbest_detect classical.py:195-261 via evaluation._kbest_grids
 * :87-111).  Breadth-first over the streams U-1 .. 0 after a QR of the
 * B x U channel, keeping the k best partial paths (k <= NRX_CL_MAX_K);
 * LLR = (min metric with bit 0 - min metric with bit 1) / max(n0, 1e-12),
 * +-clip when a hypothesis is missing from the list.  Data REs only (the
 * other REs of llr_out are written as zeros, like the reference's grids).
 *   h   (n_slots, U, S, T, B) complex channel (h_c128 selects double2)
 *   reference_pairing  1: reproduce the reference exactly — its interference
 *       term pairs R[level, level+1:] (ascending streams) with the decided
 *       symbols in decision order (descending streams), classical.py:220-221,
 *       which is the true interference only for U <= 2; 0: the correct
 *       pairing R[level, j] * x_j (differs from the reference for U >= 3).
 */
#define NRX_CL_MAX_K 32
int nrx_kbest(const nrx_slot_desc* slot, int bs_antennas, int n_slots, const void* y, int y_c128, const void* h,
              int h_c128, const double* n0, const int32_t* mod_order, const double* qam_points, int k,
              int reference_pairing, float clip, float* llr_out, int llr_width, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NRX_CLASSICAL_H_ */
