/*
 * nrx_ldpc.h — C ABI of the GPU LDPC layer downstream of the receiver
 * (SURVEY.md §8(f) row 2): flooding min-sum decoding of the NRX LLRs and,
 * for the scalable staircase (IRA) mother codes, encoding.
 *
 * Entry point -> reference interface it replaces (/root/reference/pkg/src/nrxsim):
 *   nrx_ldpc_create      LdpcCode (ldpc.py:28-75): the parity-check structure
 *                        (row_cols / col_rows / col_slots), the information
 *                        positions and the rate-matching pattern (punctured,
 *                        shortened, ldpc.py:303-330), uploaded once.
 *   nrx_ldpc_decode      LdpcCode.decode (ldpc.py:99-178): logit LLRs of the
 *                        transmitted bits -> information bits + success
 *                        flags; bit-identical to the reference (same float32
 *                        operation order, same early exit on parity).
 *   nrx_ldpc_encode      LdpcCode.encode (ldpc.py:88-90) for codes with a
 *                        staircase parity part (chain_cols != NULL): the
 *                        reference's dense GF(2) encoder (encode_mat_t,
 *                        ldpc.py:80) is O(k*m) and does not scale to a
 *                        273-PRB codeword; the staircase encoder is O(edges).
 *
 * Columns may have degree < 3 (-1 padded), so both the reference's
 * column-weight-3 codes and the IRA codes (parity columns of degree 2 / 1)
 * go through the same decoder.  Work is enqueued on `stream`; nothing but
 * nrx_ldpc_create allocates or synchronises.
 */
#ifndef NRX_LDPC_H_
#define NRX_LDPC_H_

#include <stddef.h>
#include <stdint.h>

#include "nrx_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define NRX_LDPC_MAX_COL_DEG 3
#define NRX_LDPC_MAX_ROW_DEG 64

/* Host description of one code (all arrays host memory, int32). */
typedef struct nrx_ldpc_desc {
  int32_t n;               /* mother code length                          */
  int32_t m;               /* parity checks                               */
  int32_t k;               /* information positions of the mother code    */
  int32_t dmax;            /* row_cols width                              */
  int32_t cdeg;            /* col_rows / col_slots width (<= 3)           */
  const int32_t* row_cols;       /* (m, dmax), -1 padded                  */
  const int32_t* col_rows;       /* (n, cdeg), -1 padded                  */
  const int32_t* col_slots;      /* (n, cdeg): slot of the column in row  */
  const int32_t* info_positions; /* (k) ascending                         */
  int32_t n_punctured;
  const int32_t* punctured;      /* coded positions not transmitted       */
  int32_t n_shortened;
  const int32_t* shortened;      /* info positions fixed to 0, not sent   */
  const int32_t* chain_cols;     /* (m) staircase parity column of chain
                                    position i, or NULL: decode only      */
  int32_t chain_step;            /* Z: check i holds chain positions i-Z
                                    and i (Z interleaved accumulators)    */
} nrx_ldpc_desc;

typedef struct nrx_ldpc_code nrx_ldpc_code;   /* device-resident, opaque */

/* Validates and uploads (cudaMalloc + copies on the current device). */
int nrx_ldpc_create(const nrx_ldpc_desc* desc, nrx_ldpc_code** out);
void nrx_ldpc_destroy(nrx_ldpc_code* code);
/* out4 = {n, k_eff, num_tx_bits, m} */
int nrx_ldpc_dims(const nrx_ldpc_code* code, int32_t* out4);
size_t nrx_ldpc_workspace_bytes(const nrx_ldpc_code* code, int n_codewords);

/*
 * llr      (n_codewords, num_tx_bits) float32 logit LLRs (positive: bit 1)
 * info_out (n_codewords, k_eff) uint8 decoded information bits
 * success  (n_codewords) uint8: all parity checks satisfied at exit
 */
int nrx_ldpc_decode(const nrx_ldpc_code* code, int n_codewords, const float* llr, int iterations,
                    uint8_t* info_out, uint8_t* success, void* workspace, size_t workspace_bytes,
                    void* stream);

/* info (n_codewords, k_eff) uint8 -> tx_bits (n_codewords, num_tx_bits) uint8 */
int nrx_ldpc_encode(const nrx_ldpc_code* code, int n_codewords, const uint8_t* info, uint8_t* tx_bits,
                    void* workspace, size_t workspace_bytes, void* stream);

/* ---- coded Monte-Carlo glue (evaluation._evaluate_chunk, evaluation.py:165-209) ----
 * Per UE u of a slot batch: E = num_data_res * m coded bits fill the data REs
 * subcarrier-major, m bits per RE, first bit = most significant label bit
 * (assemble_slot slot.py:204-209); extract_data_llrs (slot.py:225-228) is the
 * inverse on the receiver's LLR grid. */

/* payload / info bits: out (rows, cols) uint8 iid Bernoulli(1/2), Philox
 * keyed by (seed, first_row + row) so a row never depends on the batch. */
int nrx_random_bits(uint64_t seed, uint64_t first_row, int rows, int cols, uint8_t* out, void* stream);

/* bits (n_slots, E) of UE `ue` -> labels[:, ue] (n_slots, U, S, T) uint8
 * (label index of each data RE; pilot / null REs untouched). */
int nrx_bits_to_labels(const nrx_slot_desc* slot, int n_slots, int ue, int mod_order, const uint8_t* bits,
                       uint8_t* labels, void* stream);

/* llr (n_slots, U, S, T, llr_width) -> out (n_slots, E) of UE `ue`,
 * clipped to [-clip, clip] (evaluation.py:200-201). */
int nrx_extract_llrs(const nrx_slot_desc* slot, int n_slots, int ue, int mod_order, const float* llr,
                     int llr_width, float clip, float* out, void* stream);

/* errors[row] += number of positions where a != b, rows x cols uint8. */
int nrx_count_mismatches(int rows, int cols, const uint8_t* a, const uint8_t* b, unsigned long long* errors,
                         void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NRX_LDPC_H_ */
