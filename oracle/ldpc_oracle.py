"""CPU oracle of the LDPC layer (test infrastructure only).

Restates the reference's flooding min-sum decoder and parity check
(/root/reference/pkg/src/nrxsim/ldpc.py:99-178) in numpy, generalised to
columns of degree <= 3 with -1 padding (the staircase parity columns of the
scalable IRA mother codes have degree 2 / 1), plus a plain encoder for those
codes.  Only tests/ may import this module.  Pinned bit-for-bit against the
reference's own decoder on the reference's own codes by
tests/golden/make_golden_ldpc.py -> tests/golden/ldpc_*.npz
(tests/test_ldpc_cpu.py).

Float32 operation order follows the reference exactly:
  total = chan + ((c2v_0 + c2v_1) + c2v_2)          (np.sum over 3, ldpc.py:144-145)
  v2c   = total[row_cols] - c2v                      (ldpc.py:154)
  c2v   = row_sign * sgn * (min2 at argmin else min1) (ldpc.py:155-165)
so a CUDA decoder that keeps the order is bit-identical.
"""

from __future__ import annotations

import numpy as np

SHORTENED_LLR = 60.0   # ldpc.py:25


def check_parity(row_cols, bits):
    """(..., n) bits -> (...,) all checks satisfied (ldpc.py:91-97)."""
    c = np.asarray(bits, dtype=np.uint8)
    pad = np.concatenate([c, np.zeros(c.shape[:-1] + (1,), dtype=np.uint8)], axis=-1)
    return (pad[..., row_cols].sum(axis=-1) % 2 == 0).all(axis=-1)


def decode(code, llrs, iterations=20):
    """Min-sum decode of (B, num_tx_bits) logit LLRs -> (info (B, k_eff), ok (B,)).

    `code` needs n, row_cols (M, dmax), col_rows / col_slots (n, <=3, -1 padded),
    info_positions, punctured, shortened, tx_positions."""
    llrs = np.asarray(llrs, dtype=np.float32)
    batch = llrs.shape[0]
    n = code.n
    chan = np.zeros((batch, n), dtype=np.float32)
    chan[:, code.tx_positions] = -llrs
    chan[:, code.shortened] = np.float32(SHORTENED_LLR)
    row_cols = np.asarray(code.row_cols)
    col_rows = np.asarray(code.col_rows)
    col_slots = np.asarray(code.col_slots)
    m, dmax = row_cols.shape
    valid = row_cols >= 0
    rows_safe = np.where(valid, row_cols, 0)
    cvalid = col_rows >= 0
    cr = np.where(cvalid, col_rows, 0)
    cs = np.where(cvalid, col_slots, 0)
    c2v = np.zeros((batch, m, dmax), dtype=np.float32)
    hard = np.zeros((batch, n), dtype=np.uint8)
    done = np.zeros(batch, dtype=bool)

    def totals():
        g = np.where(cvalid[None], c2v[:, cr, cs], np.float32(0))   # (B, n, deg)
        s = g[..., 0]
        for t in range(1, g.shape[-1]):
            s = s + g[..., t]
        return chan + s

    for _ in range(iterations):
        total = totals()
        bits = (total < 0).astype(np.uint8)
        ok = check_parity(row_cols, bits)
        newly = ok & ~done
        hard[newly] = bits[newly]
        done |= newly
        if done.all():
            break
        v2c = total[:, rows_safe] - c2v
        mag = np.where(valid, np.abs(v2c), np.float32(np.inf))
        sgn = np.where(valid & (v2c < 0), np.float32(-1), np.float32(1))
        row_sign = sgn.prod(axis=-1)
        amin = mag.argmin(axis=-1)
        min1 = np.take_along_axis(mag, amin[..., None], axis=-1)[..., 0]
        tmp = mag.copy()
        np.put_along_axis(tmp, amin[..., None], np.float32(np.inf), axis=-1)
        min2 = tmp.min(axis=-1)
        use2 = np.arange(dmax)[None, None, :] == amin[..., None]
        c2v = row_sign[..., None] * sgn * np.where(use2, min2[..., None], min1[..., None])
        c2v[:, ~valid] = 0.0
    else:
        bits = (totals() < 0).astype(np.uint8)
        hard[~done] = bits[~done]
    keep = ~np.isin(code.info_positions, code.shortened)
    return hard[:, code.info_positions][:, keep], done


def staircase_codeword(code, info):
    """Mother codeword of an IRA code from (B, k_eff) info bits: shortened
    info bits are zero, the parity chains p_i = s_i ^ p_{i-Z} over the
    checks' info syndromes s (check i holds chain positions i-Z, i)."""
    info = np.asarray(info, dtype=np.uint8)
    b = info.shape[0]
    u = np.zeros((b, code.k), dtype=np.uint8)
    keep = ~np.isin(code.info_positions, code.shortened)
    u[:, keep] = info
    cw = np.zeros((b, code.n), dtype=np.uint8)
    cw[:, code.info_positions] = u
    rc = np.asarray(code.row_cols)
    is_info = np.zeros(code.n + 1, dtype=bool)
    is_info[np.asarray(code.info_positions)] = True
    syn = np.zeros((b, rc.shape[0]), dtype=np.uint8)
    pad = np.concatenate([cw, np.zeros((b, 1), np.uint8)], axis=1)
    for r in range(rc.shape[0]):
        cols = rc[r][(rc[r] >= 0) & is_info[rc[r]]]
        syn[:, r] = pad[:, cols].sum(axis=1) % 2
    z = int(getattr(code, "chain_step", 1))
    par = np.zeros((b, rc.shape[0]), dtype=np.uint8)
    for i, col in enumerate(np.asarray(code.chain_cols)):
        par[:, i] = syn[:, i] ^ (par[:, i - z] if i >= z else 0)
        cw[:, col] = par[:, i]
    return cw
