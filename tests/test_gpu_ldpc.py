"""GPU LDPC layer.

Decoder: bit-identical to the reference decoder on the reference's own codes
(golden fixtures, 20 and 3 iterations, converged and non-converged
codewords) and to the CPU oracle on IRA codes.  Encoder: bit-identical to the
oracle's staircase encoder; codewords satisfy every parity check.  Glue:
bits <-> labels <-> LLR extraction round trips.  Pipeline: the coded
Monte-Carlo loop is deterministic across batch sizes / ranks and its TBLER
falls with SNR for a trained receiver."""

import numpy as np
import pytest

from oracle import ldpc_oracle as lo
from test_ldpc_cpu import golden_names, load_golden

pytestmark = pytest.mark.gpu


def _t():
    import torch
    return torch


@pytest.mark.parametrize("name", golden_names())
def test_decoder_bit_exact_vs_reference(name):
    torch = _t()
    from paper_2409_02912_b200.ldpc import GpuLdpc
    code, a = load_golden(name)
    g = GpuLdpc(code)
    llr = torch.from_numpy(a["llr"]).cuda()
    for it, dk, ok in ((20, "dec20", "ok20"), (3, "dec3", "ok3")):
        dec, done = g.decode(llr, it)
        np.testing.assert_array_equal(done.cpu().numpy(), a[ok])
        np.testing.assert_array_equal(dec.cpu().numpy(), a[dk])
    g.close()


def test_decoder_bit_exact_vs_oracle_on_ira():
    torch = _t()
    from paper_2409_02912_b200.ldpc import GpuLdpc, rate_matched_ira_code
    code = rate_matched_ira_code(4 * 1152, 553 / 1024)
    rng = np.random.default_rng(5)
    info = (rng.random((12, code.k_eff)) < 0.5).astype(np.uint8)
    tx = lo.staircase_codeword(code, info)[:, code.tx_positions].astype(np.float64)
    sig = np.repeat([0.55, 0.7, 0.85, 1.0], 3)[:, None]
    llr = np.clip(2 * ((2 * tx - 1) + sig * rng.normal(size=tx.shape)) / sig ** 2, -20, 20).astype(np.float32)
    g = GpuLdpc(code)
    dec, ok = g.decode(torch.from_numpy(llr).cuda(), 20)
    ref_dec, ref_ok = lo.decode(code, llr, 20)
    np.testing.assert_array_equal(ok.cpu().numpy(), ref_ok)
    np.testing.assert_array_equal(dec.cpu().numpy(), ref_dec)
    assert 0 < ref_ok.sum() < 12          # both converging and failing codewords exercised


def test_decoder_multi_group_ragged_vs_oracle():
    """70 codewords = three 32-lane groups, the last one ragged, all
    decoded concurrently; results match the oracle at 20, 4, 1 and 0
    iterations (the first iteration takes its zero messages implicitly)."""
    torch = _t()
    from paper_2409_02912_b200.ldpc import GpuLdpc, rate_matched_ira_code
    code = rate_matched_ira_code(2 * 1152, 553 / 1024, seed=3)
    rng = np.random.default_rng(11)
    info = (rng.random((70, code.k_eff)) < 0.5).astype(np.uint8)
    tx = lo.staircase_codeword(code, info)[:, code.tx_positions].astype(np.float64)
    sig = np.linspace(0.5, 1.05, 70)[:, None]
    llr = np.clip(2 * ((2 * tx - 1) + sig * rng.normal(size=tx.shape)) / sig ** 2, -20, 20).astype(np.float32)
    g = GpuLdpc(code)
    for it in (20, 4, 1, 0):
        dec, ok = g.decode(torch.from_numpy(llr).cuda(), it)
        ref_dec, ref_ok = lo.decode(code, llr, it)
        np.testing.assert_array_equal(ok.cpu().numpy(), ref_ok)
        np.testing.assert_array_equal(dec.cpu().numpy(), ref_dec)
        if it == 20:
            assert 0 < ref_ok.sum() < 70
    g.close()


def _regular_code(n, m, seed):
    """Column weight 3, row weight 3n/m (socket permutation, no repeated
    check in a column), first n - m positions as information, a few
    punctured / shortened positions: exercises the decoder's row widths other
    than the IRA codes' 5 and the reference codes' 6."""
    from paper_2409_02912_b200.ldpc import LdpcCode
    rng = np.random.default_rng(seed)
    dr = 3 * n // m
    while True:
        sockets = rng.permutation(np.repeat(np.arange(m), dr))[: 3 * n].reshape(n, 3)
        if all(len(set(r)) == 3 for r in sockets):
            break
    row_cols = np.full((m, dr), -1, dtype=np.int32)
    col_slots = np.zeros((n, 3), dtype=np.int32)
    fill = np.zeros(m, dtype=np.int64)
    for j in range(n):
        for t in range(3):
            r = sockets[j, t]
            row_cols[r, fill[r]] = j
            col_slots[j, t] = fill[r]
            fill[r] += 1
    k = n - m
    return LdpcCode(n, k, row_cols, sockets.astype(np.int32), col_slots, np.arange(k),
                    punctured=np.array([n - 1, n - 2]), shortened=np.array([0, 3]))


@pytest.mark.parametrize("n,m", [(700, 300), (640, 240), (900, 300)])
def test_decoder_other_row_widths_vs_oracle(n, m):
    """Row widths 7, 8 (fixed-width check kernels) and 9 (generic): all-zero
    codeword over AWGN at noise levels across the waterfall, 40 codewords."""
    torch = _t()
    from paper_2409_02912_b200.ldpc import GpuLdpc
    code = _regular_code(n, m, seed=n + m)
    rng = np.random.default_rng(7)
    ntx = code.num_tx_bits
    sig = np.linspace(0.4, 1.0, 40)[:, None]
    llr = np.clip(2 * (-1 + sig * rng.normal(size=(40, ntx))) / sig ** 2, -20, 20).astype(np.float32)
    g = GpuLdpc(code)
    for it in (20, 2):
        dec, ok = g.decode(torch.from_numpy(llr).cuda(), it)
        ref_dec, ref_ok = lo.decode(code, llr, it)
        np.testing.assert_array_equal(ok.cpu().numpy(), ref_ok)
        np.testing.assert_array_equal(dec.cpu().numpy(), ref_dec)
        if it == 20:
            assert 0 < ref_ok.sum() < 40
    g.close()


@pytest.mark.parametrize("e,rate", [(1152, 553 / 1024), (900, 0.33), (3276 * 12 * 4, 553 / 1024)])
def test_encoder_matches_oracle_and_round_trips(e, rate):
    torch = _t()
    from paper_2409_02912_b200.ldpc import GpuLdpc, rate_matched_ira_code
    code = rate_matched_ira_code(e, rate)
    g = GpuLdpc(code)
    rng = np.random.default_rng(6)
    b = 3 if e > 100000 else 8
    info = (rng.random((b, code.k_eff)) < 0.5).astype(np.uint8)
    tx = g.encode(torch.from_numpy(info).cuda()).cpu().numpy()
    cw = lo.staircase_codeword(code, info)
    np.testing.assert_array_equal(tx, cw[:, code.tx_positions])
    assert lo.check_parity(code.row_cols, cw).all()
    dec, ok = g.decode(torch.from_numpy(20.0 * (2 * tx.astype(np.float32) - 1)).cuda(), 20)
    assert ok.all()
    np.testing.assert_array_equal(dec.cpu().numpy(), info)


def test_glue_bits_labels_llrs():
    torch = _t()
    import ctypes
    from paper_2409_02912_b200 import _lib
    from paper_2409_02912_b200.config import SlotConfig
    from paper_2409_02912_b200.slotgen import labels_to_bits
    lib = _lib.load()
    cfg = SlotConfig(num_subcarriers=60, num_ues=2)
    s = _lib.slot_desc(cfg)
    n, orders = 3, (4, 6)
    st = torch.cuda.current_stream().cuda_stream
    labels = torch.zeros((n, 2, 60, 14), dtype=torch.uint8, device="cuda")
    bits = []
    for u, m in enumerate(orders):
        b = torch.empty((n, cfg.num_data_res * m), dtype=torch.uint8, device="cuda")
        assert lib.nrx_random_bits(77, 10 * u, n, b.shape[1], b.data_ptr(), st) == 0
        assert lib.nrx_bits_to_labels(ctypes.byref(s), n, u, m, b.data_ptr(), labels.data_ptr(), st) == 0
        bits.append(b.cpu().numpy())
    back = labels_to_bits(labels.cpu().numpy(), cfg, orders)
    for u, m in enumerate(orders):
        np.testing.assert_array_equal(back[u].reshape(n, -1), bits[u])
        assert 0.45 < bits[u].mean() < 0.55
    # Philox rows do not depend on the batch they were drawn in
    one = torch.empty((1, 500), dtype=torch.uint8, device="cuda")
    lib.nrx_random_bits(77, 11, 1, 500, one.data_ptr(), st)
    two = torch.empty((3, 500), dtype=torch.uint8, device="cuda")
    lib.nrx_random_bits(77, 10, 3, 500, two.data_ptr(), st)
    assert torch.equal(one[0], two[1])
    # LLR extraction: data REs subcarrier-major, clipped (slot.py:225-228, evaluation.py:200-201)
    llr = torch.randn((n, 2, 60, 14, 6), device="cuda") * 30
    out = torch.empty((n, cfg.num_data_res * 6), dtype=torch.float32, device="cuda")
    assert lib.nrx_extract_llrs(ctypes.byref(s), n, 1, 6, llr.data_ptr(), 6, 20.0, out.data_ptr(), st) == 0
    s_idx, t_idx = np.nonzero(cfg.data_mask)
    want = np.clip(llr.cpu().numpy()[:, 1][:, s_idx, t_idx, :6].reshape(n, -1), -20, 20)
    np.testing.assert_array_equal(out.cpu().numpy(), want)
    errs = torch.zeros(n, dtype=torch.int64, device="cuda")
    a = torch.from_numpy(bits[0]).cuda()
    b2 = a.clone()
    b2[1, :7] ^= 1
    assert lib.nrx_count_mismatches(n, a.shape[1], a.data_ptr(), b2.data_ptr(), errs.data_ptr(), st) == 0
    assert errs.tolist() == [0, 7, 0]


def _desk_long():
    """Desk receiver trained further by the reference trainer (4-24 dB,
    tests/golden/train_desk_long.py); its uncoded 16-QAM BER floors near
    0.17, so the coded tests use a low code rate (the MCS row is a labelled
    test setting: index 14, 16-QAM, rate 0.2)."""
    import os
    from paper_2409_02912_b200.config import McsEntry, SlotConfig, checkpoint_load
    from paper_2409_02912_b200.engine import NrxEngine
    from paper_2409_02912_b200.slotgen import GpuSlotSource
    here = os.path.dirname(os.path.abspath(__file__))
    config, w = checkpoint_load(os.path.join(here, "golden", "desk_d16_it2_long.nrxw"))
    cfg = SlotConfig(num_subcarriers=96, num_ues=2)
    mcs = (McsEntry(14, 4, 0.2), McsEntry(14, 4, 0.2))
    return cfg, mcs, GpuSlotSource(cfg), NrxEngine(config, w, precision="fp16")


def test_coded_pipeline_world_size_invariant_and_tbler_falls():
    from paper_2409_02912_b200.ldpc import evaluate_coded, slot_code
    cfg, mcs, src, eng = _desk_long()
    codes = [slot_code(cfg, m) for m in mcs]
    full = evaluate_coded(eng, src, mcs, [0.0, 25.0], n_slots=40, batch=16, seed=2, codes=codes)
    parts = [evaluate_coded(eng, src, mcs, [0.0, 25.0], n_slots=40, batch=7, seed=2, rank=r, world=2, codes=codes)
             for r in range(2)]
    for k in range(2):
        a, p0, p1 = full[k], parts[0][k], parts[1][k]
        assert (a.blocks, a.block_errors, a.bit_errors, a.bits) == (
            p0.blocks + p1.blocks, p0.block_errors + p1.block_errors, p0.bit_errors + p1.bit_errors,
            p0.bits + p1.bits)
    assert full[0].blocks == 80 and full[0].bits == 40 * 2 * codes[0].k_eff
    assert full[0].tbler > 0.9 and full[1].tbler < 0.5          # decodes at high SNR, not at 0 dB


def test_coded_pipeline_matches_host_recomputation():
    """Every step of evaluate_coded re-done on the host from the same
    streams: payload bits (device Philox), oracle staircase encoder, labels,
    the same GPU slots and receiver LLRs, oracle min-sum decoder -> identical
    block and bit error counts."""
    import ctypes
    torch = _t()
    from paper_2409_02912_b200 import _lib
    from paper_2409_02912_b200.ldpc import LLR_CLIP, evaluate_coded, slot_code
    from paper_2409_02912_b200.nrx import noise_features
    cfg, mcs, src, eng = _desk_long()
    codes = [slot_code(cfg, m) for m in mcs]
    n, snr, seed = 6, 12.0, 5
    rec = evaluate_coded(eng, src, mcs, [snr], n_slots=n, batch=n, seed=seed, codes=codes)[0]
    lib = _lib.load()
    st = torch.cuda.current_stream().cuda_stream
    key = (seed << 20) + (0 << 4)                     # SNR point k = 0 (evaluate_coded's stream keys)
    s_idx, t_idx = np.nonzero(cfg.data_mask)
    labels = np.zeros((n, 2, cfg.num_subcarriers, cfg.num_symbols), np.uint8)
    payload = []
    for u, code in enumerate(codes):
        info = torch.empty((n, code.k_eff), dtype=torch.uint8, device="cuda")
        lib.nrx_random_bits(key + u, 0, n, code.k_eff, info.data_ptr(), st)
        info = info.cpu().numpy()
        tx = lo.staircase_codeword(code, info)[:, code.tx_positions].reshape(n, s_idx.size, 4)
        labels[:, u, s_idx, t_idx] = tx.astype(np.int64) @ np.array([8, 4, 2, 1])
        payload.append(info)
    n0 = 10 ** (-snr / 10)
    sb = src.generate(n, [4, 4], n0, seed=key + 15, first_slot=0, variates={"labels": labels})
    llr = torch.empty((n, 2, cfg.num_subcarriers, cfg.num_symbols, 4), dtype=torch.float32, device="cuda")
    chest = torch.empty((n, 2, cfg.num_subcarriers, cfg.num_symbols, 4), dtype=torch.complex64, device="cuda")
    eng.forward_device(cfg, sb.y, sb.pilots, torch.from_numpy(noise_features(n0, n)).cuda(), sb.mod_order,
                       eng.config.num_iterations, llr, chest)
    l = llr.cpu().numpy()
    blocks = bit_errs = 0
    for u, code in enumerate(codes):
        cw_llr = np.clip(l[:, u][:, s_idx, t_idx, :4].reshape(n, -1), -LLR_CLIP, LLR_CLIP)
        dec, _ = lo.decode(code, cw_llr, 20)
        e = (dec != payload[u]).sum(axis=1)
        blocks += int((e > 0).sum())
        bit_errs += int(e.sum())
    assert (rec.block_errors, rec.bit_errors) == (blocks, bit_errs)
    assert rec.blocks == 2 * n
