"""The drop-in inside the reference's own harness.

``oracle/_ref`` holds the unmodified reference package (oracle/build_ref.sh;
test infrastructure only).  With ``paper_2409_02912_b200.nrx.install`` applied
to ``nrxsim.evaluation``, the reference's own callers run the receiver on the
GPU with the reference's own objects (SlotConfig / McsEntry / PilotBook /
NrxConfig, ``ad.Tensor`` weights with requires_grad from ``checkpoint_load``
and ``init_weights``):

  ReceiverBank.run("nrx")   evaluation.py:144-154  vs the uninstalled CPU run, fp32 gate
  latency_bench             evaluation.py:322-363  returns a LatencyReport
  evaluate_tbler            evaluation.py:212-256  4 workers == 1 worker; vs the CPU run
  nrxsim CLI bench / eval   cli.py:95-129          write their CSVs
"""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
CKPT = os.path.join(ROOT, "tests", "golden", "desk_d16_it2.nrxw")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "nrxsim")):
        pytest.skip("oracle/_ref (the reference package) is not built")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import nrxsim.cli
    import nrxsim.evaluation
    import nrxsim.nrx
    return nrxsim


@pytest.fixture
def installed(ref):
    from paper_2409_02912_b200 import nrx as gnrx
    prev = gnrx.install(ref.evaluation)
    try:
        yield
    finally:
        ref.evaluation.nrx_forward = prev


def _table(ref):
    from nrxsim import configio
    return configio.build_mcs_table(configio.load_config())


def _chunk(ref, cfg, entries, n, snr_db=8.0, seed=3):
    """Slots built exactly as evaluation._evaluate_chunk builds them."""
    from nrxsim.channel import ChannelRealization, apply_channel, doubletdl
    from nrxsim.slot import assemble_slot, beamform, generate_pilots, random_payloads
    source = doubletdl()
    n0 = 10.0 ** (-snr_db / 10.0)
    y = np.empty((n, cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas), np.complex128)
    h_eff = np.empty((n, cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas), np.complex128)
    books = []
    for i in range(n):
        rng = np.random.default_rng((seed, 1, i, 1))
        tx = assemble_slot(cfg, entries, random_payloads(cfg, entries, rng), int(rng.integers(0, 2 ** 62)))
        h = source.sample(cfg, (seed, 1, i, 2))
        ants = np.stack([beamform(tx.grids[u].symbols, cfg.beam_matrix[u]) for u in range(cfg.num_ues)])
        real = ChannelRealization(h=h, n0=n0)
        y[i] = apply_channel(ants, real, np.random.default_rng((seed, 1, i, 3)))
        h_eff[i] = real.effective(cfg)
        books.append(tx.pilot_book)
    return y, books, h_eff, n0


def test_receiver_bank_nrx_on_gpu_matches_cpu(ref):
    from nrxsim import evaluation as ev
    from nrxsim.nrx import checkpoint_load
    from nrxsim.slot import SlotConfig
    from paper_2409_02912_b200 import nrx as gnrx
    table = _table(ref)
    cfg = SlotConfig(num_subcarriers=48)
    config, w = checkpoint_load(CKPT)
    assert all(getattr(t, "requires_grad", False) for t in w.values())  # reference ad.Tensor weights
    ecfg = ev.EvalConfig(snr_grid_db=(8.0,), receivers=("nrx",), mcs_indices=(14, 14), seed=3)
    bank = ev.ReceiverBank(ecfg, cfg, table, nrx_model=(config, w))
    y, books, h_eff, n0 = _chunk(ref, cfg, bank.entries, 6)
    cpu = bank.run("nrx", y, books, h_eff, n0)
    prev = gnrx.install(ev)
    try:
        gpu = bank.run("nrx", y, books, h_eff, n0)
    finally:
        ev.nrx_forward = prev
    scale = max(float(np.abs(c).max()) for c in cpu)
    for c, g in zip(cpu, gpu):
        assert g.shape == c.shape and g.dtype == np.float32
        assert np.abs(g.astype(np.float64) - c).max() <= 1e-5 * scale


def test_latency_bench_returns_report(ref, installed, tmp_path):
    from nrxsim import evaluation as ev
    from nrxsim.nrx import init_weights
    from nrxsim.nrx import NrxConfig
    from nrxsim.slot import SlotConfig
    table = _table(ref)
    cfg = SlotConfig(num_subcarriers=48)
    config = NrxConfig.from_table(table, (14,), d_s=16, num_iterations=4)
    rep = ev.latency_bench((config, init_weights(config, seed=0)), cfg, table, depths=(1, 2, 4), runs=5, warmup=2)
    assert isinstance(rep, ev.LatencyReport)
    assert set(rep.median_s) == {1, 2, 4} and all(0 < v < 0.05 for v in rep.median_s.values())
    path = tmp_path / "latency.csv"
    ev.write_latency_csv(rep, path)  # the reference's latency CSV schema (evaluation.py:404-410)
    lines = path.read_text().splitlines()
    assert lines[0] == "n_it,median_s,p10_s,p90_s" and [int(x.split(",")[0]) for x in lines[1:4]] == [1, 2, 4]
    assert lines[4].startswith("# fit a=")


def test_check_finite_follows_reference_switch(ref):
    """autodiff.CHECK_FINITE (autodiff.py:27-29,130-131) makes the reference
    raise FloatingPointError on a non-finite forward; with install() applied
    the GPU drop-in follows the same switch, and stays silent without it."""
    from nrxsim import autodiff, evaluation as ev
    from nrxsim.nrx import checkpoint_load
    from nrxsim.slot import SlotConfig
    from paper_2409_02912_b200 import nrx as gnrx
    table = _table(ref)
    cfg = SlotConfig(num_subcarriers=48)
    config, w = checkpoint_load(CKPT)
    ecfg = ev.EvalConfig(snr_grid_db=(8.0,), receivers=("nrx",), mcs_indices=(14, 14), seed=3)
    bank = ev.ReceiverBank(ecfg, cfg, table, nrx_model=(config, w))
    y, books, h_eff, n0 = _chunk(ref, cfg, bank.entries, 2)
    y[1, 5, 3, 0] = np.nan
    prev_flag = autodiff.CHECK_FINITE
    autodiff.CHECK_FINITE = True
    try:
        with pytest.raises(FloatingPointError):
            bank.run("nrx", y, books, h_eff, n0)       # the reference on the CPU
        prev = gnrx.install(ev)
        try:
            with pytest.raises(FloatingPointError, match="non-finite"):
                bank.run("nrx", y, books, h_eff, n0)   # the drop-in
            autodiff.CHECK_FINITE = False
            out = bank.run("nrx", y, books, h_eff, n0)
            assert not all(np.isfinite(o).all() for o in out)
        finally:
            ev.nrx_forward = prev
    finally:
        autodiff.CHECK_FINITE = prev_flag


def test_evaluate_tbler_workers_and_cpu(ref):
    from nrxsim import evaluation as ev
    from nrxsim.channel import doubletdl
    from nrxsim.nrx import checkpoint_load
    from nrxsim.slot import SlotConfig
    from paper_2409_02912_b200 import nrx as gnrx
    table = _table(ref)
    cfg = SlotConfig(num_subcarriers=48)
    model = checkpoint_load(CKPT)
    base = dict(snr_grid_db=(6.0, 10.0), receivers=("nrx",), mcs_indices=(14, 14), seed=5, min_block_errors=10_000,
                max_blocks=48, chunk_slots=6)
    cpu = ev.evaluate_tbler(cfg, doubletdl(), ev.EvalConfig(**base), table, nrx_model=model)
    prev = gnrx.install(ev)
    try:
        one = ev.evaluate_tbler(cfg, doubletdl(), ev.EvalConfig(**base, num_workers=1), table, nrx_model=model)
        four = ev.evaluate_tbler(cfg, doubletdl(), ev.EvalConfig(**base, num_workers=4), table, nrx_model=model)
    finally:
        ev.nrx_forward = prev
    assert one == four  # bit-reproducible for any worker count, like the reference
    for c, g in zip(cpu, one):
        assert (c.receiver, c.snr_db, c.blocks, c.bits) == (g.receiver, g.snr_db, g.blocks, g.bits)
        # LLRs agree to the fp32 gate; an LDPC decode sitting exactly on the edge may flip
        assert abs(c.block_errors - g.block_errors) <= 1
        assert abs(c.bit_errors - g.bit_errors) <= max(4, 0.02 * c.bit_errors)


def test_cli_bench_and_eval(ref, installed, tmp_path):
    from nrxsim import cli
    lat = tmp_path / "lat.csv"
    assert cli.main(["bench", "--seed", "0", "--depths", "1,2", "--runs", "3", "--out", str(lat),
                     "--slot.num_subcarriers=48"]) == 0
    lines = lat.read_text().splitlines()
    assert lines[0] == "n_it,median_s,p10_s,p90_s" and len(lines) == 4
    out = tmp_path / "eval.csv"
    assert cli.main(["eval", "--seed", "1", "--ckpt", CKPT, "--out", str(out), "--slot.num_subcarriers=48",
                     "--eval.receivers=nrx", "--eval.snr_grid_db=8", "--eval.max_blocks=16",
                     "--eval.chunk_slots=4"]) == 0
    rows = out.read_text().splitlines()
    assert rows[0].startswith("receiver,snr_db,blocks") and rows[1].startswith("nrx,8,16,")
