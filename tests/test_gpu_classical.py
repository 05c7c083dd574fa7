"""GPU classical baseline: the ls_lmmse receiver
against the reference's own outputs (golden fixtures, float64 arithmetic on
both sides; LLRs compared at float32 output precision) and the CPU oracle at
C2 size; plus the GPU Monte-Carlo loops run it as the comparison receiver."""

import numpy as np
import pytest

from oracle import classical_oracle as co
from oracle import slotgen_oracle as so
from slotgen_cases import case_names, load_case
from test_classical_cpu import GOLDEN, load_cl

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", case_names())
def test_ls_lmmse_matches_reference(name):
    from paper_2409_02912_b200.classical import ls_lmmse_llrs
    from paper_2409_02912_b200.config import McsEntry, PilotBook
    c = load_case(name)
    cfg = c.cfg
    books = []
    for i in range(c.n):
        vals = np.zeros((cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols), complex)
        for u in range(cfg.num_ues):
            sc = np.arange(u % cfg.comb_size, cfg.num_subcarriers, cfg.comb_size)
            vals[u][np.ix_(sc, list(cfg.pilot_symbols))] = c.a["pilots"][i, u, :sc.size]
        books.append(PilotBook(vals, cfg))
    mcs = [McsEntry(0, m, 0.5) for m in c.orders]
    got = ls_lmmse_llrs(c.a["y"], books, cfg, mcs, c.n0)
    for g, r in zip(got, load_cl(name)):
        assert g.shape == r.shape and g.dtype == np.float32
        np.testing.assert_allclose(g, r, rtol=2e-6, atol=2e-5)


def test_ls_lmmse_c2_vs_oracle_and_ber():
    torch = __import__("torch")
    from paper_2409_02912_b200.classical import GpuLsLmmse
    from paper_2409_02912_b200.config import SlotConfig
    from paper_2409_02912_b200.slotgen import GpuSlotSource, labels_to_bits
    cfg = SlotConfig(num_subcarriers=3276, num_ues=2)
    n0 = 0.05
    b = GpuSlotSource(cfg).generate(2, (4, 6), n0, seed=3, y_dtype=torch.complex128,
                                    pilots_dtype=torch.complex128)
    rx = GpuLsLmmse(4, 6)
    llr = torch.empty((2, 2, 3276, 14, 6), dtype=torch.float32, device="cuda")
    rx.forward_device(cfg, b.y, b.pilots, None, b.mod_order, 1, llr, n0=b.n0)
    got = llr.cpu().numpy()
    ref = co.ls_lmmse_llrs(cfg, b.y.cpu().numpy(), b.pilots.cpu().numpy(), n0, (4, 6), so.gray_points)
    for u, m in enumerate((4, 6)):
        np.testing.assert_allclose(got[:, u, ..., :m], ref[u], rtol=2e-6, atol=2e-5)
        assert not got[:, u, ..., m:].any()
    # a sane receiver: uncoded BER well below 1/2 at 13 dB on the TDL channels
    s_idx, t_idx = np.nonzero(cfg.data_mask)
    bits = labels_to_bits(b.labels.cpu().numpy(), cfg, (4, 6))
    for u, m in enumerate((4, 6)):
        ber = np.mean((got[:, u][:, s_idx, t_idx, :m] > 0) != bits[u])
        assert ber < 0.2, ber


@pytest.mark.parametrize("k", [16, 4])
@pytest.mark.parametrize("name", case_names())
def test_kbest_matches_reference(name, k):
    """perfect_kbest on the true channel vs the reference (float64 both
    sides; list membership can differ only on metric ties at the K-th place,
    so all but a negligible fraction of LLRs must agree)."""
    from paper_2409_02912_b200.classical import kbest_llrs
    from paper_2409_02912_b200.config import McsEntry
    c = load_case(name)
    mcs = [McsEntry(0, m, 0.5) for m in c.orders]
    got = kbest_llrs(c.a["y"], c.a["h_eff"], c.cfg, mcs, c.n0, k=k)
    with np.load(f"{GOLDEN}/kb_{name}.npz") as z:
        ref = [z[f"k{k}_llr_{u}"] for u in range(len(c.orders))]
    for g, r in zip(got, ref):
        assert g.shape == r.shape
        close = np.isclose(g, r, rtol=1e-5, atol=1e-4)
        assert close.mean() > 0.999, (name, k, close.mean())


def test_kbest_pairing_modes():
    """The two interference pairings agree for U <= 2 and differ for U = 3,
    where the corrected one decides at least as well (reference defect at
    classical.py:220-221)."""
    from paper_2409_02912_b200.classical import kbest_llrs
    from paper_2409_02912_b200.config import McsEntry
    from paper_2409_02912_b200.slotgen import labels_to_bits
    for name in ("sg_desk", "sg_u3_comb4"):
        c = load_case(name)
        mcs = [McsEntry(0, m, 0.5) for m in c.orders]
        a = kbest_llrs(c.a["y"], c.a["h_eff"], c.cfg, mcs, c.n0, k=16)
        b = kbest_llrs(c.a["y"], c.a["h_eff"], c.cfg, mcs, c.n0, k=16, reference_pairing=False)
        same = all(np.array_equal(x, z) for x, z in zip(a, b))
        assert same == (len(c.orders) <= 2)
        if not same:
            s_idx, t_idx = np.nonzero(c.cfg.data_mask)
            bits = labels_to_bits(c.a["labels"], c.cfg, c.orders)
            err = lambda g: sum(int(((x[:, s_idx, t_idx] > 0) != bb).sum()) for x, bb in zip(g, bits))
            assert err(b) <= err(a)


def test_monte_carlo_loops_run_the_baseline():
    from paper_2409_02912_b200.classical import GpuLsLmmse
    from paper_2409_02912_b200.config import McsEntry, SlotConfig, default_mcs_table
    from paper_2409_02912_b200.ldpc import evaluate_coded
    from paper_2409_02912_b200.slotgen import GpuSlotSource, evaluate_uncoded
    cfg = SlotConfig(num_subcarriers=96, num_ues=2)
    src = GpuSlotSource(cfg)
    rx = GpuLsLmmse(4, 4)
    t = default_mcs_table()
    unc = evaluate_uncoded(rx, src, (t[14], t[14]), [0.0, 30.0], n_slots=16, batch=8, receiver="ls_lmmse")
    assert unc[0].ber > unc[1].ber and unc[1].ber < 0.05
    mcs = (McsEntry(14, 4, 0.3), McsEntry(14, 4, 0.3))
    cod = evaluate_coded(rx, src, mcs, [0.0, 30.0], n_slots=16, batch=8, receiver="ls_lmmse")
    assert cod[0].receiver == "ls_lmmse" and cod[0].tbler > cod[1].tbler
    assert cod[1].tbler < 0.2
    from paper_2409_02912_b200.classical import GpuKBest
    kb = evaluate_uncoded(GpuKBest(4, 4, 16), src, (t[14], t[14]), [0.0, 30.0], n_slots=16, batch=8,
                          receiver="perfect_kbest")
    assert kb[1].ber < unc[1].ber + 1e-3 and kb[0].ber < unc[0].ber   # true channel beats LS


def _lm(name):
    with np.load(f"{GOLDEN}/lm_{name}.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("name", ["sg_desk", "sg_mixed", "sg_b8_t7"])
def test_covariance_reference_stream(name):
    from paper_2409_02912_b200.classical import estimate_covariance
    from paper_2409_02912_b200.slotgen import GpuSlotSource
    c = load_case(name)
    g = _lm(name)
    cov = estimate_covariance(GpuSlotSource(c.cfg, c.profiles), 120, seed=4, reference_stream=True)
    np.testing.assert_allclose(cov.freq.cpu().numpy(), g["r_f"], rtol=0, atol=1e-12 * np.abs(g["r_f"]).max())
    np.testing.assert_allclose(cov.time.cpu().numpy(), g["r_t"], rtol=0, atol=1e-12 * np.abs(g["r_t"]).max())


@pytest.mark.parametrize("name", ["sg_desk", "sg_mixed", "sg_b8_t7"])
def test_lmmse_kbest_matches_reference(name):
    torch = __import__("torch")
    from paper_2409_02912_b200.classical import CovarianceModel, GpuLmmseKBest, lmmse_estimate, lmmse_weights
    c = load_case(name)
    g = _lm(name)
    cov = CovarianceModel(torch.from_numpy(g["r_f"]).cuda(), torch.from_numpy(g["r_t"]).cuda(), 120)
    y = torch.from_numpy(c.a["y"]).cuda()
    pil = torch.from_numpy(c.a["pilots"]).cuda()
    h = lmmse_estimate(c.cfg, y, pil, lmmse_weights(c.cfg, cov, c.n0)).cpu().numpy()
    np.testing.assert_allclose(h, g["h_est"], rtol=0, atol=1e-10 * np.abs(g["h_est"]).max())
    U = c.cfg.num_ues
    rx = GpuLmmseKBest(cov, c.cfg.bs_antennas, max(c.orders), 16)
    mods = torch.tensor(list(c.orders) * c.n, dtype=torch.int32, device="cuda")
    llr = torch.empty((c.n, U, c.cfg.num_subcarriers, c.cfg.num_symbols, max(c.orders)), dtype=torch.float32,
                      device="cuda")
    rx.forward_device(c.cfg, y, pil, None, mods, 1, llr, n0=torch.full((c.n,), c.n0, dtype=torch.float64,
                                                                      device="cuda"))
    got = llr.cpu().numpy()
    for u, m in enumerate(c.orders):
        close = np.isclose(got[:, u, ..., :m], g[f"llr_{u}"], rtol=1e-5, atol=1e-4)
        assert close.mean() > 0.999, (name, close.mean())
