"""Generate golden vectors for the NRX forward pass from the REFERENCE itself.

Run in the build container (where the read-only reference lives):

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/make_golden.py

For every case it builds synthetic slots with the reference's own generators
(``generate_pilots``, ``build_constellation(m).map_bits`` on the data REs,
``beamform``, ``TdlChannelSource`` + ``apply_channel``; LDPC is bypassed as
SURVEY.md finding 5 prescribes), weights with ``init_weights`` (optionally
bias-perturbed), and records the reference ``nrx_forward`` outputs plus the
assembled features (``assemble_features(y, ls_features(...))``).  The
fixtures are the anchor that pins ``oracle/nrx_oracle.py`` and, through it,
the CUDA path.  Nothing here is needed at run time on the GPU box.
"""

from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = os.environ.get("NRX_REFERENCE_SRC", "/root/reference/pkg/src")
if REF not in sys.path:
    sys.path.insert(0, REF)

from nrxsim import nrx  # noqa: E402
from nrxsim.channel import ChannelRealization, TdlChannelSource, apply_channel, tdl_b, tdl_c  # noqa: E402
from nrxsim.constellation import build_constellation  # noqa: E402
from nrxsim.slot import McsEntry, SlotConfig, beamform, default_mcs_table, generate_pilots  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
TABLE = default_mcs_table()


def synth_slots(cfg: SlotConfig, mcs, n_slots: int, n0: float, seed: int):
    """Reference-generated received grids y (N,S,T,B), per-slot books, data bits."""
    s_idx, t_idx = cfg.data_re_indices()
    ys, books, bits_all = [], [], []
    profiles = [tdl_b(), tdl_c()] * 4
    for i in range(n_slots):
        book = generate_pilots(cfg, slot_seed=seed * 1000 + i)
        rng = np.random.default_rng((seed, i))
        antennas, bits_u = [], []
        for u in range(cfg.num_ues):
            m = mcs[u].modulation_order
            bits = (rng.random((s_idx.size, m)) < 0.5).astype(np.uint8)
            sym = np.array(book.values[u])
            sym[s_idx, t_idx] = build_constellation(m).map_bits(bits)
            antennas.append(beamform(sym, cfg.beam_matrix[u]))
            bits_u.append(bits)
        h = TdlChannelSource(profiles[:cfg.num_ues]).sample(cfg, (seed, i))
        y = apply_channel(np.stack(antennas), ChannelRealization(h=h, n0=n0), rng)
        ys.append(y)
        books.append(book)
        bits_all.append(bits_u)
    return np.stack(ys), books, bits_all


def config_dict(obj) -> dict:
    d = dataclasses.asdict(obj)
    d.pop("beams", None)
    return {k: (list(v) if isinstance(v, tuple) else v) for k, v in d.items()}


CASES = [
    # name, slot kwargs, nrx kwargs (from_table), mcs indices, n_slots, n0, bias perturb, squeeze
    ("c1_small", dict(num_subcarriers=24, num_ues=1, comb_size=2),
     dict(supported=(14,), variant="single", d_s=16, num_iterations=2), (14,), 2, 0.1, False, False),
    ("mu2_masking_bias", dict(num_subcarriers=36, num_ues=2, comb_size=2),
     dict(supported=(9, 14, 19), variant="masking", d_s=16, num_iterations=3), (9, 19), 2, 0.05, True, False),
    ("mu3_var_io", dict(num_subcarriers=24, num_ues=3, comb_size=3),
     dict(supported=(9, 14, 19), variant="var_io", d_s=8, num_iterations=2), (14, 9, 19), 1, 0.2, True, True),
    ("t7_flags_off", dict(num_subcarriers=16, num_symbols=7, pilot_symbols=(2, 5), num_ues=2, comb_size=2),
     dict(supported=(14,), variant="single", d_s=12, num_iterations=2, hidden_width=20,
          include_noise_plane=False, include_freq_encoding=False), (14, 14), 2, 0.1, True, False),
    ("rt_d56", dict(num_subcarriers=48, num_ues=2, comb_size=2),
     dict(supported=(14,), variant="single", d_s=56, num_iterations=2), (14, 14), 1, 0.1, True, False),
    ("kernel5", dict(num_subcarriers=20, num_ues=2, comb_size=2),
     dict(supported=(14,), variant="single", d_s=8, num_iterations=2, kernel_size=5), (14, 14), 1, 0.1, True, False),
    ("one_pilot_odd_s", dict(num_subcarriers=25, pilot_symbols=(3,), num_ues=2, comb_size=2),
     dict(supported=(9, 14), variant="masking", d_s=8, num_iterations=2), (14, 9), 2, 0.3, True, False),
    ("comb4", dict(num_subcarriers=32, pilot_symbols=(2, 7, 11), num_ues=2, comb_size=4),
     dict(supported=(9, 14, 19), variant="var_io", d_s=16, num_iterations=2), (19, 19), 2, 0.1, True, False),
]


def perturb(w, seed=99, scale=0.1):
    rng = np.random.default_rng(seed)
    for name in sorted(w):
        if name.endswith(".b"):
            w[name].data[...] = rng.normal(0.0, scale, size=w[name].data.shape).astype(np.float32)


def main():
    index = []
    for name, skw, nkw, mcs_idx, n_slots, n0, bias, squeeze in CASES:
        cfg = SlotConfig(**skw)
        nkw = dict(nkw)
        supported = nkw.pop("supported")
        variant = nkw.pop("variant")
        config = nrx.NrxConfig.from_table(TABLE, supported, variant=variant, **nkw)
        w = nrx.init_weights(config, seed=7)
        if bias:
            perturb(w)
        mcs = tuple(TABLE[i] for i in mcs_idx)
        y, books, bits = synth_slots(cfg, mcs, n_slots, n0, seed=len(index) + 1)
        n0_arg = n0 if n_slots == 1 else np.linspace(n0, 2 * n0, n_slots)
        if squeeze:
            y_in, books_in = y[0], books[0]
        else:
            y_in, books_in = y, books
        llrs, chest = nrx.nrx_forward(y_in, books_in, cfg, mcs, w, config, n0_arg)
        n0_vec = np.full(n_slots, n0, dtype=np.float64) if np.isscalar(n0_arg) else np.asarray(n0_arg)
        feats = nrx.assemble_features(y, nrx.ls_features(y, books, cfg), n0_vec, cfg, config)
        meta = dict(name=name, slot=config_dict(cfg), nrx=config_dict(config),
                    mcs=[[m.index, m.modulation_order, m.code_rate] for m in mcs],
                    squeeze=squeeze, n0_scalar=bool(np.isscalar(n0_arg)))
        arrays = {"meta": np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8),
                  "y": y, "pilots": np.stack([b.values for b in books]), "n0": n0_vec,
                  "features": feats, "chest": chest}
        for u, l in enumerate(llrs):
            arrays[f"llr{u}"] = l
        for k, t in w.items():
            arrays[f"w:{k}"] = t.data
        for u in range(cfg.num_ues):
            arrays[f"bits{u}"] = np.stack([b[u] for b in bits])
        path = os.path.join(OUT, f"{name}.npz")
        np.savez_compressed(path, **arrays)
        index.append(name)
        print(f"{name}: y{y.shape} llr widths {[l.shape[-1] for l in llrs]} -> {os.path.getsize(path)} B")
    with open(os.path.join(OUT, "index.json"), "w") as fh:
        json.dump(index, fh, indent=1)


if __name__ == "__main__":
    main()
