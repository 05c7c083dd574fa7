"""Golden vectors for the GPU slot generator, made by the REFERENCE itself.

Run in the build container (where the read-only reference lives):

    PYTHONPATH=/root/reference/pkg/src python -B tests/golden/make_golden_slotgen.py

Per case it runs the reference's own transmitter and channel on the uncoded
recipe of make_golden.py (generate_pilots, Constellation.map_bits on the data
REs, beamform, TdlChannelSource.sample, apply_channel,
ChannelRealization.effective) and stores the received grids, effective
channels, transmitted labels and pilot values, plus the variates the
reference drew (re-drawn here with the same numpy generators and seeds) and
the profiles' declared taps.  Nothing here is needed on the GPU box.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
REF = os.environ.get("NRX_REFERENCE_SRC", "/root/reference/pkg/src")
if REF not in sys.path:
    sys.path.insert(0, REF)

from nrxsim import channel as ch  # noqa: E402
from nrxsim.constellation import build_constellation  # noqa: E402
from nrxsim.slot import SlotConfig, beamform, generate_pilots  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

CASES = [
    dict(name="sg_desk", slot=dict(num_subcarriers=48, num_ues=2), orders=(4, 4),
         profiles=("tdl_b", "tdl_c"), n0=0.1, n_slots=3, seed=3),
    dict(name="sg_mixed", slot=dict(num_subcarriers=60, num_ues=2), orders=(2, 6),
         profiles=("tdl_a", "tdl_d"), n0=0.05, n_slots=2, seed=5),
    dict(name="sg_u3_comb4", slot=dict(num_subcarriers=40, num_ues=3, comb_size=4, ue_antennas=1,
                                       pilot_symbols=(3,)),
         orders=(2, 4, 6), profiles=("tdl_b", "tdl_c", "tdl_a"), n0=0.3, n_slots=2, seed=8),
    dict(name="sg_beam_noiseless", slot=dict(num_subcarriers=36, num_ues=1, bs_antennas=2,
                                             beams=((0.6, 0.8j),)),
         orders=(4,), profiles=("tdl_b",), doppler0=True, n0=0.0, n_slots=2, seed=9),
    dict(name="sg_b8_t7", slot=dict(num_subcarriers=30, num_symbols=7, pilot_symbols=(1, 5), bs_antennas=8,
                                    num_ues=2),
         orders=(6, 2), profiles=("tdl_c", "tdl_b"), n0=1.0, n_slots=2, seed=12),
]


def run_case(c):
    cfg = SlotConfig(**c["slot"])
    profiles = [ch.PROFILES[p]() for p in c["profiles"]]
    if c.get("doppler0"):
        profiles = [p.with_doppler(0.0) for p in profiles]
    U, S, T, B, Nu = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, cfg.bs_antennas, cfg.ue_antennas
    L, NS = max(p.delays_s.size for p in profiles), ch.NUM_SINUSOIDS
    F, K = -(-S // cfg.comb_size), len(cfg.pilot_symbols)
    s_idx, t_idx = cfg.data_re_indices()
    n, seed = c["n_slots"], c["seed"]
    out = dict(y=np.zeros((n, S, T, B), complex), h_eff=np.zeros((n, U, S, T, B), complex),
               labels=np.zeros((n, U, S, T), np.uint8), pilots=np.zeros((n, U, F, K), complex),
               angles=np.zeros((n, U, B, Nu, L, NS)), phases=np.zeros((n, U, B, Nu, L, NS)),
               noise=np.zeros((n, S, T, B), complex))
    for i in range(n):
        book = generate_pilots(cfg, slot_seed=seed * 1000 + i)
        rng = np.random.default_rng((seed, i))
        antennas = []
        for u in range(U):
            m = c["orders"][u]
            bits = (rng.random((s_idx.size, m)) < 0.5).astype(np.uint8)
            sym = np.array(book.values[u])
            sym[s_idx, t_idx] = build_constellation(m).map_bits(bits)
            antennas.append(beamform(sym, cfg.beam_matrix[u]))
            out["labels"][i, u, s_idx, t_idx] = bits.astype(np.int64) @ (1 << np.arange(m - 1, -1, -1))
            sc = cfg.comb_subcarriers(u)
            out["pilots"][i, u, :sc.size] = book.values[u][np.ix_(sc, list(cfg.pilot_symbols))]
        h = ch.TdlChannelSource(profiles).sample(cfg, (seed, i))
        real = ch.ChannelRealization(h=h, n0=c["n0"])
        state = rng.bit_generator.state
        out["y"][i] = ch.apply_channel(np.stack(antennas), real, rng)
        out["h_eff"][i] = real.effective(cfg)
        # the variates the reference consumed, re-drawn with the same generators
        rng.bit_generator.state = state
        re = rng.standard_normal((S, T, B))
        out["noise"][i] = re + 1j * rng.standard_normal((S, T, B))
        for u in range(U):
            r = np.random.default_rng((seed, i, u))
            nt = profiles[u].delays_s.size
            out["angles"][i, u, :, :, :nt] = r.uniform(0.0, 2.0 * np.pi, size=(B, Nu, nt, NS))
            out["phases"][i, u, :, :, :nt] = r.uniform(0.0, 2.0 * np.pi, size=(B, Nu, nt, NS))
    for u, p in enumerate(profiles):
        out[f"delays_{u}"] = p.delays_s
        out[f"powers_{u}"] = p.powers
    for m in (2, 4, 6):
        out[f"qam_{m}"] = build_constellation(m).points
    meta = dict(name=c["name"], slot=c["slot"], orders=list(c["orders"]), profiles=list(c["profiles"]),
                doppler=[p.doppler_hz for p in profiles], n0=c["n0"], n_slots=n, seed=seed)
    return out, meta


def main():
    index = []
    for c in CASES:
        arrays, meta = run_case(c)
        np.savez_compressed(os.path.join(OUT, f"{c['name']}.npz"), **arrays)
        index.append(meta)
        print(c["name"], {k: v.shape for k, v in arrays.items() if k in ("y", "h_eff")})
    with open(os.path.join(OUT, "slotgen_index.json"), "w") as f:
        json.dump(index, f, indent=1, default=lambda o: o if not isinstance(o, complex) else [o.real, o.imag])


if __name__ == "__main__":
    main()
