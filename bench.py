#!/usr/bin/env python
"""Benchmark of the B200 NRX forward pass (the path BASELINE.json names).

Workload (BASELINE.json configs[1] geometry, batched as configs[4]): slots of
273 PRB (S=3276 subcarriers) x 14 symbols, 2 UEs (16-QAM), 4 RX antennas,
the real-time NRX (d_s=56, N_it=2, 137,156 random-init weights).  A "step"
is one batched forward over --slots-per-step independent slots per GPU with
inputs resident in HBM; ranks shard independent slots (weak scaling, no
data-path collective).  The JSON line also carries the single-slot latency
p50/p99 (device-resident, CUDA graph), the end-to-end number through the
public host API (pinned H2D of inputs + D2H of LLRs/chest inside the timed
region), the roofline of the dominant kernel, and the reference CPU path
timed on this host.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

S_C2, U_C2, D_S, N_IT = 3276, 2, 56, 2
DATA = ("synthetic: GPU slot generator on the SURVEY §8d recipe (doubletdl TDL-B/TDL-C Jakes fading, Gray "
        "16-QAM, per-slot QPSK pilots, AWGN n0=0.1); random-init weights")
METRIC = "NRX forward slots/s at 273 PRB (2 UE, 4 RX, RT d_s=56 N_it=2); p50/p99 single-slot latency in latency_us"


DTYPES = {"fp32": "fp32", "fp32_simt": "fp32", "bf16": "bf16", "fp16": "fp16"}
PRECISION_NOTES = {
    "fp32": "fp32x3: every fp32 operand split into fp16 hi + lo (22 significant bits); per K step two tcgen05 "
            "kind::f16 MMAs (hi and lo planes) against [W_hi | W_lo] (all four products) into fp32 TMEM "
            "accumulators; parity gate max|dLLR| <= 1e-5 max|LLR_ref| (the reference's fp32 gate)",
    "fp32_simt": "fp32 FFMA (SIMT), fp64 LS and sum of others; same gate",
    "bf16": "bf16 operands on tcgen05, fp32 accumulate, fp32 residual stream; gate 2e-2 (max) / 5e-3 (p99)",
    "fp16": "fp16 operands on tcgen05, fp32 accumulate; gate 5e-3 (max) / 1.5e-3 (p99)"}


def c2_setup():
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, default_mcs_table, init_weights
    table = default_mcs_table()
    cfg = SlotConfig(num_subcarriers=S_C2, num_ues=U_C2, comb_size=2)
    config = NrxConfig.from_table(table, (14,), variant="single", d_s=D_S, num_iterations=N_IT)
    return cfg, config, init_weights(config, seed=0), (table[14], table[14])


def gpu_batch(cfg, n_slots: int, dev, seed: int = 0, first_slot: int = 0):
    """(y c64 (N,S,T,B), pilots c64 (N,U,F,K), noise feature (N,), mods (N*U,))
    device tensors of n_slots distinct slots from the GPU slot generator, on
    the SURVEY.md §8d recipe: doubletdl channels (UE0 TDL-B 400 Hz / 100 ns,
    UE1 TDL-C 100 Hz / 300 ns, 32-sinusoid Jakes fading, 4 RX x 2 TX with the
    default beams), Gray 16-QAM on every data RE, per-slot QPSK pilots on
    each UE's comb, AWGN at n0 = 0.1 (SNR 10 dB)."""
    import torch
    from paper_2409_02912_b200.nrx import noise_features
    from paper_2409_02912_b200.slotgen import GpuSlotSource
    src = GpuSlotSource(cfg, device=dev)
    b = src.generate(n_slots, [4] * cfg.num_ues, 0.1, seed=seed, first_slot=first_slot)
    nf = torch.from_numpy(noise_features(0.1, n_slots)).to(dev)
    torch.cuda.synchronize(dev)
    return b.y, b.pilots, nf, b.mod_order


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, period_ms: int = 50):
        self.gpu = gpu_index
        self.period_ms = period_ms
        self.samples = []
        self._proc = None
        self._lines = []
        self._start = 0

    def _read(self):
        for line in self._proc.stdout:
            if line.strip():
                self._lines.append(line)

    def __enter__(self):
        # one long-running nvidia-smi polling at period_ms (spawning per sample is too slow);
        # the timed region starts once its first sample has arrived, and only the samples
        # taken from then until the region ends are kept
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period_ms)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self._proc = None
        t0 = time.time()
        while self._proc is not None and not self._lines and time.time() - t0 < 10:
            time.sleep(0.01)
        self._start = len(self._lines)
        return self

    def __exit__(self, *exc):
        if self._proc is not None:
            t0 = time.time()   # a region shorter than one period still gets the next sample
            while len(self._lines) <= self._start and time.time() - t0 < 2:
                time.sleep(0.01)
            lines = self._lines[self._start:]
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
            self.samples = [[x.strip() for x in line.split(",")] for line in lines]
        return False

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        pw = [float(s[3]) for s in self.samples if len(s) > 3 and s[3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 5 + i and s[5 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w": float(np.median(pw)) if pw else None}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def conv_update0_flops_per_slab_re(d=D_S, k=3):
    return 2 * k * k * (2 * d + 2) * d


def executed_flops(precision, B, S=S_C2, U=U_C2, T=14, d=D_S):
    """Tensor-core FLOPs update.conv0 actually issues per launch (padded
    shapes: 128-row tiles over S*(T+1) rows; K per tap = 2d with the
    positional channels folded out of the GEMM (upd0_posf: fp32x3, d = 16 / 56),
    else rup(d+2, 16) + rup(d, 16); N = rup(d, 16);
    fp32x3: two planes x N = 2 x3_np(d) per tap and K step; fp32_simt: none)."""
    if precision == "fp32_simt":
        return 0
    rup = lambda a, m: -(-a // m) * m  # noqa: E731
    rows = rup(S * (T + 1), 128)
    posf = precision == "fp32" and d in (16, 56)
    K = 2 * d if posf else rup(d + 2, 16) + rup(d, 16)
    if precision == "fp32":
        npx = 56 if rup(d, 8) == 56 else rup(d, 16)
        return 2 * rows * U * B * 9 * K * 2 * (2 * npx)
    return 2 * rows * U * B * 9 * K * rup(d, 16)


def algorithmic_flops_per_slab_re(d=D_S, h=D_S, n_it=N_IT, m=4, B=4, cin=19, k=3):
    """MAC = 9 Cin d + 9 d^2 + N_it (2 d h + 9 (2d+2) d + 9 d^2) + (d h + h m) + (d h + h 2B)."""
    kk = k * k
    mac = kk * cin * d + kk * d * d + n_it * (2 * d * h + kk * (2 * d + 2) * d + kk * d * d) \
        + (d * h + h * m) + (d * h + h * 2 * B)
    return 2 * mac


def traffic_from_profiles(kernel: str, precision: str, slots: int):
    """DRAM bytes (read + write) per launch of `kernel` at `slots` slots per
    launch, scaled from the committed ncu --set full capture (profiles/traffic.json)."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)[precision][kernel]
        return int(t["dram_bytes_per_slot"] * slots)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# reference arm: the unmodified reference nrx_forward on this host's CPUs
# ---------------------------------------------------------------------------


def reference_impl():
    """(nrx_forward, kind): oracle/_ref (pip-installed reference) or the oracle port."""
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "nrxsim")):
        sys.path.insert(0, ref_dir)
        from nrxsim.nrx import nrx_forward
        return nrx_forward, "reference"
    from oracle.nrx_oracle import nrx_forward
    return nrx_forward, "port"


def reference_recipe_slots(cfg, n: int, seed: int = 11):
    """Host slots of the same SURVEY §8d recipe the GPU arm generates
    (doubletdl, 16-QAM, per-slot pilots, n0 = 0.1), built from the reference
    recipe's numpy variates by the CPU generator oracle."""
    from oracle import slotgen_oracle as so
    from paper_2409_02912_b200.config import PilotBook
    from paper_2409_02912_b200.slotgen import doubletdl, reference_variates
    prof = doubletdl()
    v = reference_variates(cfg, prof, (4, 4), range(n), seed=seed)
    ys, books = [], []
    for i in range(n):
        y, _ = so.synth_slot(cfg, prof, (4, 4), 0.1, v["angles"][i], v["phases"][i], v["labels"][i],
                             v["noise"][i], v["pilots"][i])
        vals = np.zeros((cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols), complex)
        for u in range(cfg.num_ues):
            sc = np.arange(u % cfg.comb_size, cfg.num_subcarriers, cfg.comb_size)
            vals[u][np.ix_(sc, list(cfg.pilot_symbols))] = v["pilots"][i, u, :sc.size]
        ys.append(y)
        books.append(PilotBook(values=vals, config=cfg))
    return np.stack(ys), books


def run_reference(args, slots: int, warmup: int):
    """Time the reference CPU path: one slot per call (latency_bench style,
    evaluation.py:341-349) -> slots/s."""
    fwd, kind = reference_impl()
    cfg, config, w, mcs = c2_setup()
    y, books = reference_recipe_slots(cfg, min(slots, 2))
    if kind == "reference":
        # the reference's own types (its isinstance checks need them) and
        # weights as recorded autodiff tensors, exactly as cli.cmd_bench builds them
        import dataclasses
        from nrxsim import autodiff as ad
        from nrxsim import nrx as rnrx
        from nrxsim import slot as rslot
        cfg = rslot.SlotConfig(**{f.name: getattr(cfg, f.name) for f in dataclasses.fields(rslot.SlotConfig)})
        config = rnrx.NrxConfig(**{f.name: getattr(config, f.name) for f in dataclasses.fields(rnrx.NrxConfig)})
        mcs = tuple(rslot.McsEntry(m.index, m.modulation_order, m.code_rate) for m in mcs)
        books = [rslot.PilotBook(values=b.values, config=cfg) for b in books]
        w = {k: ad.Tensor(v, requires_grad=True) for k, v in w.items()}
    for i in range(warmup):
        fwd(y[i % len(y)], books[i % len(y)], cfg, mcs, w, config, 0.1)
    times = []
    for i in range(slots):
        t0 = time.perf_counter()
        fwd(y[i % len(y)], books[i % len(y)], cfg, mcs, w, config, 0.1)
        times.append(time.perf_counter() - t0)
    times = np.asarray(times)
    return {"value": float(1.0 / times.mean()), "unit": "slots/s", "kind": kind,
            "cores": int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1)),
            "p50_ms": float(np.median(times) * 1e3), "p99_ms": float(np.percentile(times, 99) * 1e3),
            "sample": f"{slots} single-slot nrx_forward calls at C2 (273 PRB, 2 UE, d_s=56, N_it=2) after {warmup} warm-up"}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_subprocess(slots=5, warmup=1, threads=None):
    """Run the reference arm in a child process so OpenBLAS gets all cores
    (or `threads`); >= 1 warm-up, >= 5 runs at 273 PRB."""
    env = dict(os.environ)
    env["OPENBLAS_NUM_THREADS"] = str(threads or os.cpu_count() or 1)
    env.pop("WORLD_SIZE", None); env.pop("RANK", None); env.pop("LOCAL_RANK", None)
    cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--cpu-json",
           "--steps", str(slots), "--warmup", str(warmup)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900).stdout
        res = json.loads(out.strip().splitlines()[-1])
        res["cpu_model"] = cpu_model()
        return res
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "slots/s", "kind": "unavailable", "cores": os.cpu_count(),
                "sample": f"failed: {e!r}"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2409_02912_b200 import _lib
    from paper_2409_02912_b200.engine import NrxEngine
    from paper_2409_02912_b200.shard import max_over_ranks

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    cfg, config, w, mcs = c2_setup()
    eng = NrxEngine(config, w, precision=args.precision, device=dev)
    B = args.slots_per_step
    U, S, T, BR = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, config.num_rx_ant

    # two device-resident input sets, alternated so consecutive steps never
    # re-read the same inputs from L2 (per-step activations are GBs anyway)
    sets = [gpu_batch(cfg, B, dev, seed=1, first_slot=(2 * rank + s) * B) for s in range(2)]
    llr = torch.empty((B, U, S, T, 4), dtype=torch.float32, device=dev)
    chest = torch.empty((B, U, S, T, BR), dtype=torch.complex64, device=dev)
    stream = torch.cuda.current_stream(dev)
    ws = eng.workspace(cfg, B)

    def step(i):
        y, pil, nf, mods = sets[i & 1]
        eng.forward_device(cfg, y, pil, nf, mods, N_IT, llr, chest, workspace=ws, stream=stream)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler, _lib.KernelTimer(("conv_update0", "ls_feat"), max_records=4 * args.steps * N_IT + 16) as kt:
        e0.record(stream)
        for i in range(args.steps):
            step(i)
        e1.record(stream)
        torch.cuda.synchronize()
        kt_rec = kt.collect()
        kernel_ms = kt_rec.get("conv_update0", [])
        lsfeat_ms = kt_rec.get("ls_feat", [])
    elapsed = e0.elapsed_time(e1) / 1e3
    if world > 1:
        t = torch.tensor([elapsed], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
        dist.barrier()
    torch.cuda.synchronize()
    slots_total = B * args.steps * world
    value = slots_total / elapsed
    ms_per_step = elapsed / args.steps * 1e3

    # N > 1: the same step followed by the gather of its LLRs to rank 0 over
    # NCCL (SURVEY.md §8e "with gather"); compute-only stays the headline value
    with_gather = None
    if world > 1:
        from paper_2409_02912_b200.shard import StepGather
        gat = StepGather(llr)
        n_g = max(5, args.steps // 4)
        dist.barrier()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for i in range(n_g):
            step(i)
            gat(llr)
        g1.record(stream)
        torch.cuda.synchronize()
        tg = max_over_ranks(g0.elapsed_time(g1) / 1e3, dev)
        with_gather = {"value": round(B * n_g * world / tg, 2), "unit": "slots/s", "steps": n_g,
                       "gather_bytes_per_step_into_rank0": gat.bytes_per_step(llr),
                       "note": "each step's (B,U,S,T,4) float32 LLRs of every rank gathered to rank 0 (NCCL)"}

    # roofline of the dominant kernel (conv_update0), device time of each launch
    peaks, peak_src = load_peaks()
    flops_launch = conv_update0_flops_per_slab_re() * B * U * S * T
    kavg = float(np.mean(kernel_ms)) / 1e3 if kernel_ms else float("nan")
    achieved = flops_launch / kavg / 1e12
    if args.precision in ("bf16", "fp16"):  # same tcgen05 kind::f16 rate for both
        peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
        peak_note = f"bf16 dense, sustained ({peak_src}); fp16 runs at the same tensor rate"
    elif args.precision == "fp32":
        # fp32x3: a two-piece fp16 split needs at least three fp16 MACs per fp32 MAC (hi*Whi, hi*Wlo,
        # lo*Whi); the kernel issues four (two N = 2 np MMAs on [W_hi | W_lo]), i.e. runs at most at
        # bf16 / 4 -- the conservative / 3 ceiling is the one reported as `peak`
        peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")) / 3.0
        peak_note = (f"fp32-equivalent tensor-core ceiling = bf16 dense sustained ({peak_src}) / 3 (the minimum "
                     "of three fp16 MACs per fp32 MAC for a two-piece split); the kernel issues four "
                     "(hi and lo planes x [W_hi | W_lo]): its executed tensor rate is executed_tensor_tflops, "
                     "compared with the measured bf16 sustained GEMM in executed_vs_bf16_sustained")
    else:
        sm_mhz = peaks.get("sm_max_mhz", 1965.0)
        peak = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12
        peak_note = "fp32 FFMA nominal (148 SM x 128 lanes x 2 x max clock)"
    traffic = traffic_from_profiles("conv_update0", args.precision, B)
    lsfeat = lsfeat_bandwidth(lsfeat_ms, B, cfg, config, args.precision, peaks, peak_src)

    # single-slot latency (device resident), CUDA graph of the whole forward
    lat = latency_single_slot(eng, cfg, dev, args.latency_runs) if rank == 0 else None
    lat_other = other_config_latencies(args.precision, dev, max(100, args.latency_runs // 4)) \
        if rank == 0 and not args.no_precision_sweep else None

    # end to end through the public host API: pinned H2D + D2H inside the region
    e2e = e2e_throughput(eng, cfg, B, max(4, args.steps // 2), world, dev)

    # Monte-Carlo pipeline: GPU slot generation -> receiver -> bit-error count
    mc = monte_carlo_pipeline(eng, cfg, B, max(5, args.steps // 4), world, rank, dev)
    # the other §8(f) rows on the same slots: LDPC decode / encode, classical baselines
    nxt = next_rows(cfg, B, dev) if rank == 0 and not args.no_precision_sweep else None

    # the C5 job: 4096 independent slots, contiguous shards per rank
    c5 = c5_job(eng, cfg, args.c5_slots, B, world, rank, dev) if args.c5_slots > 0 else None

    # the other precisions on the same device-resident workload (shorter runs)
    by_prec = {args.precision: {"slots_per_s": round(value, 2), "ms_per_step": round(ms_per_step, 4),
                                "latency_us": {k: lat[k] for k in ("p50", "p99")} if lat else None}}
    if not args.no_precision_sweep:
        for prec in ("fp32", "fp32_simt", "bf16", "fp16"):
            if prec == args.precision:
                continue
            other = NrxEngine(config, w, precision=prec, device=dev)
            ows = other.workspace(cfg, B)

            def ostep(i, other=other, ows=ows):
                y, pil, nf, mods = sets[i & 1]
                other.forward_device(cfg, y, pil, nf, mods, N_IT, llr, chest, workspace=ows, stream=stream)

            n_steps = max(3, args.steps // (10 if prec == "fp32_simt" else 4))
            for i in range(3):
                ostep(i)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for i in range(n_steps):
                ostep(i)
            b.record(stream)
            torch.cuda.synchronize()
            t = max_over_ranks(a.elapsed_time(b) / 1e3, dev)
            by_prec[prec] = {"slots_per_s": round(B * n_steps * world / t, 2),
                             "ms_per_step": round(t / n_steps * 1e3, 4), "steps": n_steps}
            if rank == 0:
                ol = latency_single_slot(other, cfg, dev, max(200, args.latency_runs // 10))
                by_prec[prec]["latency_us"] = {k: ol[k] for k in ("p50", "p99")}
            del other, ows
            torch.cuda.empty_cache()

    n_launch = eng.launch_count(cfg, N_IT)
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": "slots/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": DTYPES[args.precision], "data": DATA,
        "precision_note": PRECISION_NOTES[args.precision],
        "config": {"workload": f"C5-style batches of C2 slots: {B} slots/GPU/step of 273 PRB x 14 sym, "
                               f"2 UE 16-QAM, 4 RX; RT NRX d_s=56 N_it=2 (configs[1] geometry)",
                   "slots_per_step_per_gpu": B, "precision": args.precision,
                   "l2": "inputs alternate between two device buffers (188 MB) and per-step activations "
                         "are > 1 GB, i.e. far larger than the 126 MB L2"},
        "latency_us": lat,
        "latency_other_configs_us": lat_other,
        "e2e": e2e,
        "with_gather": with_gather,
        "monte_carlo": mc,
        "next_rows": nxt,
        "roofline": {"kernel": "conv_update0 (iteration.update.conv0, 3x3 114->56, implicit GEMM)",
                     "bound": "tensor", "achieved": round(achieved, 2), "peak": round(peak, 1),
                     "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "peak_source": peak_note,
                     "algorithmic_flops_per_launch": flops_launch,
                     "avg_launch_ms": round(kavg * 1e3, 4), "launches_timed": len(kernel_ms),
                     "executed_tensor_tflops": round(executed_flops(args.precision, B) / kavg / 1e12, 1)
                     if kernel_ms else None,
                     "executed_vs_bf16_sustained": round(executed_flops(args.precision, B) / kavg / 1e12
                                                         / peaks.get("bf16_tflops_sustained", 1375.3), 4)
                     if kernel_ms and args.precision != "fp32_simt" else None,
                     "executed_vs_clock_peak": (
                         round(executed_flops(args.precision, B) / kavg
                               / (148 * 8192 * sampler.summary()["sm_mhz"] * 1e6), 4)
                         if kernel_ms and args.precision != "fp32_simt" and sampler.summary()["sm_mhz"] else None),
                     "clock_peak_note": "dense fp16 tensor rate at the timed region's median SM clock: 148 SMs x "
                                        "8192 FLOP/cycle (one 128x112x16 MMA per 56 cycles per SM, the floor "
                                        "update.conv0 reaches)",
                     "share_of_step": round(kavg * 1e3 * N_IT / ms_per_step, 4) if kernel_ms else None},
        "whole_path": {"algorithmic_tflops": round(algorithmic_flops_per_slab_re() * U * S * T * value / world / 1e12, 2),
                       "flop_per_slot": algorithmic_flops_per_slab_re() * U * S * T},
        "memory_bound_stage": lsfeat,
        "c5_job": c5,
        "by_precision": by_prec,
        "gpu_launches": n_launch * args.steps,
        "launches_per_step": n_launch,
        "clocks": sampler.summary(),
    }
    if rank == 0 and world == 1 and not args.no_precision_sweep:
        out["dropin_single_slot"] = dropin_latency(cfg, config, w, mcs)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_subprocess()
        one = cpu_baseline_subprocess(slots=2, warmup=1, threads=1)
        out["cpu_baseline"]["single_thread"] = {k: one.get(k) for k in ("value", "p50_ms", "cores", "sample")}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def lsfeat_bandwidth(ms_list, B, cfg, config, precision, peaks, peak_src):
    """Achieved HBM bandwidth of K1 (LS + feature assembly, the HBM-bound stage
    SURVEY §8d names): bytes it moves per launch / its device time."""
    if not ms_list:
        return None
    from paper_2409_02912_b200 import _lib
    geo = _lib.buffer_geometry(config, cfg, precision)
    U, S, T, BR = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, config.num_rx_ant
    F = -(-S // cfg.comb_size)
    y_bytes = B * S * T * BR * 8
    pil_bytes = B * U * F * len(cfg.pilot_symbols) * 8
    planes = 2 if precision == "fp32" else 1
    esz = 4 if precision == "fp32_simt" else 2
    written = B * U * geo["rows_slab"] * geo["Cf"] * esz * planes     # every row and channel of the buffer
    cin = 4 * BR + 2 + int(bool(config.include_noise_plane))
    alg = y_bytes + pil_bytes + B * U * S * T * cin * esz * planes   # y + pilots + C_in features
    t = float(np.mean(ms_list)) / 1e3
    peak = peaks.get("hbm_gbs", 6450.0)
    return {"kernel": "ls_feat (LS + feature assembly, K1)", "bound": "hbm", "avg_launch_ms": round(t * 1e3, 4),
            "bytes_moved_per_launch": int(y_bytes + pil_bytes + written), "algorithmic_bytes_per_launch": int(alg),
            "achieved_gbs": round((y_bytes + pil_bytes + written) / t / 1e9, 1),
            "algorithmic_gbs": round(alg / t / 1e9, 1), "peak_gbs": peak,
            "frac": round((y_bytes + pil_bytes + written) / t / 1e9 / peak, 4),
            "peak_source": f"measured HBM copy bandwidth ({peak_src})", "launches_timed": len(ms_list)}


def c5_job(eng, cfg, total, B, world, rank, dev):
    """BASELINE.json configs[4] / SURVEY §8e: `total` independent C2 slots,
    contiguous shards (slot i -> rank floor(i world / total)), every slot
    distinct (GPU generator keyed by the global slot index) and pre-staged in
    HBM; each rank runs its shard in batches of B.  Timed compute-only and
    with the gather of every batch's LLRs to rank 0 (NCCL over NVLink), on
    the device, max over ranks."""
    import torch
    from paper_2409_02912_b200.shard import StepGather, max_over_ranks, shard_slots
    shard = shard_slots(total, rank, world)
    U, S, T = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols
    batches = []
    for b0 in range(shard.start, shard.stop, B):
        nb = min(B, shard.stop - b0)
        batches.append(gpu_batch(cfg, nb, dev, seed=4096, first_slot=b0))
    llr = torch.empty((B, U, S, T, 4), dtype=torch.float32, device=dev)
    chest = torch.empty((B, U, S, T, 4), dtype=torch.complex64, device=dev)
    ws = eng.workspace(cfg, B)
    st = torch.cuda.current_stream(dev)
    gat = StepGather(llr) if world > 1 else None

    def run(gather):
        for y, pil, nf, mods in batches:
            nb = y.shape[0]
            eng.forward_device(cfg, y, pil, nf, mods, N_IT, llr[:nb], chest[:nb], workspace=ws, stream=st)
            if gather and gat is not None:
                gat(llr)

    out = {"total_slots": total, "slots_this_rank": len(shard), "batches_per_rank": len(batches),
           "batch_slots": B}
    run(False)  # warm-up (also the NCCL communicator)
    if gat is not None:
        run(True)
    for name, gather in (("compute_only", False), ("with_gather", True)):
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        run(gather)
        b.record(st)
        torch.cuda.synchronize()
        t = max_over_ranks(a.elapsed_time(b) / 1e3, dev)
        out[name] = {"job_s": round(t, 5), "slots_per_s": round(total / t, 1)}
    out["gather_bytes_into_rank0"] = int(llr.numel() * llr.element_size() * len(batches) * max(0, world - 1))
    out["note"] = ("inputs generated on each rank's GPU before timing; with_gather adds NCCL gathers of every "
                   "batch's (B,U,S,T,4) float32 LLRs into rank 0 (at N=1 rank 0 already holds them)")
    del batches
    torch.cuda.empty_cache()
    return out


def latency_single_slot(eng, cfg, dev, runs: int, n_it: int = N_IT, orders=None, width: int = 4,
                        note: str = "one C2 slot"):
    import torch
    y, pil, nf, mods = gpu_batch(cfg, 1, dev, seed=7)
    if orders is not None:
        mods = torch.tensor(orders, dtype=torch.int32, device=dev)
    llr = torch.empty((1, cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, width), dtype=torch.float32,
                      device=dev)
    chest = torch.empty((1, cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols, 4), dtype=torch.complex64, device=dev)
    ws = torch.empty_like(eng.workspace(cfg, 1))
    side = torch.cuda.Stream(dev)
    mode = "cuda_graph"
    with torch.cuda.stream(side):
        for _ in range(3):
            eng.forward_device(cfg, y, pil, nf, mods, n_it, llr, chest, workspace=ws, stream=side)
    side.synchronize()
    try:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            eng.forward_device(cfg, y, pil, nf, mods, n_it, llr, chest, workspace=ws, stream=side)
        run = g.replay
    except Exception:
        mode = "stream"

        def run():
            eng.forward_device(cfg, y, pil, nf, mods, n_it, llr, chest, workspace=ws,
                               stream=torch.cuda.current_stream(dev))
    for _ in range(20):
        run()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(runs)]
    cur = torch.cuda.current_stream(dev)
    for a, b in ev:
        a.record(cur)
        run()
        b.record(cur)
    torch.cuda.synchronize()
    us = np.array([a.elapsed_time(b) * 1e3 for a, b in ev])
    return {"p50": round(float(np.median(us)), 2), "p99": round(float(np.percentile(us, 99)), 2),
            "min": round(float(us.min()), 2), "runs": runs, "mode": mode,
            "note": f"{note}, device-resident inputs (no host copies), back-to-back launches"}


def other_config_latencies(precision, dev, runs: int):
    """Single-slot latency of BASELINE.json configs[0], [2], [3] (C1 24 PRB /
    1 UE; C3 dynamic MCS QPSK + 256-QAM extension through the masked readout;
    C4 large N_it = 8 with the affine depth fit, evaluation.py:351-363)."""
    from paper_2409_02912_b200.config import NrxConfig, SlotConfig, extended_mcs_table, init_weights
    from paper_2409_02912_b200.engine import NrxEngine
    t = extended_mcs_table()
    out = {}
    cfg1 = SlotConfig(num_subcarriers=288, num_ues=1, comb_size=2)
    c1 = NrxConfig.from_table(t, (14,), d_s=56, num_iterations=2)
    out["C1_24prb_1ue"] = latency_single_slot(NrxEngine(c1, init_weights(c1, 0), precision, dev), cfg1, dev, runs,
                                              note="C1 slot (24 PRB, 1 UE, RT d_s=56 N_it=2)")
    for d, n in ((16, 2), (16, 4)):  # the desk models of configs[0] (configio.py:43-50)
        cd = NrxConfig.from_table(t, (14,), d_s=d, num_iterations=n)
        out[f"C1_24prb_1ue_d{d}_it{n}"] = latency_single_slot(
            NrxEngine(cd, init_weights(cd, 0), precision, dev), cfg1, dev, runs, n_it=n,
            note=f"C1 slot (24 PRB, 1 UE, desk d_s={d} N_it={n})")
    cfg = SlotConfig(num_subcarriers=S_C2, num_ues=2, comb_size=2)
    c3 = NrxConfig.from_table(t, (9, 14, 19, 27), variant="masking", d_s=56, num_iterations=2)
    out["C3_mixed_qpsk_256qam"] = latency_single_slot(
        NrxEngine(c3, init_weights(c3, 0), precision, dev), cfg, dev, runs, orders=[2, 8], width=8,
        note="C3 slot (273 PRB, UE0 QPSK + UE1 256-QAM ext., masking m_max=8)")
    cv = NrxConfig.from_table(t, (9, 14, 19), variant="var_io", d_s=56, num_iterations=2)
    out["C3_var_io_qpsk_64qam"] = latency_single_slot(
        NrxEngine(cv, init_weights(cv, 0), precision, dev), cfg, dev, runs, orders=[2, 6], width=6,
        note="C3 slot (273 PRB, UE0 QPSK + UE1 64-QAM, var_io: per-order input / output weight sets)")
    c4 = NrxConfig.from_table(t, (14,), d_s=56, num_iterations=8)
    e4 = NrxEngine(c4, init_weights(c4, 0), precision, dev)
    depth = {}
    for n in (1, 2, 4, 8):
        depth[n] = latency_single_slot(e4, cfg, dev, max(50, runs // 4), n_it=n,
                                       note=f"C4 slot (273 PRB, 2 UE, large d_s=56) at depth {n}")
    xs = np.array(list(depth))
    ys = np.array([depth[n]["p50"] for n in depth])
    b, a = np.polyfit(xs, ys, 1)
    out["C4_large_nit8"] = dict(depth[8], depth_p50_us={int(k): v["p50"] for k, v in depth.items()},
                                affine_fit_us={"overhead": round(float(a), 2), "per_iteration": round(float(b), 2)})
    return out


def monte_carlo_pipeline(eng, cfg, B, steps, world, rank, dev):
    """Slots/s of (a) the GPU slot generator alone and (b) the uncoded
    Monte-Carlo step generate -> nrx_forward -> count_bit_errors, all on the
    device, B distinct slots per step (the reference builds one such slot on
    the host in 48.6 ms)."""
    import torch
    from paper_2409_02912_b200.nrx import noise_features
    from paper_2409_02912_b200.shard import max_over_ranks
    from paper_2409_02912_b200.slotgen import GpuSlotSource, count_bit_errors
    U, S, T = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols
    src = GpuSlotSource(cfg, device=dev)
    mods = torch.full((B * U,), 4, dtype=torch.int32, device=dev)
    n0 = torch.full((B,), 0.1, dtype=torch.float64, device=dev)
    nf = torch.from_numpy(noise_features(0.1, B)).to(dev)
    llr = torch.empty((B, U, S, T, 4), dtype=torch.float32, device=dev)
    chest = torch.empty((B, U, S, T, 4), dtype=torch.complex64, device=dev)
    errs = torch.zeros(B * U, dtype=torch.int64, device=dev)
    ws = eng.workspace(cfg, B)
    st = torch.cuda.current_stream(dev)
    box = {}

    def gen(i):
        box["b"] = src.generate(B, mods, n0, seed=17, first_slot=(i * world + rank) * B, out=box.get("b"))

    def full(i):
        gen(i)
        b = box["b"]
        eng.forward_device(cfg, b.y, b.pilots, nf, b.mod_order, N_IT, llr, chest, workspace=ws, stream=st)
        count_bit_errors(cfg, llr, b.labels, b.mod_order, out=errs)

    res = {}
    for name, fn in (("generate", gen), ("pipeline", full)):
        for i in range(3):
            fn(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for i in range(steps):
            fn(3 + i)
        b.record(st)
        torch.cuda.synchronize()
        t = max_over_ranks(a.elapsed_time(b) / 1e3, dev)
        res[name] = {"slots_per_s": round(B * steps * world / t, 1), "ms_per_step": round(t / steps * 1e3, 4)}
    bits = cfg.num_data_res * 4 * U
    return {"generate_slots_per_s": res["generate"]["slots_per_s"],
            "generate_us_per_slot": round(res["generate"]["ms_per_step"] * 1e3 / B, 2),
            "pipeline_slots_per_s": res["pipeline"]["slots_per_s"], "steps": steps, "slots_per_step": B,
            "uncoded_ber_last_steps": round(float(errs.sum().item()) / (bits * B * (steps + 3)), 4),
            "launches_per_step": 2 + eng.launch_count(cfg, N_IT) + 1,
            "note": "device Philox variates, doubletdl channels, 16-QAM, n0 = 0.1; random-init receiver, so the "
                    "BER is ~0.5 by construction"}


def dropin_latency(cfg, config, w, mcs, runs: int = 20):
    """The drop-in ``nrx_forward`` exactly as the reference arm is timed: one C2
    slot per call, numpy complex128 in, numpy LLRs / chest out (host copies,
    pilot stacking, MCS checks and the weight fingerprint inside the call)."""
    from paper_2409_02912_b200.nrx import nrx_forward
    from paper_2409_02912_b200.synth import synth_slots
    y, books, _ = synth_slots(cfg, [4, 4], 2, 0.1, seed=5)
    out = {}
    for prec in ("fp32", "fp32_simt", "fp16"):
        for i in range(3):
            nrx_forward(y[i % 2], books[i % 2], cfg, mcs, w, config, 0.1, precision=prec)
        ts = []
        for i in range(runs):
            t0 = time.perf_counter()
            nrx_forward(y[i % 2], books[i % 2], cfg, mcs, w, config, 0.1, precision=prec)
            ts.append(time.perf_counter() - t0)
        ts = np.asarray(ts)
        out[prec] = {"p50_ms": round(float(np.median(ts) * 1e3), 3), "slots_per_s": round(float(1.0 / ts.mean()), 1)}
    out["note"] = ("paper_2409_02912_b200.nrx.nrx_forward with the reference signature, one C2 slot per call "
                   "(numpy in / numpy out), the call pattern the reference arm is timed with")
    return out


def next_rows(cfg, B, dev, reps: int = 3):
    """Device time of the widened §8(f) rows at C2: LDPC encode and decode of
    the 16-QAM stream codeword (IRA, n0 = 169,840; decode at a noise level
    below the code's threshold, so all 20 iterations run), and the ls_lmmse
    and perfect_kbest (K = 16) baseline receivers on B slots."""
    import torch
    from paper_2409_02912_b200.classical import GpuKBest, GpuLsLmmse
    from paper_2409_02912_b200.config import default_mcs_table
    from paper_2409_02912_b200.ldpc import GpuLdpc, slot_code
    from paper_2409_02912_b200.slotgen import GpuSlotSource

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    U = cfg.num_ues
    code = slot_code(cfg, default_mcs_table()[14])
    g = GpuLdpc(code, dev)
    ncw = B * U
    info = (torch.rand((ncw, code.k_eff), device=dev) < 0.5).to(torch.uint8)
    enc_ms = timed(lambda: g.encode(info))
    tx = g.encode(info).float()
    llr = torch.clamp(2 * ((2 * tx - 1) + 1.2 * torch.randn_like(tx)) / 1.44, -20, 20)
    dec_ms = timed(lambda: g.decode(llr, 20))
    g.close()
    src = GpuSlotSource(cfg, device=dev)
    sb = src.generate(B, [4] * U, 0.1, seed=9, with_h_eff=True)
    out = torch.empty((B, U, cfg.num_subcarriers, cfg.num_symbols, 4), dtype=torch.float32, device=dev)
    ls = GpuLsLmmse(cfg.bs_antennas, 4)
    ls_ms = timed(lambda: ls.forward_device(cfg, sb.y, sb.pilots, None, sb.mod_order, 1, out, n0=sb.n0))
    kb = GpuKBest(cfg.bs_antennas, 4, 16)
    kb_ms = timed(lambda: kb.forward_device(cfg, sb.y, None, None, sb.mod_order, 1, out, n0=sb.n0, h_eff=sb.h_eff))
    return {"ldpc_codeword": {"n": code.n, "k_eff": code.k_eff, "num_tx_bits": code.num_tx_bits},
            "ldpc_encode_us_per_codeword": round(enc_ms * 1e3 / ncw, 2),
            "ldpc_decode_us_per_codeword_20_iterations": round(dec_ms * 1e3 / ncw, 2),
            "ls_lmmse_us_per_slot": round(ls_ms * 1e3 / B, 2),
            "perfect_kbest16_us_per_slot": round(kb_ms * 1e3 / B, 2),
            "codewords": ncw, "slots": B}


def e2e_throughput(eng, cfg, B, steps, world, dev):
    """NrxEngine.run_stream: every step copies its inputs (y, pilots, noise,
    MCS) from pinned host memory to the GPU and its LLR + chest grids back to
    pinned host memory; copies of neighbouring steps overlap the forward."""
    import torch
    import torch.distributed as dist
    U, S, T = cfg.num_ues, cfg.num_subcarriers, cfg.num_symbols
    rank = dist.get_rank() if world > 1 else 0
    hosts = [tuple(t.cpu().pin_memory() for t in gpu_batch(cfg, B, dev, seed=3, first_slot=(2 * rank + s) * B))
             for s in range(2)]
    outs = [(torch.empty((B, U, S, T, 4), dtype=torch.float32).pin_memory(),
             torch.empty((B, U, S, T, 4), dtype=torch.complex64).pin_memory()) for _ in range(2)]
    inputs = [hosts[i & 1] for i in range(steps)]
    outputs = [outs[i & 1] for i in range(steps)]
    eng.run_stream(cfg, inputs[:2], outputs[:2], N_IT)   # warm-up
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    eng.run_stream(cfg, inputs, outputs, N_IT)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([el], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    h2d = sum(t.numel() * t.element_size() for t in hosts[0])
    d2h = sum(t.numel() * t.element_size() for t in outs[0])
    # the e2e roofline: bare pinned copies of one step's outputs (D2H alone),
    # and of its inputs and outputs at once (H2D and D2H on two streams, as
    # run_stream overlaps them)
    dev_outs = [torch.empty(o.shape, dtype=o.dtype, device=dev) for o in outs[0]]
    dev_ins = [torch.empty(h.shape, dtype=h.dtype, device=dev) for h in hosts[0]]
    s_a, s_b = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

    def timed(h2d_too, reps=10):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        done_a, done_b = torch.cuda.Event(), torch.cuda.Event()
        torch.cuda.synchronize()
        ev0.record()
        s_a.wait_event(ev0)
        s_b.wait_event(ev0)
        for _ in range(reps):
            with torch.cuda.stream(s_a):
                for o, g in zip(outs[0], dev_outs):
                    o.copy_(g, non_blocking=True)
            if h2d_too:
                with torch.cuda.stream(s_b):
                    for g, h in zip(dev_ins, hosts[0]):
                        g.copy_(h, non_blocking=True)
        done_a.record(s_a)
        done_b.record(s_b)
        torch.cuda.current_stream().wait_event(done_a)
        torch.cuda.current_stream().wait_event(done_b)
        ev1.record()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / 1e3 / reps   # seconds per step

    timed(True, 2)
    t_d2h, t_duplex = timed(False), timed(True)
    del dev_outs, dev_ins
    pcie = {"d2h_copy_gbs": round(d2h / t_d2h / 1e9, 1),
            "d2h_bound_slots_per_s": round(B * world / t_d2h, 1),
            "duplex_bound_slots_per_s": round(B * world / t_duplex, 1),
            "note": "bare pinned copies of one step's outputs (D2H) and of its inputs + outputs on two "
                    "streams (duplex); the e2e value cannot exceed the duplex bound"}
    return {"value": round(B * steps * world / el, 2), "unit": "slots/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "pcie": pcie,
            "api": "NrxEngine.run_stream (pinned host inputs -> GPU -> pinned host LLR/chest every step; "
                   "H2D/compute/D2H overlapped across steps; wall clock incl. final sync)"}


def relaunch_under_torchrun(args):
    """`python bench.py --gpus N` (N > 1) without a torchrun environment:
    re-exec this script as N ranks (one process per GPU) under
    torch.distributed.run on 127.0.0.1, failing loudly when fewer than N GPUs
    are visible (the reference arm and --launch-check need no GPUs)."""
    if args.impl == "ours" and not args.launch_check:
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} requested but only {n} CUDA device(s) are visible")
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def launch_check():
    """One process per rank joins a process group (NCCL with GPUs, else gloo)
    and rank 0 prints the world size and the ranks that answered."""
    import torch
    import torch.distributed as dist
    world, rank, local = dist_env()
    if world > 1:
        backend = "nccl" if torch.cuda.is_available() and torch.cuda.device_count() >= world else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dev = torch.device("cuda", local)
        else:
            dist.init_process_group("gloo")
            dev = torch.device("cpu")
        t = torch.tensor([rank], dtype=torch.int64, device=dev)
        got = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(got, t)
        ranks = [int(x.item()) for x in got]
        dist.destroy_process_group()
    else:
        backend, ranks = "none", [0]
    if rank == 0:
        print(json.dumps({"launch_check": True, "world": world, "ranks": ranks, "backend": backend}), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--precision", choices=("fp32", "fp32_simt", "bf16", "fp16"),
                    default=os.environ.get("NRX_BENCH_PRECISION", "fp32"),
                    help="fp32: the reference's fp32 accuracy on the tensor cores (headline); fp32_simt: same "
                         "gate on FFMA; bf16 / fp16: reduced-precision modes (reported in by_precision)")
    ap.add_argument("--c5-slots", type=int, default=4096, help="C5 job size (BASELINE.json configs[4]); 0: skip")
    ap.add_argument("--launch-check", action="store_true",
                    help="only start the ranks (re-exec under torch.distributed.run for --gpus N > 1), join a "
                         "process group and print the world size rank 0 sees")
    ap.add_argument("--slots-per-step", type=int, default=32)
    ap.add_argument("--latency-runs", type=int, default=10000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-precision-sweep", action="store_true",
                    help="skip timing the other precisions (by_precision)")
    ap.add_argument("--cpu-json", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and (args.impl == "ours" or args.launch_check):
        relaunch_under_torchrun(args)  # does not return
    if world != args.gpus and args.impl == "ours" and not args.launch_check:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if args.launch_check:
        launch_check()
        return
    if args.impl == "reference":
        world, rank, _ = dist_env()
        if rank != 0:
            return
        res = run_reference(args, slots=max(1, args.steps), warmup=max(1, min(args.warmup, 2)))
        if args.cpu_json:
            print(json.dumps(res))
            return
        cfg_desc = {"workload": "single C2 slot per step (273 PRB x 14 sym, 2 UE 16-QAM, 4 RX; RT NRX "
                                "d_s=56 N_it=2), the reference's own nrx_forward on host CPUs",
                    "slots_per_step": 1}
        secs = 1.0 / res["value"]
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": round(res["value"], 4), "unit": "slots/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(secs * 1e3, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
            "data": DATA.replace("GPU slot generator", "host generator"), "config": cfg_desc,
            "latency_us": {"p50": round(res["p50_ms"] * 1e3, 1), "p99": round(res["p99_ms"] * 1e3, 1)},
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "kind", "cores", "sample")},
            "e2e": {"value": round(res["value"], 4), "unit": "slots/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "gpu_launches": 0}), flush=True)
        return
    run_ours(args)


if __name__ == "__main__":
    main()
