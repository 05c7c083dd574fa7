"""Summarise an `ncu --set full` report into profiles/ JSON and update the
per-slot DRAM traffic table bench.py reads (profiles/traffic.json).

  python scripts/ncu_summary.py gpurun_out/x3.ncu-rep --slots 8 --precision fp32 \
      --command "<the ncu command>" --out profiles/r2_ncu_kernels_fp32.json
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
           "launch__cluster_dim_x", "launch__registers_per_thread", "smsp__inst_executed.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed"]

# kernel template -> bench / profile_kernels name, in launch order of one forward
NAMES = [(r"k_ls_feat", "ls_feat"), (r"k_conv_x3<\d+, 0, 3, 2, 0|k_conv_tc<.*64, 0, 0, 3, 2, 0\b", "conv_state_init0"),
         (r"k_conv_x3<\d+, 1,|k_conv_tc<.*64, 1,", "conv_state_init1"), (r"k_msg_tc", "msg_agg"),
         (r"k_conv_x3<\d+, 0, 3, (4, 4|7, 0)|k_conv_tc<.*64, 0, 0, 3, 4, 4>", "conv_update0"),
         (r"k_conv_x3<\d+, 2,|k_conv_tc<.*64, 2,", "conv_update1"), (r"k_readout_tc", "readout")]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--slots", type=int, required=True)
    ap.add_argument("--precision", required=True)
    ap.add_argument("--command", default="")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                       "profiles", "traffic.json"))
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        k = {"Kernel Name": d["Kernel Name"]}
        for m in METRICS:
            col = m if m in d else next((h for h in head if h.endswith("." + m)), None)  # section-prefixed names
            if col is not None:
                k[m] = f"{d[col]} {u.get(col, '')}".strip()
        kernels.append(k)
    with open(args.out, "w") as fh:
        json.dump({"command": args.command, "slots_per_launch": args.slots, "precision": args.precision,
                   "kernels": kernels}, fh, indent=1)
    try:
        with open(args.traffic) as fh:
            traffic = json.load(fh)
    except FileNotFoundError:
        traffic = {}
    tab = traffic.setdefault(args.precision, {})
    seen = set()
    for k in kernels:
        name = next((n for pat, n in NAMES if re.search(pat, k["Kernel Name"])), None)
        if name is None or name in seen:
            continue
        seen.add(name)

        def val(m):
            return float(k[m].split()[0].replace(",", ""))

        def to_bytes(m):
            unit = k[m].split()[1] if len(k[m].split()) > 1 else "byte"
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return val(m) * scale
        tab[name] = {"dram_bytes_per_slot": (to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum"))
                     / args.slots, "measured_slots": args.slots,
                     "kernel_us": val("gpu__time_duration.sum"),
                     "source": f"ncu --set full, {os.path.basename(args.out)}"}
    with open(args.traffic, "w") as fh:
        json.dump(traffic, fh, indent=1)
    print(f"wrote {args.out}; traffic[{args.precision}] = {sorted(tab)}")


if __name__ == "__main__":
    main()
