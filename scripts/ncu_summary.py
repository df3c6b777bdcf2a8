"""Summarise ncu captures into profiles/ (tracked): key metrics per kernel launch + traffic.

  python scripts/ncu_summary.py gpurun_out/prof_k2mma.ncu-rep [...] --out profiles/r01_ncu_full.md
"""
import argparse
import csv
import io
import json
import os
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 (DFMA) pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(hdr, units, r) for r in rows[2:]]


def to_bytes(v, unit):
    v = float(v)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return v * scale


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic", default="profiles/ncu_traffic.json")
    ap.add_argument("--n", type=int, required=True, help="qubits of the captured run (alg bytes = 32*4^n)")
    ap.add_argument("--bytes-per-amp", type=float, default=32.0,
                    help="algorithmic bytes per amplitude of the captured launches (24 in mirror mode)")
    ap.add_argument("--name-map", default="gate_kernel<1=gate_k1,gate_kernel<2=gate_k2,gate2_mma=gate_k2,group_kernel=group_dmma")
    args = ap.parse_args()
    nmap = [kv.split("=") for kv in args.name_map.split(",")]
    traffic = json.load(open(args.traffic)) if os.path.exists(args.traffic) else {}  # merged
    lines = ["| kernel | " + " | ".join(k[1] for k in KEYS) + " |",
             "|---|" + "---|" * len(KEYS)]
    seen = set()
    for rep in args.reps:
        for hdr, units, r in rows_of(rep):
            col = {h: i for i, h in enumerate(hdr)}
            name = r[col["Kernel Name"]]
            vals = []
            for key, _ in KEYS:
                i = col.get(key)
                vals.append(f"{r[i]} {units[i]}".strip() if i is not None else "n/a")
            lines.append(f"| `{name[:60]}` | " + " | ".join(vals) + " |")
            rd, wr = col.get("dram__bytes_read.sum"), col.get("dram__bytes_write.sum")
            if rd is not None and wr is not None:
                tb = to_bytes(r[rd], units[rd]) + to_bytes(r[wr], units[wr])
                for pat, short in nmap:
                    if pat in name:
                        if short in seen:
                            continue
                        seen.add(short)
                        alg = args.bytes_per_amp * 4 ** args.n
                        traffic[short] = {"dram_bytes_per_launch": tb, "algorithmic_bytes_per_launch": alg,
                                          "ratio": tb / alg, "n_qubits": args.n,
                                          "source": os.path.basename(rep)}
    with open(args.out, "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(args.traffic, "w") as f:
        json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
