"""Write workloads/plan_counts.json: the fused-gate-update count of the GPU plan of every bench
workload (host planner only: tanq_plan_create_host, no device work).

bench.py's reference arm (the CPU oracle) reports the same metric -- fused-gate updates per
second -- so it needs the count of updates one circuit represents.  It reads this table
instead of loading libtanq.so, so the reference process never touches the product library.
tests/test_bench_contract.py checks the table against the live planner.

  python scripts/plan_counts.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "workloads", "plan_counts.json")
CASES = [(3, 7), (2, 10), (3, 14), (4, 12), (4, 13), (4, 14), (4, 16), (5, 16), (5, 18)]


def key(config, n, world, fuse, kmax):
    return f"config{config}:n{n}:gpus{world}:fuse{fuse}:kmax{kmax}"


def compute():
    import workloads as W
    from paper_2404_13184_b200.tanq import Plan
    table = {}
    for config, n in CASES:
        c, nm = W.config_workload(config, n=n)
        for world in (1, 2, 4, 8):
            if 2 * n - (world.bit_length() - 1) < 8:
                continue
            for fuse, kmax in ((2, 3), (2, 4), (2, 5)):
                info = Plan(None, c, nm, fuse=fuse, k_max=kmax, world_size=world).info()
                table[key(config, n, world, fuse, kmax)] = {
                    "gates": len(c.ops), "gate_updates": info["gate_updates"],
                    "kernel_ops": info["ops_fused"]}
    return table


if __name__ == "__main__":
    t = compute()
    with open(OUT, "w") as f:
        json.dump(t, f, indent=1, sort_keys=True)
    print(f"wrote {len(t)} entries to {OUT}")
