"""One dense k=3 channel launch (has3 group kernel) for ncu A/B captures.

  ncu --set full -k regex:group_kernel -s 1 -c 1 python scripts/prof_k3.py --n 14 --qubits 0,1,2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("KBENCH_PKG_ROOT"):
    sys.path.insert(0, os.environ["KBENCH_PKG_ROOT"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=14)
    ap.add_argument("--qubits", default="0,1,2")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import workloads as W
    from paper_2404_13184_b200 import Simulator
    qs = tuple(int(x) for x in args.qubits.split(","))
    Ks = W.random_kraus(np.random.default_rng(0), 2 ** len(qs), 2)
    with Simulator(args.n) as sim:
        for _ in range(args.reps):
            sim.apply_channel(qs, Ks)
        sim.sync()


if __name__ == "__main__":
    main()
