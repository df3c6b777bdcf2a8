"""One fused group launch for ncu captures: a chain of random 2-qubit channels on the given
qubit pairs, fused into one group (fuse=2, k_max=3), applied `--reps` times.

  ncu --set full -k regex:tile_kernel -s 1 -c 1 python scripts/prof_group.py --n 14 --pairs 5,13:13,12
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=14)
    ap.add_argument("--pairs", default="5,13:13,12")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import workloads as W
    from paper_2404_13184_b200 import Simulator
    rng = np.random.default_rng(0)
    pairs = [tuple(int(x) for x in p.split(",")) for p in args.pairs.split(":")]
    ops = [W.Op("kraus", qs, kraus=W.random_kraus(rng, 2 ** len(qs), 2)) for qs in pairs]
    with Simulator(args.n) as sim:
        plan = sim.plan(W.Circuit(args.n, ops), None, fuse=2, k_max=3)
        for _ in range(args.reps):
            plan.exec(sim)
        sim.sync()
        print(plan.info())


if __name__ == "__main__":
    main()
