"""Short driver for ncu captures: run the first `--ops` fused ops of a config's plan once.

  ncu --set full -k regex:gate_kernel -s 5 -c 1 python scripts/prof_driver.py --config 3 --n 14
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=14)
    ap.add_argument("--depth", type=int, default=None)
    ap.add_argument("--kmax", type=int, default=3)
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    import workloads as W
    from paper_2404_13184_b200 import Simulator
    c, nm = W.config_workload(args.config, n=args.n, depth=args.depth)
    with Simulator(c.n) as sim:
        p = sim.plan(c, nm, fuse=2, k_max=args.kmax)
        for _ in range(args.reps):
            st = p.exec(sim)
        sim.sync()
    print(st)


if __name__ == "__main__":
    main()
