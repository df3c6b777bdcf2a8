"""Per-call timing of the public run_circuit path (plan cache + graph replay) on a small
config: where does an end-to-end call spend its time?  TANQ_GRAPH_DEBUG=1 logs graph
capture / replay decisions.

  TANQ_GRAPH_DEBUG=1 python scripts/e2e_probe.py --config 2
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=8)
    args = ap.parse_args()
    import torch
    import workloads as W
    from paper_2404_13184_b200 import Simulator, CReadout
    c, nm = W.config_workload(args.config)
    with Simulator(c.n) as sim:
        for r in range(args.reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sim.reset()
            t1 = time.perf_counter()
            st = sim.run_circuit(c, nm)
            t2 = time.perf_counter()
            sim.sync()
            t3 = time.perf_counter()
            sim.probs(CReadout.of(nm))
            t4 = time.perf_counter()
            print(f"rep {r}: reset {1e3*(t1-t0):.3f} run {1e3*(t2-t1):.3f} sync {1e3*(t3-t2):.3f} "
                  f"probs {1e3*(t4-t3):.3f} ms plan_ms {st['plan_ms']:.3f}", flush=True)


if __name__ == "__main__":
    main()
