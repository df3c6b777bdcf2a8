"""Per-kernel microbenchmark: time apply_superop for k=1,2,3 at several target positions.

  TANQ_K2=fma|mma python scripts/kbench.py --n 14
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("KBENCH_PKG_ROOT"):  # A/B runs against another build of the package
    sys.path.insert(0, os.environ["KBENCH_PKG_ROOT"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=14)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--kmax", type=int, default=3, help="group size limit for the group cases")
    ap.add_argument("--groups-only", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2404_13184_b200 import Simulator
    n = args.n
    rng = np.random.default_rng(0)
    cases = [(0,), (1,), (n - 1,), (0, 1), (1, 2), (0, n - 1), (5, n - 1), (n - 2, n - 1),
             (0, 1, 2), (3, 7, n - 1)]
    amps = 4 ** n
    out = []
    with Simulator(n) as sim:
        st = torch.cuda.Stream()
        torch.cuda.set_stream(st)
        sim.set_stream(st.cuda_stream)
        import workloads as W
        for qs in ([] if args.groups_only else cases):
            k = len(qs)
            Ks = W.random_kraus(rng, 2 ** k, 2)  # CPTP: Hermiticity-preserving (mirror mode)
            for _ in range(3):
                sim.apply_channel(qs, Ks)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.reps):
                sim.apply_channel(qs, Ks)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.reps
            gbs = 32 * amps / (ms * 1e-3) / 1e9
            tf = 8 * 4 ** k * amps / (ms * 1e-3) / 1e12
            out.append({"qubits": qs, "k": k, "ms": ms, "GBs": gbs, "alg_TFs": tf})
            print(json.dumps(out[-1]), flush=True)
        # K3 groups: chains of k=2 channels inside 3 qubits, one pass (fuse=2, k_max=3)
        groups = [[(0, 1), (1, 2)], [(1, 2), (2, 3), (1, 3)], [(5, n - 1), (n - 1, n - 2)],
                  [(0, 1), (1, 2), (0, 2), (2, 1)], [(3, 7), (7, n - 1), (3, n - 1), (7, 3), (3, 7)],
                  [(8, 10), (10, 12), (8, 12)], [(n - 3, n - 2), (n - 2, n - 1), (n - 3, n - 1), (n - 2, n - 3)]]
        if args.kmax >= 4:  # 4-qubit groups
            groups += [[(0, 1), (2, 3), (1, 2), (0, 3)], [(n - 4, n - 3), (n - 2, n - 1), (n - 3, n - 2), (n - 4, n - 1)],
                       [(5, 9), (11, 13), (9, 11), (5, 13)]]
        for g in groups:
            ops = [W.Op("kraus", qs, kraus=W.random_kraus(rng, 4, 2)) for qs in g]
            plan = sim.plan(W.Circuit(n, ops), None, fuse=2, k_max=args.kmax)
            info = plan.info()
            for _ in range(3):
                plan.exec(sim)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(args.reps):
                plan.exec(sim)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.reps
            out.append({"group": g, "kernels": info["ops_fused"], "gate_updates": info["gate_updates"],
                        "ms": ms, "GBs_per_pass": 32 * amps * info["ops_fused"] / (ms * 1e-3) / 1e9,
                        "ms_per_update": ms / info["gate_updates"]})
            print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
