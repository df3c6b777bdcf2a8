"""Whole-circuit parity of the bench plan against the CPU oracle at a given size (one-off
evidence runs on the GPU box; the oracle needs 16 * 4^n bytes of host RAM).

  python scripts/fullsize_parity.py --config 4 --n 14 [--prefix G]

Runs the circuit (or its first G basis gates) with the bench plan (fuse 2, k_max 3, packed
layout, default kernels) on cuda:0, reads the state back by column blocks, runs the oracle
(oracle/dense.c, all host cores) on the same circuit and prints one JSON line: max |delta|,
relative Frobenius error, readout-noisy probability error, plan shape and both run times.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n", type=int, default=14)
    ap.add_argument("--prefix", type=int, default=0, help="first G basis gates only (0 = all)")
    ap.add_argument("--depth", type=int, default=None, help="config 3 depth override")
    args = ap.parse_args()
    import numpy as np
    import workloads as W
    from oracle import dense
    from paper_2404_13184_b200 import Simulator, CReadout

    c, nm = W.config_workload(args.config, n=args.n, depth=args.depth)
    if args.prefix:
        c = W.Circuit(c.n, c.ops[:args.prefix])
    n, N = c.n, 2 ** c.n
    ro = dense.readout_of(nm)
    with Simulator(n) as sim:
        t0 = time.perf_counter()
        st = sim.run_circuit(c, nm)
        p_gpu = sim.probs(CReadout.of(nm))
        t_gpu = time.perf_counter() - t0
        t1 = time.perf_counter()
        rho = dense.run(c, nm)
        t_orc = time.perf_counter() - t1
        p_orc = dense.probs(rho, n, ro)
        worst, num, den = 0.0, 0.0, 0.0
        cols = max(1, (1 << 24) // N)
        for c0 in range(0, N, cols):
            got = sim.get_state(c0 * N, cols * N).reshape(cols, N)
            ref = rho[:, c0:c0 + cols].T
            d = got - ref
            worst = max(worst, float(np.abs(d).max()))
            num += float(np.vdot(d, d).real)
            den += float(np.vdot(ref, ref).real)
    rel = (num / den) ** 0.5
    line = {"config": args.config, "n_qubits": n, "basis_gates": len(c.ops),
            "plan": {k: st[k] for k in ("ops_fused", "gate_updates", "n_k1", "n_k2", "n_k3")},
            "max_abs": worst, "rel_frobenius": rel,
            "probs_max_abs": float(np.abs(p_gpu - p_orc).max()),
            "pass": bool(worst <= 1e-10 and rel <= 1e-12),
            "gpu_s_incl_planning": t_gpu, "oracle_s": t_orc, "host_cores": os.cpu_count()}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
