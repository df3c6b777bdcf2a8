"""Per-config measurement table (one B200): every BASELINE.json config at the largest size
that fits one GPU, timed through the public API with CUDA events.  Writes one JSON object
per config to stdout (profiles/r01_suite.jsonl).

  python scripts/suite.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import workloads as W
    from paper_2404_13184_b200 import Simulator, CReadout
    from paper_2404_13184_b200.tanq import Plan

    cases = [(1, None, "GHZ-3 + depolarizing + readout (worked example)"),
             (2, 10, "QFT-10, thermal + over-rotation"),
             (3, 14, "random layered n=14 depth 100, depol + thermal"),
             (4, 16, "QPE-16, calibrated noise (68.7 GB)"),
             (5, 16, "VQE ansatz at n=16 (n=18 needs 8 GPUs) + its Pauli-string Hamiltonian")]
    for cfg, n, name in cases:
        c, nm = W.config_workload(cfg, n=n)
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        with Simulator(c.n) as sim:
            sim.set_stream(stream.cuda_stream)
            plan = Plan(sim, c, nm, graph=(c.n <= 12))
            ro = CReadout.of(nm)
            reps = 20 if c.n <= 12 else 3
            for _ in range(3):
                sim.reset()
                st = plan.exec(sim)
                sim.probs(ro)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(reps):
                sim.reset()
                plan.exec(sim)
                sim.probs(ro)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            out = {"config": cfg, "name": name, "n": c.n, "gates": len(c.ops),
                   "kernels": st["ops_fused"], "gate_updates": st["gate_updates"],
                   "ms_per_circuit": ms, "fused_gate_updates_per_s": st["gate_updates"] / (ms * 1e-3),
                   "circuit_gates_per_s": len(c.ops) / (ms * 1e-3), "graph": c.n <= 12}
            if c.paulis:
                t0 = time.perf_counter()
                vals = [sim.expect_pauli(x, z).real for x, z in c.paulis]
                out["pauli_terms"] = len(vals)
                out["ms_per_pauli_expectation"] = (time.perf_counter() - t0) * 1e3 / len(vals)
                out["energy"] = sum(vals)
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
