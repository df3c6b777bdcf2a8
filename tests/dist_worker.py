"""Worker for tests/test_gpu_dist.py (not a test module): one rank of the multi-process path
(tanq_create_dist) on a random noisy circuit whose top qubits are global, checked against the
CPU oracle on rank 0.  Launched with torch.distributed.run; the NCCL calls of libtanq go to
TANQ_NCCL_LIB (the host-staged shim when all ranks share one GPU)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--qubits", type=int, default=6)
    ap.add_argument("--seed", type=int, default=5)
    ap.add_argument("--depth", type=int, default=60)
    ap.add_argument("--config", type=int, default=0,
                    help="BASELINE config workload (scaled to --qubits) instead of a random circuit")
    args = ap.parse_args()
    import numpy as np
    import torch.distributed as dist
    import workloads as W
    from paper_2404_13184_b200 import Simulator, nccl_unique_id

    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    dist.init_process_group("gloo")  # bootstrap of the unique id only
    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    n = args.qubits
    if args.config:
        c, nm = W.config_workload(args.config, n=n)
    else:
        c = W.random_circuit(n, args.depth, seed=args.seed, kmax=3)
        nm = W.synthetic_calibration(c, args.seed, depol=True, thermal=True, overrot=True)
    xm, zm = 0b11 << (n - 2), 0b101 << (n - 3)      # touches the global qubits
    paulis = list(c.paulis) or [(xm, zm)]
    from paper_2404_13184_b200 import CReadout
    with Simulator(n, world_size=world, rank=rank, device=0, nccl_uid=uid[0]) as sim:
        st = sim.run_circuit(c, nm, fuse=2, k_max=3)
        vec = sim.get_state()                        # whole vec(rho), all-reduced
        p = sim.probs()
        pr = sim.probs(CReadout.of(nm))              # readout-noisy distribution
        zs = [sim.expect_pauli(x, z) for x, z in paulis]
    if rank == 0:
        from oracle import dense
        ref = dense.run(c, nm)
        N = 2 ** n
        got = vec.reshape(N, N).T
        err = float(np.abs(got - ref).max())
        rel = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
        perr = max(float(np.abs(p - np.diag(ref).real).max()),
                   float(np.abs(pr - dense.probs(ref, n, dense.readout_of(nm))).max()))
        zerr = max(abs(z - dense.expect_pauli(ref, n, x, zz)) for z, (x, zz) in zip(zs, paulis))
        ok = err <= 1e-10 and rel <= 1e-12 and perr <= 1e-10 and zerr <= 1e-10 and st["n_remaps"] > 0
        print(f"DIST world={world} n={n} config={args.config} paulis={len(paulis)} remaps={st['n_remaps']} remap_bytes={st['remap_bytes']} max_abs={err:.3e} rel={rel:.3e} "
              f"probs={perr:.3e} expect={zerr:.3e} {'OK' if ok else 'MISMATCH'}", flush=True)
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
