"""Multi-process path (tanq_create_dist, one process per shard) on real hardware (-m gpu).

The pool has one GPU per box and NCCL refuses several ranks on one device, so the ranks'
NCCL calls go to tests/nccl_shim/nccl_shim.cpp (TANQ_NCCL_LIB): a host-staged implementation
of exactly the calls libtanq makes.  Everything else is the product path: per-rank shards on
the device, the remap schedule, half selection, chunked pack / unpack kernels, bit-map
bookkeeping and the all-reduced probabilities / expectations / state gather -- checked
against the CPU oracle at the north-star bar for world sizes 2, 4 and 8 (the top qubit, then
the top qubit and a bit of the next, global).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from __graft_entry__ import build
    build()
    out = str(tmp_path_factory.mktemp("shim") / "libnccl_shim.so")
    r = subprocess.run(["g++", "-O2", "-shared", "-fPIC", "-std=c++17", "-I/usr/local/cuda/include",
                        os.path.join(ROOT, "tests", "nccl_shim", "nccl_shim.cpp"), "-o", out,
                        "-L/usr/local/cuda/lib64", "-lcudart", "-lpthread"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


@pytest.mark.parametrize("world,n,seed,batch,xlog", [
    (2, 6, 5, "1", "23"), (2, 7, 6, "1", "23"), (4, 6, 7, "1", "23"), (8, 6, 8, "1", "23"),
    (4, 7, 9, "1", "23"), (4, 6, 7, "0", "23"), (8, 6, 8, "0", "23"),
    (2, 7, 6, "1", "5"), (4, 7, 9, "1", "6"), (8, 6, 8, "0", "4"),
    # shard-local parity layout with the packed kernels (>= 6 fully local qubits)
    (2, 8, 10, "1", "23"), (4, 8, 11, "1", "6"), (8, 9, 12, "1", "23"), (2, 9, 13, "1", "5")])
def test_dist_remap_parity(shim, world, n, seed, batch, xlog):
    """batch = 1: two swaps of one op run as one 4-way exchange (remap_swap2); 0: pairwise.
    xlog: staging slot of 2^xlog amplitudes -- small slots run the pipelined exchange over
    many chunks (comm on its own stream, pack / unpack overlapped)."""
    env = dict(os.environ, TANQ_NCCL_LIB=shim, OMP_NUM_THREADS="2", TANQ_REMAP_BATCH=batch,
               TANQ_XCHUNK_LOG2=xlog)
    port = 29600 + 10 * world + n + 100 * int(batch) + int(xlog)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
                        "--nproc-per-node", str(world), "--master-addr", "127.0.0.1",
                        "--master-port", str(port), os.path.join(ROOT, "tests", "dist_worker.py"),
                        "--qubits", str(n), "--seed", str(seed)],
                       env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("DIST")]
    assert line and line[-1].endswith("OK"), out[-4000:]
    print(line[-1])


@pytest.mark.parametrize("world,config,n", [(8, 5, 8), (4, 4, 7), (2, 4, 9), (8, 5, 9)])
def test_dist_config_workloads(shim, world, config, n):
    """BASELINE configs 5 (VQE ansatz + its Pauli-string Hamiltonian, the 8-GPU config) and 4
    (QPE with calibrated noise + readout) scaled down, on `world` ranks: state, readout-noisy
    probabilities and every Pauli expectation against the oracle."""
    env = dict(os.environ, TANQ_NCCL_LIB=shim, OMP_NUM_THREADS="2")
    port = 29800 + 10 * world + config
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes", "1",
                        "--nproc-per-node", str(world), "--master-addr", "127.0.0.1",
                        "--master-port", str(port), os.path.join(ROOT, "tests", "dist_worker.py"),
                        "--qubits", str(n), "--config", str(config)],
                       env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("DIST")]
    assert line and line[-1].endswith("OK"), out[-4000:]
    print(line[-1])
