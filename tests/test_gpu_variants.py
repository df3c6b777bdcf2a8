"""GPU parity of every group / k=2 kernel variant (-m gpu).

The library picks a kernel per launch (per-warp tiles, cooperative 4- or 2-warp tiles with one
or two buffers, direct or tiled k=2); the choice is read once per process from TANQ_GROUP /
TANQ_K2PATH, so each forced variant runs in its own interpreter.  Every variant must match the
CPU oracle at the north-star bar on random noisy circuits (groups of 3 and 4 qubits, mirror
mode on and off, ragged small registers).
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r"""
import numpy as np, sys
sys.path.insert(0, %(root)r)
import workloads as W
from oracle import dense
from paper_2404_13184_b200 import Simulator
worst = 0.0
for seed in range(4):
    n = 4 + seed                              # 4..7 qubits: one partial tile up to many tiles
    c = W.random_circuit(n, 60, seed=4200 + seed, kmax=3)
    nm = W.synthetic_calibration(c, seed, depol=True, thermal=True, overrot=True)
    ref = dense.run(c, nm)
    N = 2 ** n
    for kmax in (3, 4):
        for mirror in (True, False):
            with Simulator(n) as sim:
                sim.run_circuit(c, nm, fuse=2, k_max=kmax, mirror=mirror)
                p = sim.probs()                   # diagonal: valid in the packed layout
                z = sim.expect_pauli(0, 0b11)
                got = sim.get_state().reshape(N, N).T
            np.testing.assert_allclose(p, np.diag(ref).real, atol=1e-10)
            assert abs(z - dense.expect_pauli(ref, n, 0, 0b11)) < 1e-10
            d = got - ref
            mx = np.abs(d).max()
            rel = np.linalg.norm(d) / np.linalg.norm(ref)
            assert mx <= 1e-10 and rel <= 1e-12, (seed, kmax, mirror, mx, rel)
            worst = max(worst, mx)
for n in (7, 9):                              # QPE: sparse noisy CX / CP superoperators
    c, nm = W.config_workload(4, n=n)
    ref = dense.run(c, nm)
    N = 2 ** n
    with Simulator(n) as sim:
        sim.run_circuit(c, nm, fuse=2, k_max=3)
        got = sim.get_state().reshape(N, N).T
    mx = np.abs(got - ref).max()
    assert mx <= 1e-10 and np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12, (n, mx)
    worst = max(worst, mx)
print("OK", worst)
"""


@pytest.mark.parametrize("group,k2path,mirror,sparse", [
    ("warp", "direct", "1", "0"), ("q1", "tile", "1", "0"), ("o1", "auto", "1", "0"),
    ("auto", "auto", "1", "0"), ("auto", "direct", "0", "0"), ("q1", "auto", "0", "0"),
    ("warp", "tile", "0", "0"), ("o1", "tile", "0", "0"),
    ("auto", "auto", "1", "64"), ("auto", "auto", "0", "64"),
    ("auto", "auto", "1", "rb"), ("auto", "auto", "0", "rb")])
def test_kernel_variant_parity(group, k2path, mirror, sparse):
    """sparse = 64: the block kernel's sparse DFMA sub-op (TANQ_SPARSE_MAX) for every k=2
    sub-op with at most 64 nonzeros; sparse = rb: the real-basis block programs
    (TANQ_RBASIS=1)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, TANQ_GROUP=group, TANQ_K2PATH=k2path, TANQ_MIRROR=mirror,
               TANQ_SPARSE_MAX="0" if sparse == "rb" else sparse,
               TANQ_RBASIS="1" if sparse == "rb" else "0")
    r = subprocess.run([sys.executable, "-c", SNIPPET % {"root": ROOT}], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.strip().splitlines()[-1].startswith("OK")
