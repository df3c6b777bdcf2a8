"""Parity of the exact launch configuration behind the headline number (-m gpu).

bench.py times config 4 with fuse=2, k_max=3, the packed Hermitian layout and the default
kernel choice, so almost every pass is a K3 group kernel whose warps loop over thousands of
tiles.  These tests run that plan -- nothing forced, nothing reduced -- against the CPU oracle:

* the whole config-4 QPE circuit at n = 12 and 13 and config 3 (random layered) at n = 12:
  every entry of rho, plus the readout-noisy probabilities (Eq. (dmsim));
* full-size registers (n = 16, 68.7 GB, and n = 14): a cluster circuit whose gates never couple
  two clusters of qubits spread over the whole register, so rho_out is the tensor product of
  per-cluster oracle runs (tests/_product.py) and every entry has an exact oracle value;
* small registers with the persistent grid capped (TANQ_GRID_CAP) so each warp walks many
  tiles, including the canonical-block skipping and self-transposed blocks.

Bar (BASELINE.json north star): max |delta rho_ij| <= 1e-10, relative Frobenius <= 1e-12.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import workloads as W
from oracle import dense

from _product import compare_column_blocks

pytestmark = pytest.mark.gpu

ABS, REL = 1e-10, 1e-12
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def Sim():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from __graft_entry__ import build
    build()
    from paper_2404_13184_b200 import Simulator
    return Simulator


def _plan_info(c, nm):
    from paper_2404_13184_b200.tanq import Plan
    return Plan(None, c, nm, fuse=2, k_max=3).info()


def _full_compare(sim, ref, n):
    N = 2 ** n
    worst, num, den = 0.0, 0.0, 0.0
    cols = max(1, (1 << 24) // N)
    for c0 in range(0, N, cols):
        got = sim.get_state(c0 * N, cols * N).reshape(cols, N)
        d = got - ref[:, c0:c0 + cols].T
        worst = max(worst, float(np.abs(d).max()))
        num += float(np.vdot(d, d).real)
        den += float(np.vdot(ref[:, c0:c0 + cols], ref[:, c0:c0 + cols]).real)
    return worst, (num / den) ** 0.5


@pytest.mark.parametrize("n", [12, 13])
def test_bench_plan_qpe_whole_circuit_vs_oracle(Sim, n):
    c, nm = W.config_workload(4, n=n)
    info = _plan_info(c, nm)
    assert info["n_k3"] >= 10, info                      # the group kernel carries the plan
    ref = dense.run(c, nm)
    ro = dense.readout_of(nm)
    with Sim(n) as sim:
        st = sim.run_circuit(c, nm)                     # defaults = bench plan (fuse 2, k_max 3)
        assert st["n_k3"] == info["n_k3"]
        p = sim.probs(ro)                               # straight from the packed layout
        mx, rel = _full_compare(sim, ref, n)
    assert mx <= ABS and rel <= REL, (mx, rel)
    np.testing.assert_allclose(p, dense.probs(ref, n, ro), atol=ABS, rtol=0)


def test_bench_plan_config3_vs_oracle(Sim):
    c, nm = W.config_workload(3, n=12, depth=20)
    info = _plan_info(c, nm)
    assert info["n_k3"] >= 10, info
    ref = dense.run(c, nm)
    with Sim(12) as sim:
        sim.run_circuit(c, nm)
        p = sim.probs()
        mx, rel = _full_compare(sim, ref, 12)
    assert mx <= ABS and rel <= REL, (mx, rel)
    np.testing.assert_allclose(p, dense.probs(ref, 12), atol=ABS, rtol=0)


CLUSTERS = {
    16: [(0, 5, 10, 15), (1, 6, 11, 12), (2, 7, 8, 13), (3, 4, 9, 14)],
    14: [(0, 4, 7, 13), (1, 6, 9, 12), (2, 8, 11), (3, 5, 10)],
}


@pytest.mark.parametrize("n", [14, 16])
def test_fullsize_cluster_product_vs_oracle(Sim, n):
    """Full-size register, bench plan: every K3 group lands on qubits spread over the whole
    index range (up to the top qubit, whose blocks are never stored in place)."""
    c, nm, subs = W.cluster_product_workload(n, CLUSTERS[n], layers=6, seed=W.BASE_SEED + 40 + n)
    info = _plan_info(c, nm)
    assert info["n_k3"] >= 8, info
    parts = [(qs, dense.run(sc, snm)) for qs, sc, snm in subs]
    N = 2 ** n
    full = os.environ.get("TANQ_FULLSIZE") == "1" or n <= 14
    width = 16
    rng = np.random.default_rng(n)
    starts = (np.arange(0, N, width) if full else
              np.sort(rng.choice(N // width, 256, replace=False)) * width)
    with Sim(n) as sim:
        st = sim.run_circuit(c, nm)
        assert st["n_k3"] == info["n_k3"]
        # the diagonal touches every self-transposed block of every pass
        p = sim.probs()
        x = np.arange(N, dtype=np.int64)
        pe = np.ones(N)
        from _product import local_index
        for qs, rho in parts:
            pe *= np.real(np.diag(rho))[local_index(x, qs)]
        assert np.abs(p - pe).max() <= ABS
        worst, num, den = compare_column_blocks(sim, parts, n, starts, width)
    assert worst <= ABS and (num / den) ** 0.5 <= REL, (worst, (num / den) ** 0.5)


GRID_SNIPPET = r"""
import numpy as np, sys
sys.path.insert(0, %(root)r)
import workloads as W
from oracle import dense
from paper_2404_13184_b200 import Simulator
from paper_2404_13184_b200.tanq import Plan
worst = 0.0
for n in (7, 8, 9):
    c = W.random_circuit(n, 70, seed=9100 + n, kmax=3)
    nm = W.synthetic_calibration(c, n, depol=True, thermal=True, overrot=True)
    ref = dense.run(c, nm)
    N = 2 ** n
    for kmax in (3, 4, 5):
        inf = Plan(None, c, nm, fuse=2, k_max=kmax).info()
        assert inf["n_k3"] + inf["n_k4"] + inf["n_k5"] > 0
        with Simulator(n) as sim:
            sim.run_circuit(c, nm, fuse=2, k_max=kmax)
            p = sim.probs()
            got = sim.get_state().reshape(N, N).T
        np.testing.assert_allclose(p, np.diag(ref).real, atol=1e-10)
        d = got - ref
        mx, rel = np.abs(d).max(), np.linalg.norm(d) / np.linalg.norm(ref)
        assert mx <= 1e-10 and rel <= 1e-12, (n, kmax, mx, rel)
        worst = max(worst, mx)
print("OK", worst)
"""


@pytest.mark.parametrize("cap", ["1", "3"])
def test_group_kernel_many_tiles_per_warp(cap):
    """TANQ_GRID_CAP caps the persistent grids, so at n = 7..9 every warp of the group, tile and
    k=2 kernels runs dozens of tiles: the loop-carried paths (next canonical block, per-tile
    packed placement, named barriers of self-transposed blocks) that full-size launches take."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, TANQ_GRID_CAP=cap)
    r = subprocess.run([sys.executable, "-c", GRID_SNIPPET % {"root": ROOT}], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.strip().splitlines()[-1].startswith("OK")


@pytest.mark.skipif(os.environ.get("TANQ_FULLSIZE") != "1", reason="needs ~70 GB host RAM, ~25 min")
def test_qpe16_prefix_bench_plan_vs_oracle(Sim):
    """n = 16 QPE prefix under the bench plan (k_max = 3): X(target), H on counting qubits
    0, 3, 7, 10, 14, CP(q -> 15) for each and two inverse-QFT-style CP pairs -- 51 basis gates
    fused into three 3-qubit groups on low, middle and top qubits (incl. the target 15)."""
    c, nm = W.config_workload(4)
    ops = [c.ops[0]]
    for q in (0, 3, 7, 10, 14):
        ops += W.basis_h(q)
    for q, lam in ((0, 0.7), (7, -1.3), (14, 2.1), (3, 0.4), (10, -0.9)):
        ops += W.basis_cp(q, 15, lam)
    ops += W.basis_cp(0, 7, 0.3) + W.basis_cp(3, 10, -0.6)
    prefix = W.Circuit(16, ops)
    info = _plan_info(prefix, nm)
    assert info["n_k3"] >= 3, info
    ref = dense.run(prefix, nm)
    with Sim(16) as sim:
        st = sim.run_circuit(prefix, nm)
        assert st["n_k3"] == info["n_k3"]
        mx, rel = _full_compare(sim, ref, 16)
    assert mx <= ABS and rel <= REL, (mx, rel)


@pytest.mark.parametrize("config,n", [(4, 9), (3, 9), (4, 10), (2, 10)])
def test_block_groups_kmax5(Sim, config, n):
    """k_max = 5: block groups of up to 5 qubits (at most 3 outside {0, 1}) on the block
    kernel, each sub-op with its own warp-half split, packed and full layouts."""
    from paper_2404_13184_b200.tanq import Plan
    c, nm = W.config_workload(config, n=n, **({"depth": 20} if config == 3 else {}))
    assert Plan(None, c, nm, fuse=2, k_max=5).info()["n_k5"] > 0
    ref = dense.run(c, nm)
    N = 2 ** n
    for mirror in (True, False):
        with Sim(n) as sim:
            sim.run_circuit(c, nm, fuse=2, k_max=5, mirror=mirror)
            p = sim.probs(dense.readout_of(nm))
            got = sim.get_state().reshape(N, N).T
        np.testing.assert_allclose(p, dense.probs(ref, n, dense.readout_of(nm)), atol=ABS)
        d = got - ref
        assert np.abs(d).max() <= ABS and np.linalg.norm(d) / np.linalg.norm(ref) <= REL
