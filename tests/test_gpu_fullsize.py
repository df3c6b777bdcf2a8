"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (-m gpu).

* config 3 (n=14, 4.3 GB): noisy prefix (one full layer, 77 gates) element by element against
  the CPU oracle; the full depth-100 noiseless circuit against the brute-force state vector
  (diagonal + sampled columns); the full noisy circuit against invariants.
* config 4 (n=16, 68.7 GB): noiseless QPE peak (closed form: counting register = m,
  target = |1>), noisy QPE invariants.
All runs use the bench plan (fuse=2, k_max=3: K3 group kernels); the n=16 noisy prefix against
the oracle lives in tests/test_gpu_headline.py.
"""

import numpy as np
import pytest

import workloads as W
from oracle import dense, statevector

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def Sim():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from __graft_entry__ import build
    build()
    from paper_2404_13184_b200 import Simulator
    return Simulator


def _compare_columns_with_oracle(sim, rho_ref, n, chunk_cols=256):
    N = 2 ** n
    worst_abs, num, den = 0.0, 0.0, 0.0
    for c0 in range(0, N, chunk_cols):
        cols = min(chunk_cols, N - c0)
        got = sim.get_state(c0 * N, cols * N).reshape(cols, N)   # got[j] = column c0 + j
        ref = rho_ref[:, c0:c0 + cols].T
        d = got - ref
        worst_abs = max(worst_abs, float(np.abs(d).max()))
        num += float(np.vdot(d, d).real)
        den += float(np.vdot(ref, ref).real)
    return worst_abs, np.sqrt(num / den)


def test_config3_n14_noisy_prefix_vs_oracle(Sim):
    c, nm = W.config_workload(3)
    per_layer = 14 * 5 + 7
    prefix = W.Circuit(14, c.ops[:per_layer])
    ref = dense.run(prefix, nm)
    with Sim(14) as sim:
        sim.run_circuit(prefix, nm, fuse=2, k_max=3)
        mx, rel = _compare_columns_with_oracle(sim, ref, 14)
        p = sim.probs()
    assert mx <= 1e-10 and rel <= 1e-12, (mx, rel)
    np.testing.assert_allclose(p, dense.probs(ref, 14), atol=1e-10)


def test_config3_n14_noiseless_full_depth_vs_statevector(Sim):
    c = W.random_layered(14, 100, seed=W.BASE_SEED + 3)
    psi = statevector.run(c)
    N = 2 ** 14
    rng = np.random.default_rng(3)
    with Sim(14) as sim:
        st = sim.run_circuit(c, fuse=2, k_max=3)
        assert st["ops_fused"] < 700
        p = sim.probs()
        np.testing.assert_allclose(p, np.abs(psi) ** 2, atol=1e-12)
        for col in rng.choice(N, 8, replace=False):
            got = sim.get_state(int(col) * N, N)
            assert np.abs(got - psi * np.conj(psi[col])).max() < 1e-12


def test_config3_n14_noisy_full_depth_invariants(Sim):
    c, nm = W.config_workload(3)
    N = 2 ** 14
    rng = np.random.default_rng(4)
    with Sim(14) as sim:
        sim.run_circuit(c, nm, fuse=2, k_max=3)
        p = sim.probs()                 # raises TANQ_E_STATE if |Im diag| >= 1e-6
        assert abs(p.sum() - 1.0) < 1e-9
        assert p.min() > -1e-10
        # Hermiticity on sampled entries: rho[r][c] = conj(rho[c][r])
        for _ in range(64):
            r, col = (int(x) for x in rng.integers(0, N, 2))
            a = sim.get_state(r + col * N, 1)[0]
            b = sim.get_state(col + r * N, 1)[0]
            assert abs(a - np.conj(b)) < 1e-12


def test_config4_n16_qpe_noiseless_peak(Sim):
    c = W.qpe_circuit(16)
    with Sim(16) as sim:
        sim.run_circuit(c, fuse=2, k_max=3)
        p = sim.probs()
    peak = c.m | (1 << 15)
    assert abs(p[peak] - 1.0) < 1e-10
    assert np.abs(np.delete(p, peak)).max() < 1e-10


def test_config4_n16_qpe_noisy_invariants(Sim):
    c, nm = W.config_workload(4)
    with Sim(16) as sim:
        sim.run_circuit(c, nm, fuse=2, k_max=3)
        p = sim.probs()
        ro = sim.probs(dense.readout_of(nm))
        e = sim.expect_pauli(0, 1 << 15)     # <Z_target>: target prepared in |1>
    assert abs(p.sum() - 1.0) < 1e-9 and p.min() > -1e-10
    assert abs(ro.sum() - 1.0) < 1e-9
    assert int(np.argmax(p)) == (c.m | (1 << 15))
    # two different kernels (Pauli expectation vs diagonal) agree: <Z_15> = sum_x p(x) (-1)^x_15
    x = np.arange(2 ** 16)
    z = np.where((x >> 15) & 1, -1.0, 1.0)
    assert abs(e.real - float(p @ z)) < 1e-10 and abs(e.imag) < 1e-12
    assert e.real < 0
