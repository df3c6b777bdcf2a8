"""Pins of the CPU oracle against what the paper and the mathematics fix (-m "not gpu").

Each test names the passage or closed form it pins.  A plausible mistake in the
oracle (dropped Kraus term, conj on the wrong factor, swapped row/col index,
wrong qubit-bit mapping, wrong depolarizing normalisation, wrong thermal
exponent) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

import workloads as W
from oracle import channels, dense, kron_small, statevector

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _one_qubit_state(vec):
    v = np.asarray(vec, dtype=complex)
    v = v / np.linalg.norm(v)
    return np.outer(v, v.conj())


def _apply_ops(rho, n, ops, noise=None):
    for op in ops:
        dense.apply_channel_seq(rho, n, channels.gate_channel_sequence(op, noise))
    return rho


# ---------------------------------------------------------------------------
# GHZ-3: the paper's worked example
# ---------------------------------------------------------------------------

def test_ghz3_noiseless_ground_truth():
    g = json.load(open(os.path.join(GOLD, "ghz3.json")))
    rho = dense.run(W.ghz3())
    np.testing.assert_allclose(dense.probs(rho, 3), g["noiseless_diag"], atol=1e-15)
    psi = np.zeros(8)
    psi[0] = psi[7] = 1 / math.sqrt(2)
    np.testing.assert_allclose(rho, np.outer(psi, psi), atol=1e-15)


def test_ghz3_noisy_closed_form_and_readout():
    g = json.load(open(os.path.join(GOLD, "ghz3.json")))
    p1, p2 = g["p1"], g["p2"]
    nm = W.ghz3_noise(p1, p2, g["p10"], g["p01"])
    rho = dense.run(W.ghz3(), nm)
    diag = dense.probs(rho, 3)
    np.testing.assert_allclose(diag, g["diag"], atol=1e-15)
    # closed form (derivation in SURVEY §8(c)): P(000)=P(111), P(q=011)=P(100), rest p2/8
    a = (1 - p2) * ((1 - p2) / 2 + p2 / 4) + p2 / 8
    b = (1 - p2) * p2 / 4 + p2 / 8
    np.testing.assert_allclose(diag, [a, b, p2 / 8, p2 / 8, p2 / 8, p2 / 8, b, a], atol=1e-15)
    assert abs(rho[0, 7] - (1 - p1) * (1 - p2) ** 2 / 2) < 1e-15
    assert abs(rho[0, 7] - g["rho_0_7"]) < 1e-15
    ro = dense.probs(rho, 3, dense.readout_of(nm))
    np.testing.assert_allclose(ro, g["readout_probs"], atol=g["readout_tolerance"])
    # brute-force confusion: p'(y) = sum_x prod_q M[y_q][x_q] p(x)
    M = np.array([[1 - g["p10"], g["p01"]], [g["p10"], 1 - g["p01"]]])
    bf = [sum(np.prod([M[(y >> q) & 1, (x >> q) & 1] for q in range(3)]) * diag[x]
              for x in range(8)) for y in range(8)]
    np.testing.assert_allclose(ro, bf, atol=1e-15)


# ---------------------------------------------------------------------------
# channels in isolation (S:273-335 worked examples; Table 2 methodology P:238-257)
# ---------------------------------------------------------------------------

def _run1(rho0, seq):
    rho = np.ascontiguousarray(rho0.astype(complex))
    dense.apply_channel_seq(rho, 1, seq)
    return rho


def test_depolarizing_examples():
    g = json.load(open(os.path.join(GOLD, "channels.json")))
    plus = _one_qubit_state([1, 1])
    r = _run1(plus, [("depol", (0,), 0.2)])
    assert abs(r[0, 1] - g["depol_p0.2_plus_offdiag"]) < 1e-15
    np.testing.assert_allclose(r, [[0.5, 0.4], [0.4, 0.5]], atol=1e-15)
    # p = 1 -> I/2 for any input
    rng = np.random.default_rng(3)
    rho = W.random_density(rng, 1)
    np.testing.assert_allclose(_run1(rho, [("depol", (0,), 1.0)]), np.eye(2) / 2, atol=1e-15)
    # 2q joint depolarizing with p=1 -> I/4 (not the product of two 1q channels)
    rho2 = np.ascontiguousarray(W.random_density(rng, 2))
    dense.apply_depolarizing(rho2, 2, (0, 1), 1.0)
    np.testing.assert_allclose(rho2, np.eye(4) / 4, atol=1e-15)
    # fixed point and trace preservation; and the Pauli-Kraus form (independent)
    for p in np.linspace(0, 1, 51):
        for k in (1, 2):
            rho = np.ascontiguousarray(W.random_density(rng, 3))
            ref = sum(K @ rho @ K.conj().T for K in
                      [kron_small.embed(K, list(range(k)), 3) for K in kron_small.depol_pauli_kraus(k, p)])
            dense.apply_depolarizing(rho, 3, tuple(range(k)), p)
            assert np.abs(rho - ref).max() < 1e-15


def test_amplitude_and_phase_damping_examples():
    g = json.load(open(os.path.join(GOLD, "channels.json")))
    one = _one_qubit_state([0, 1])
    r = _run1(one, [("kraus", (0,), channels.amplitude_damping(0.36))])
    np.testing.assert_allclose(np.diag(r).real, g["ad_gamma0.36_one_diag"], atol=1e-15)
    plus = _one_qubit_state([1, 1])
    r = _run1(plus, [("kraus", (0,), channels.phase_damping(0.19))])
    assert abs(abs(r[0, 1]) - g["pd_lambda0.19_plus_offdiag"]) < 1e-15
    # gamma = 1 on |1> -> |0>; lambda = 1 on |+> -> diag
    r = _run1(one, [("kraus", (0,), channels.amplitude_damping(1.0))])
    np.testing.assert_allclose(r, [[1, 0], [0, 0]], atol=1e-15)
    r = _run1(plus, [("kraus", (0,), channels.phase_damping(1.0))])
    np.testing.assert_allclose(r, np.eye(2) / 2, atol=1e-15)


def test_thermal_relaxation_closed_form():
    g = json.load(open(os.path.join(GOLD, "channels.json")))["thermal_T1_100_T2_80_t1_plus"]
    nm = W.NoiseModel(1, [W.QubitCal(100.0, 80.0)])
    nm.gates[("id", (0,))] = W.GateCal(0.0, 1000.0, 0.0)  # 1000 ns = 1 us
    plus = _one_qubit_state([1, 1])
    # the thermal part only: |+> is invariant under ID
    r = np.ascontiguousarray(plus.astype(complex))
    _apply_ops(r, 1, [W.Op("id", (0,))], nm)
    assert abs(r[0, 1] - g["rho01"]) < g["tol"]
    assert abs(r[0, 1] - 0.5 * math.exp(-1 / 80)) < 1e-15
    # |1> population decays as e^{-t/T1}
    one = np.ascontiguousarray(_one_qubit_state([0, 1]).astype(complex))
    _apply_ops(one, 1, [W.Op("id", (0,))], nm)
    assert abs(one[1, 1] - math.exp(-1 / 100)) < 1e-15
    # off-diagonal decays as e^{-t/T2} for any T2 <= 2 T1 and t
    rng = np.random.default_rng(4)
    for _ in range(50):
        t1 = rng.uniform(20, 200)
        t2 = rng.uniform(0.05, 2.0) * t1
        t = rng.uniform(0, 3 * t1)
        nm = W.NoiseModel(1, [W.QubitCal(t1, t2)])
        nm.gates[("id", (0,))] = W.GateCal(0.0, t * 1e3, 0.0)
        rho = np.ascontiguousarray(W.random_density(rng, 1))
        r0 = rho.copy()
        _apply_ops(rho, 1, [W.Op("id", (0,))], nm)
        assert abs(rho[0, 1] - r0[0, 1] * math.exp(-t / t2)) < 1e-14
        assert abs(rho[1, 1] - r0[1, 1] * math.exp(-t / t1)) < 1e-14
    # t = 1e6 T1 -> |0><0|
    nm = W.NoiseModel(1, [W.QubitCal(50.0, 70.0)])
    nm.gates[("id", (0,))] = W.GateCal(0.0, 50.0 * 1e6 * 1e3, 0.0)
    rho = np.ascontiguousarray(W.random_density(rng, 1))
    _apply_ops(rho, 1, [W.Op("id", (0,))], nm)
    np.testing.assert_allclose(rho, [[1, 0], [0, 0]], atol=1e-10)
    with pytest.raises(ValueError):
        channels.thermal_params(10.0, 25.0, 1.0)


def test_readout_single_qubit_example():
    g = json.load(open(os.path.join(GOLD, "channels.json")))
    rho = np.ascontiguousarray(np.eye(2, dtype=complex) / 2)
    p = dense.probs(rho, 1, (np.array([0.02]), np.array([0.06])))
    np.testing.assert_allclose(p, g["readout_p10_0.02_p01_0.06_half"], atol=1e-15)


def test_overrotation_x_on_zero():
    # X with over-rotation eps on |0>: E X |0> = cos(eps/2)|1> - i sin(eps/2)|0> -> P(1) = cos^2(eps/2)
    for eps in (0.0, 0.013, -0.2, 1.1):
        nm = W.NoiseModel(1, [W.QubitCal()])
        nm.gates[("x", (0,))] = W.GateCal(0.0, 0.0, eps)
        rho = dense.run(W.Circuit(1, [W.Op("x", (0,))]), nm)
        assert abs(rho[1, 1] - math.cos(eps / 2) ** 2) < 1e-15
        assert abs(rho[0, 1] - (-1j * math.sin(eps / 2)) * math.cos(eps / 2)) < 1e-15
    # 2q over-rotation on CX: pure, unitary -> purity 1
    nm = W.NoiseModel(2, [W.QubitCal(), W.QubitCal()])
    nm.gates[("cx", (0, 1))] = W.GateCal(0.0, 0.0, 0.3)
    nm.gates[("h", (0,))] = W.GateCal(0.0, 0.0, 0.1)
    rho = dense.run(W.Circuit(2, [W.Op("h", (0,)), W.Op("cx", (0, 1))]), nm)
    assert abs(np.trace(rho @ rho) - 1) < 1e-14


def test_overrotation_two_qubit_axis_closed_form():
    """Reading R10: 2q over-rotation E = exp(-i eps Z_control X_target / 2) after CX.
    On |c=1,t=0>: CX -> |11>, then E|11> = cos(eps/2)|11> + i sin(eps/2)|c=1,t=0> (Z_c = -1,
    X_t flips t).  On |00>: E|00> = cos(eps/2)|00> - i sin(eps/2)|c=0,t=1>.  A swapped axis
    (X_c Z_t) would move the sin^2 weight to the other basis state, so this fixes which factor
    is Z.  Outcome index bit q = qubit q; control = qubit 0, target = qubit 1."""
    for eps in (0.3, -0.05, 1.7):
        c, s = math.cos(eps / 2), math.sin(eps / 2)
        nm = W.NoiseModel(2, [W.QubitCal(), W.QubitCal()])
        nm.gates[("x", (0,))] = W.GateCal(0.0, 0.0, 0.0)
        nm.gates[("cx", (0, 1))] = W.GateCal(0.0, 0.0, eps)
        rho = dense.run(W.Circuit(2, [W.Op("x", (0,)), W.Op("cx", (0, 1))]), nm)
        psi = np.zeros(4, dtype=complex)
        psi[3], psi[1] = c, 1j * s                      # |c=1,t=1>, |c=1,t=0>
        assert np.abs(rho - np.outer(psi, psi.conj())).max() < 1e-15
        rho = dense.run(W.Circuit(2, [W.Op("cx", (0, 1))]), nm)
        psi = np.zeros(4, dtype=complex)
        psi[0], psi[2] = c, -1j * s                     # |00>, |c=0,t=1>
        assert np.abs(rho - np.outer(psi, psi.conj())).max() < 1e-15


def test_channel_order_closed_form():
    """Reading R5: order=0 applies thermal relaxation before depolarizing, order=1 after.
    X on |0> with AD(gamma) (+ PD, diagonal-neutral) and depolarizing p, closed forms:
      order 0: P(1) = (1-p)(1-gamma) + p/2      order 1: P(1) = (1-gamma)(1-p/2)
    (the two differ by p*gamma/2, so the order is pinned, not just self-consistent)."""
    t1, t2, dur_ns, p = 40.0, 55.0, 900.0, 0.2
    gamma = 1 - math.exp(-dur_ns * 1e-3 / t1)
    for order, want in ((0, (1 - p) * (1 - gamma) + p / 2), (1, (1 - gamma) * (1 - p / 2))):
        nm = W.NoiseModel(1, [W.QubitCal(t1, t2)], order=order)
        nm.gates[("x", (0,))] = W.GateCal(p, dur_ns, 0.0)
        rho = dense.run(W.Circuit(1, [W.Op("x", (0,))]), nm)
        assert abs(rho[1, 1].real - want) < 1e-15, (order, rho[1, 1], want)
        assert abs(rho[0, 1]) < 1e-15


def test_cluster_product_structure():
    """Pins the full-size parity method of tests/test_gpu_headline.py: a circuit that never
    couples two clusters yields the tensor product of the clusters' states (oracle vs oracle
    on relabelled sub-circuits, every entry)."""
    from _product import expected_columns
    n = 7
    c, nm, subs = W.cluster_product_workload(n, [(0, 4), (1, 5, 6), (2, 3)], layers=3, seed=31)
    full = dense.run(c, nm)
    parts = [(qs, dense.run(sc, snm)) for qs, sc, snm in subs]
    E = expected_columns(parts, n, np.arange(2 ** n))          # E[c, r] = rho[r][c]
    assert np.abs(E.T - full).max() < 1e-14


def test_rz_noiseless_under_any_device():
    # RZ carries no noise even when a calibration entry exists
    nm = W.NoiseModel(1, [W.QubitCal(50.0, 60.0, 0.1, 0.1)])
    nm.gates[("rz", (0,))] = W.GateCal(0.5, 1e5, 0.3)
    seq = channels.gate_channel_sequence(W.Op("rz", (0,), 0.7), nm)
    assert len(seq) == 1


# ---------------------------------------------------------------------------
# gate matrices and conventions
# ---------------------------------------------------------------------------

def test_gate_identities():
    U = channels.gate_unitary
    assert np.allclose(U("sx") @ U("sx"), U("x"), atol=1e-15)
    assert np.allclose(U("rz", math.pi) @ U("rz", -math.pi), np.eye(2), atol=1e-15)
    assert np.allclose(U("cx") @ U("cx"), np.eye(4))
    assert np.allclose(U("swap") @ U("swap"), np.eye(4))
    # CX(q0=control, q1=target): |c=1,t=0> (index 1) <-> |c=1,t=1> (index 3)
    assert U("cx")[3, 1] == 1 and U("cx")[1, 3] == 1 and U("cx")[0, 0] == 1 and U("cx")[2, 2] == 1
    for kind in ("id", "x", "y", "z", "h", "s", "sdg", "t", "tdg", "sx", "rx", "ry", "rz", "cx", "cz", "cp", "swap"):
        u = U(kind, 0.37)
        assert np.allclose(u.conj().T @ u, np.eye(u.shape[0]), atol=1e-14)


def _equal_up_to_phase(a, b):
    i = np.unravel_index(np.argmax(np.abs(b)), b.shape)
    ph = a[i] / b[i]
    return abs(abs(ph) - 1) < 1e-12 and np.allclose(a, ph * b, atol=1e-12)


def test_basis_decompositions_equal_logical_gates():
    """workloads' IBM-basis rewrites are the logical gates up to global phase."""
    def unitary_of(ops, n):
        cols = []
        for b in range(2 ** n):
            psi = np.zeros(2 ** n, dtype=complex)
            psi[b] = 1
            for op in ops:
                psi = statevector.apply(psi, n, channels.gate_unitary(op.kind, op.theta), op.qubits)
            cols.append(psi)
        return np.array(cols).T
    assert _equal_up_to_phase(unitary_of(W.basis_h(0), 1), channels.gate_unitary("h"))
    for lam in (0.3, -1.2, math.pi / 8):
        assert _equal_up_to_phase(unitary_of(W.basis_cp(0, 1, lam), 2), channels.gate_unitary("cp", lam))
        assert _equal_up_to_phase(unitary_of(W.basis_u3(0, lam, 0, 0), 1), channels.gate_unitary("ry", lam))
    assert _equal_up_to_phase(unitary_of(W.basis_swap(0, 1), 2), channels.gate_unitary("swap"))


# ---------------------------------------------------------------------------
# whole-circuit pins
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("n", [4, 5, 6])
def test_qft_closed_form(n):
    """Noiseless QFT|x> with final swaps: rho[r][c] = e^{2 pi i x (r-c)/2^n} / 2^n."""
    c = W.qft_circuit(n, x=(0b1011 * 7) % 2 ** n, basis=True)
    rho = dense.run(c)
    N = 2 ** n
    r = np.arange(N)
    ref = np.exp(2j * math.pi * c.x * (r[:, None] - r[None, :]) / N) / N
    assert np.abs(rho - ref).max() < 1e-13


def test_qpe_noiseless_peak():
    """QPE with phi = m/2^t exactly representable: counting register = m, target = |1>."""
    c = W.qpe_circuit(6, m=19)
    p = dense.probs(dense.run(c), 6)
    expect = np.zeros(64)
    expect[19 | (1 << 5)] = 1.0
    assert np.abs(p - expect).max() < 1e-12


@pytest.mark.parametrize("seed", range(6))
def test_noiseless_equals_statevector(seed):
    """Noiseless rho = |psi><psi| from the brute-force state vector."""
    n = 4 + seed % 4
    c = W.random_circuit(n, 40, seed=seed, kmax=3)
    c.ops = [op for op in c.ops if op.kind != "kraus"]
    psi = statevector.run(c)
    rho = dense.run(c)
    assert np.abs(rho - np.outer(psi, psi.conj())).max() < 1e-13


@pytest.mark.parametrize("seed", range(8))
def test_dense_matches_independent_kronecker(seed):
    """dense.c == full-Kronecker evolution with Pauli-Kraus depolarizing (n<=5)."""
    n = 2 + seed % 4
    c = W.random_circuit(n, 30, seed=100 + seed, kmax=min(3, n))
    nm = W.synthetic_calibration(c, seed, depol=True, thermal=True, overrot=True)
    nm.order = seed % 2
    r1 = dense.run(c, nm)
    r2 = kron_small.evolve(c, nm)
    assert np.abs(r1 - r2).max() < 1e-13


@pytest.mark.parametrize("seed", range(4))
def test_dense_matches_eq_sp_literally(seed):
    """Eq. (sp) with the dense 4^n x 4^n superoperator on vec(rho), n<=3."""
    n = 1 + seed % 3
    c = W.random_circuit(n, 12, seed=200 + seed, kmax=n)
    nm = W.synthetic_calibration(c, seed, depol=True, thermal=True, overrot=True)
    r1 = dense.run(c, nm)
    r2 = kron_small.evolve_superop(c, nm)
    assert np.abs(r1 - r2).max() < 1e-13


def test_raw_superop_block_convention():
    """apply_superop uses local vec index r + c 2^k -- kron(conj U, U) == U rho U^dag."""
    rng = np.random.default_rng(8)
    for k, qs in ((1, (2,)), (2, (0, 2)), (2, (3, 1)), (3, (1, 3, 0))):
        U = W.random_unitary(rng, 2 ** k)
        S = np.kron(U.conj(), U)
        rho = np.ascontiguousarray(W.random_density(rng, 4))
        r1 = rho.copy()
        dense.apply_superop(r1, 4, qs, S)
        r2 = rho.copy()
        dense.apply_kraus(r2, 4, qs, [U])
        assert np.abs(r1 - r2).max() < 1e-14
        # and an arbitrary (non-CP) S against the explicit 4^n expansion
        S = W.random_complex(rng, (4 ** k, 4 ** k))
        r1 = rho.copy()
        dense.apply_superop(r1, 4, qs, S)
        r3 = kron_small._apply_superop_full(rho, 4, qs, S)
        assert np.abs(r1 - r3).max() < 1e-13


def test_invariants_random_noisy():
    for seed in range(5):
        n = 3
        c = W.random_circuit(n, 40, seed=300 + seed, kmax=3)
        nm = W.synthetic_calibration(c, seed, depol=True, thermal=True, overrot=True)
        rho = dense.run(c, nm)
        inv = dense.invariants(rho, n)
        assert abs(inv["trace"] - 1) < 1e-13
        assert inv["herm"] < 1e-14
        assert np.linalg.eigvalsh(rho).min() > -1e-13


def test_depolarizing_only_limit():
    """Long depolarizing-only sequences drive any state to I/2^n."""
    n = 3
    ops = []
    for _ in range(60):
        ops += [W.Op("id", (q,)) for q in range(n)]
    c = W.Circuit(n, [W.Op("h", (0,)), W.Op("cx", (0, 1))] + ops)
    nm = W.NoiseModel(n, [W.QubitCal() for _ in range(n)])
    for q in range(n):
        nm.gates[("id", (q,))] = W.GateCal(0.5, 0.0, 0.0)
    nm.gates[("h", (0,))] = W.GateCal(0.0)
    nm.gates[("cx", (0, 1))] = W.GateCal(0.0)
    rho = dense.run(c, nm)
    assert np.abs(rho - np.eye(8) / 8).max() < 1e-12


def test_pauli_expectation():
    """tr(P rho) against np.kron-built Pauli strings, and GHZ stabilisers."""
    rng = np.random.default_rng(9)
    P = [channels.I2, channels.PX, channels.PY, channels.PZ]
    n = 4
    rho = np.ascontiguousarray(W.random_density(rng, n, rank=4))
    for _ in range(30):
        xm, zm = int(rng.integers(0, 16)), int(rng.integers(0, 16))
        full = np.array([[1.0 + 0j]])
        for q in range(n):
            s = ((xm >> q) & 1) + 2 * ((zm >> q) & 1)  # 0 I, 1 X, 2 Z, 3 Y
            full = np.kron([P[0], P[1], P[3], P[2]][s], full)
        ref = np.trace(full @ rho)
        assert abs(dense.expect_pauli(rho, n, xm, zm) - ref) < 1e-14
    g = dense.run(W.ghz3())
    assert abs(dense.expect_pauli(g, 3, 0b111, 0) - 1) < 1e-15          # XXX
    assert abs(dense.expect_pauli(g, 3, 0b111, 0b110) + 1) < 1e-15      # X Y Y
    assert abs(dense.expect_pauli(g, 3, 0, 0b011) - 1) < 1e-15          # Z0 Z1
    assert abs(dense.expect_pauli(g, 3, 0, 0b001)) < 1e-15              # Z0


def test_fused_channel_composition_matches_sequence():
    """Linearity pin: the product of block superoperators (S_b S_a) applied once equals
    applying a then b -- the identity the method's fusion relies on."""
    rng = np.random.default_rng(10)
    qs = (1, 3)
    Ka = W.random_kraus(rng, 4, 3)
    Kb = W.random_kraus(rng, 4, 2)
    Sa = sum(np.kron(K.conj(), K) for K in Ka)
    Sb = sum(np.kron(K.conj(), K) for K in Kb)
    rho = np.ascontiguousarray(W.random_density(rng, 4))
    r1 = rho.copy()
    dense.apply_kraus(r1, 4, qs, Ka)
    dense.apply_kraus(r1, 4, qs, Kb)
    r2 = rho.copy()
    dense.apply_superop(r2, 4, qs, Sb @ Sa)
    assert np.abs(r1 - r2).max() < 1e-14


def test_reset_channel():
    """Reset = {|0><0|, |0><1|} (reading R19): |1><1| -> |0><0|; in general the qubit
    ends in |0> and the rest is the partial trace over it."""
    one = np.ascontiguousarray(_one_qubit_state([0, 1]).astype(complex))
    _apply_ops(one, 1, [W.Op("reset", (0,))])
    np.testing.assert_allclose(one, [[1, 0], [0, 0]], atol=1e-15)
    rng = np.random.default_rng(12)
    rho = np.ascontiguousarray(W.random_density(rng, 3))
    r = rho.copy()
    _apply_ops(r, 3, [W.Op("reset", (1,))])
    t = rho.reshape(2, 2, 2, 2, 2, 2)                  # (q2, q1, q0 ; q2', q1', q0')
    red = np.einsum("aibcid->abcd", t)                  # trace over qubit 1
    ref = np.zeros((2, 2, 2, 2, 2, 2), dtype=complex)
    ref[:, 0, :, :, 0, :] = red
    np.testing.assert_allclose(r, ref.reshape(8, 8), atol=1e-15)
