"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle (-m gpu).

Bar (BASELINE.json north star): max |delta rho_ij| <= 1e-10 and
||delta rho||_F / ||rho_oracle||_F <= 1e-12, same bound for probabilities and expectations.
"""
import math

import numpy as np
import pytest

import workloads as W
from oracle import dense, statevector

pytestmark = pytest.mark.gpu

ABS, REL = 1e-10, 1e-12


@pytest.fixture(scope="module")
def Sim():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from __graft_entry__ import build
    build()
    from paper_2404_13184_b200 import Simulator
    return Simulator


def rho_of(sim, n):
    N = 2 ** n
    return sim.get_state().reshape(N, N).T


def assert_parity(got, ref, abs_tol=ABS, rel_tol=REL):
    d = got - ref
    mx = np.abs(d).max()
    rel = np.linalg.norm(d) / np.linalg.norm(ref)
    assert mx <= abs_tol and rel <= rel_tol, f"max abs {mx:.3e}, rel Frobenius {rel:.3e}"


# --------------------------------------------------------------------------------------
# config 1: GHZ-3 worked example
# --------------------------------------------------------------------------------------

def test_ghz3_worked_example(Sim):
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ghz3.json")))
    c, nm = W.config_workload(1)
    for fuse in (0, 1, 2):
        with Sim(3) as sim:
            sim.run_circuit(c, nm, fuse=fuse)
            rho = rho_of(sim, 3)
            assert_parity(rho, dense.run(c, nm))
            np.testing.assert_allclose(np.diag(rho).real, g["diag"], atol=1e-15)
            assert abs(rho[0, 7] - g["rho_0_7"]) < 1e-15
            p = sim.probs(dense.readout_of(nm))
            np.testing.assert_allclose(p, g["readout_probs"], atol=g["readout_tolerance"])
    with Sim(3) as sim:
        sim.run_circuit(c)
        np.testing.assert_allclose(sim.probs(), g["noiseless_diag"], atol=1e-15)
        s1 = sim.sample(500, seed=7)
        s2 = sim.sample(500, seed=7)
        assert (s1 == s2).all()                      # reproducible per seed
        assert set(np.unique(s1)) <= {0, 7}
        assert abs((s1 == 0).sum() - 250) < 5 * math.sqrt(125)


def test_sampling_statistics(Sim):
    c, nm = W.config_workload(1)
    with Sim(3) as sim:
        sim.run_circuit(c, nm)
        ro = dense.readout_of(nm)
        p = sim.probs(ro)
        shots = 200000
        s = sim.sample(shots, seed=123, readout=ro)
        counts = np.bincount(s.astype(np.int64), minlength=8)
        sigma = np.sqrt(shots * p * (1 - p))
        assert (np.abs(counts - shots * p) <= 5 * sigma + 1).all()


# --------------------------------------------------------------------------------------
# raw entry points on random states, every kernel variant
# --------------------------------------------------------------------------------------

def _random_state(rng, n):
    return W.random_density(rng, n, rank=4)


@pytest.mark.parametrize("n,qubits", [
    (1, (0,)), (3, (0,)), (3, (2,)), (5, (1,)), (6, (5,)),        # k=1, pair / strided
    (2, (0, 1)), (4, (1, 0)), (4, (3, 0)), (6, (2, 4)), (7, (6, 5)),  # k=2
    (3, (0, 1, 2)), (5, (4, 0, 2)), (6, (1, 3, 5)), (8, (7, 2, 4)), (9, (0, 8, 3)),  # k=3
])
def test_apply_superop_random(Sim, n, qubits):
    rng = np.random.default_rng(n * 100 + sum(qubits))
    k = len(qubits)
    rho = _random_state(rng, n)
    S = W.random_complex(rng, (4 ** k, 4 ** k)) * 0.3
    with Sim(n) as sim:
        sim.set_state(dense.to_vec(rho))
        sim.apply_superop(qubits, S)
        got = rho_of(sim, n)
    ref = np.ascontiguousarray(rho.copy())
    dense.apply_superop(ref, n, qubits, S)
    assert_parity(got, ref)


@pytest.mark.parametrize("n,qubits", [(3, (1,)), (4, (0, 3)), (5, (2, 1, 4)), (7, (6,))])
def test_apply_gate_and_channel(Sim, n, qubits):
    rng = np.random.default_rng(7 + n)
    k = len(qubits)
    rho = _random_state(rng, n)
    U = W.random_unitary(rng, 2 ** k)
    Ks = W.random_kraus(rng, 2 ** k, 3)
    with Sim(n) as sim:
        sim.set_state(dense.to_vec(rho))
        sim.apply_gate(qubits, U)
        sim.apply_channel(qubits, Ks, check_cptp=True)
        got = rho_of(sim, n)
    ref = np.ascontiguousarray(rho.copy())
    dense.apply_kraus(ref, n, qubits, [U])
    dense.apply_kraus(ref, n, qubits, Ks)
    assert_parity(got, ref)


# --------------------------------------------------------------------------------------
# circuits with noise, fusion modes, shards
# --------------------------------------------------------------------------------------

@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("fuse,kmax", [(0, 2), (1, 2), (2, 2), (2, 3)])
@pytest.mark.parametrize("mirror", [True, False])
def test_random_noisy_circuits(Sim, seed, fuse, kmax, mirror):
    n = 3 + seed
    c = W.random_circuit(n, 50, seed=500 + seed, kmax=3)
    nm = W.synthetic_calibration(c, seed, depol=True, thermal=True, overrot=True)
    nm.order = seed % 2
    with Sim(n) as sim:
        sim.run_circuit(c, nm, fuse=fuse, k_max=kmax, mirror=mirror)
        got = rho_of(sim, n)
    assert_parity(got, dense.run(c, nm))


@pytest.mark.parametrize("shards", [2, 4, 8])
@pytest.mark.parametrize("seed", range(3))
def test_virtual_shards_remap(Sim, shards, seed):
    """Shards on one device: global-bit remaps (A-6) must leave the result unchanged."""
    n = 5 + seed
    c = W.random_circuit(n, 60, seed=700 + seed, kmax=3)
    nm = W.synthetic_calibration(c, seed, depol=True, thermal=True)
    ref = dense.run(c, nm)
    with Sim(n, shards) as sim:
        st = sim.run_circuit(c, nm, fuse=2, k_max=3)
        got = rho_of(sim, n)
        assert st["n_remaps"] > 0
        p = sim.probs(dense.readout_of(nm))
        e = sim.expect_pauli(0b101, 0b110)
    assert_parity(got, ref)
    np.testing.assert_allclose(p, dense.probs(ref, n, dense.readout_of(nm)), atol=ABS)
    assert abs(e - dense.expect_pauli(ref, n, 0b101, 0b110)) < ABS


@pytest.mark.parametrize("n,shards,kmax,seed", [
    (8, 2, 3, 0), (8, 4, 3, 1), (9, 8, 3, 2), (9, 2, 4, 3), (10, 4, 3, 4), (10, 2, 2, 5),
    (9, 2, 5, 6)])   # k_max 5: block groups run as their sub-ops on several shards
def test_virtual_shards_parity_packed(Sim, n, shards, kmax, seed):
    """Shard-local parity layout: with >= 6 fully local qubits every shard runs
    the packed Hermitian kernels (per-shard transpose descriptor), remaps trade a half-global
    qubit for a local one (parity_swap_kernel), and the result matches the oracle."""
    c = W.random_circuit(n, 70, seed=900 + seed, kmax=3)
    nm = W.synthetic_calibration(c, seed, depol=True, thermal=True, overrot=True)
    nm.order = seed % 2
    ref = dense.run(c, nm)
    with Sim(n, shards) as sim:
        g = shards.bit_length() - 1
        assert bin(sim.info()["parity_qubits"]).count("1") == g
        st = sim.run_circuit(c, nm, fuse=2, k_max=kmax)
        assert st["n_remaps"] > 0
        p = sim.probs(dense.readout_of(nm))                   # packed: diagonal only
        z = sim.expect_pauli(0, (1 << n) - 1)                # Z string on every qubit
        e = sim.expect_pauli(0b11 << (n - 2), 0b101 << (n - 3))  # X/Y on the half-global qubits
        got = rho_of(sim, n)
        info = sim.info()
    assert_parity(got, ref)
    np.testing.assert_allclose(p, dense.probs(ref, n, dense.readout_of(nm)), atol=ABS)
    assert abs(z - dense.expect_pauli(ref, n, 0, (1 << n) - 1)) < ABS
    assert abs(e - dense.expect_pauli(ref, n, 0b11 << (n - 2), 0b101 << (n - 3))) < ABS
    # layout invariant after the remaps: fully local qubits on aligned pairs, row bits above
    F = n - g
    for q in range(n):
        if (info["parity_qubits"] >> q) & 1:
            assert 2 * F <= info["rowpos"][q] < info["local_bits"] <= info["colpos"][q]
        else:
            assert info["rowpos"][q] // 2 == info["colpos"][q] // 2 < F


def test_virtual_shards_parity_config4(Sim):
    """QPE with calibrated noise (config 4 scaled to n = 9) on 2 and 4 shards in the parity
    layout, with the packed kernels, against the oracle: state, readout-noisy probabilities."""
    c, nm = W.config_workload(4, n=9)
    ref = dense.run(c, nm)
    for shards in (2, 4):
        with Sim(9, shards) as sim:
            st = sim.run_circuit(c, nm)
            assert st["n_remaps"] > 0
            np.testing.assert_allclose(sim.probs(dense.readout_of(nm)),
                                       dense.probs(ref, 9, dense.readout_of(nm)), atol=ABS)
            assert_parity(rho_of(sim, 9), ref)


def test_config2_qft10_thermal_overrotation(Sim):
    c, nm = W.config_workload(2)
    ref = dense.run(c, nm)
    for fuse, kmax in ((1, 2), (2, 2), (2, 3)):
        with Sim(10) as sim:
            sim.run_circuit(c, nm, fuse=fuse, k_max=kmax)
            assert_parity(rho_of(sim, 10), ref)


def test_config2_qft_noiseless_closed_form(Sim):
    n = 10
    c = W.qft_circuit(n, x=613)
    with Sim(n) as sim:
        sim.run_circuit(c)
        rho = rho_of(sim, n)
    r = np.arange(2 ** n)
    closed = np.exp(2j * math.pi * 613 * (r[:, None] - r[None, :]) / 2 ** n) / 2 ** n
    assert np.abs(rho - closed).max() < 1e-12


def test_config3_scaled_random_layered(Sim):
    c, nm = W.config_workload(3, n=9, depth=12)
    ref = dense.run(c, nm)
    for kmax in (2, 3):
        with Sim(9) as sim:
            sim.run_circuit(c, nm, fuse=2, k_max=kmax)
            assert_parity(rho_of(sim, 9), ref)


def test_config4_scaled_qpe(Sim):
    c, nm = W.config_workload(4, n=8)
    ref = dense.run(c, nm)
    for shards in (1, 2, 4):
        with Sim(8, shards) as sim:
            sim.run_circuit(c, nm)
            assert_parity(rho_of(sim, 8), ref)
            np.testing.assert_allclose(sim.probs(dense.readout_of(nm)),
                                       dense.probs(ref, 8, dense.readout_of(nm)), atol=ABS)


def test_config5_scaled_vqe_expectations(Sim):
    c, nm = W.config_workload(5, n=7)
    ref = dense.run(c, nm)
    for shards in (1, 8):
        with Sim(7, shards) as sim:
            sim.run_circuit(c, nm)
            for xm, zm in c.paulis:
                e = sim.expect_pauli(xm, zm)
                r = dense.expect_pauli(ref, 7, xm, zm)
                assert abs(e.real - r.real) < ABS and abs(e.imag) < ABS


# --------------------------------------------------------------------------------------
# edge cases and errors
# --------------------------------------------------------------------------------------

def test_empty_circuit_and_reset(Sim):
    with Sim(4) as sim:
        sim.run_circuit(W.Circuit(4, []))
        p = sim.probs()
        assert p[0] == 1.0 and p[1:].sum() == 0.0
        sim.run_circuit(W.Circuit(4, [W.Op("x", (2,))]))
        sim.reset()
        assert sim.probs()[0] == 1.0


def test_argument_errors(Sim):
    from paper_2404_13184_b200 import TanqError
    with Sim(3) as sim:
        for bad in ([W.Op("x", (3,))], [W.Op("cx", (1, 1))]):
            with pytest.raises(TanqError) as e:
                sim.run_circuit(W.Circuit(3, bad))
            assert e.value.status == 1
        nm = W.NoiseModel(3, [W.QubitCal(10.0, 25.0) for _ in range(3)])
        nm.gates[("x", (0,))] = W.GateCal(0.0, 10.0)
        with pytest.raises(TanqError):
            sim.run_circuit(W.Circuit(3, [W.Op("x", (0,))]), nm)      # T2 > 2 T1
        nm = W.NoiseModel(3, [W.QubitCal() for _ in range(3)])
        with pytest.raises(TanqError):
            sim.run_circuit(W.Circuit(3, [W.Op("sx", (1,))]), nm)     # missing calibration
        with pytest.raises(TanqError):
            sim.apply_channel((0,), [np.eye(2) * 0.5], check_cptp=True)
        # state untouched by the rejected calls
        assert sim.probs()[0] == 1.0


def test_noiseless_purity_statevector(Sim):
    for n in (6, 9):
        c = W.random_layered(n, 6, seed=n)
        psi = statevector.run(c)
        with Sim(n) as sim:
            sim.run_circuit(c, fuse=2, k_max=3)
            assert np.abs(rho_of(sim, n) - np.outer(psi, psi.conj())).max() < 1e-12


# --------------------------------------------------------------------------------------
# K3 group programs: factored k=1/k=2 sub-ops, dense k=3 sub-ops, tiny tiles
# --------------------------------------------------------------------------------------

def _group_circuit(rng, n, qs3, with_dense):
    a, b, c = qs3
    ops = []
    if with_dense:
        ops.append(W.Op("u", (c, a, b), mat=W.random_unitary(rng, 8)))
    ops += [W.Op("kraus", (a, b), kraus=W.random_kraus(rng, 4, 2)),
            W.Op("u", (b,), mat=W.random_unitary(rng, 2)),
            W.Op("kraus", (c, b), kraus=W.random_kraus(rng, 4, 3)),
            W.Op("u", (c,), mat=W.random_unitary(rng, 2)),
            W.Op("kraus", (a, c), kraus=W.random_kraus(rng, 4, 2))]
    return W.Circuit(n, ops)


@pytest.mark.parametrize("n,qs3", [(3, (0, 1, 2)), (4, (3, 0, 2)), (6, (5, 1, 3)), (8, (0, 7, 4)),
                                   (9, (8, 6, 7)), (9, (3, 5, 7)), (10, (1, 4, 6))])
@pytest.mark.parametrize("with_dense", [False, True])
def test_group_programs(Sim, n, qs3, with_dense):
    from paper_2404_13184_b200.tanq import Plan
    rng = np.random.default_rng(n * 10 + int(with_dense))
    c = _group_circuit(rng, n, qs3, with_dense)
    info = Plan(None, c, None, fuse=2, k_max=3).info()
    assert info["n_k3"] >= 1
    rho = W.random_density(rng, n, rank=3)
    with Sim(n) as sim:
        sim.set_state(dense.to_vec(rho))
        st = sim.run_circuit(c, fuse=2, k_max=3)
        assert st["n_k3"] >= 1
        got = rho_of(sim, n)
    ref = dense.run(c, None, rho=np.ascontiguousarray(rho.copy()))
    assert_parity(got, ref)


def test_plan_graph_replay(Sim):
    """CUDA-graph capture of a plan (flags bit1): first exec captures, later execs replay."""
    from paper_2404_13184_b200.tanq import Plan
    n = 7
    c, nm = W.config_workload(3, n=n, depth=5)
    ref = dense.run(c, nm)
    rng = np.random.default_rng(5)
    rho0 = W.random_density(rng, n)
    ref2 = dense.run(c, nm, rho=np.ascontiguousarray(rho0.copy()))
    with Sim(n) as sim:
        plan = Plan(sim, c, nm, fuse=2, k_max=3, graph=True)
        for _ in range(3):
            sim.reset()
            plan.exec(sim)
            assert_parity(rho_of(sim, n), ref)
        sim.set_state(dense.to_vec(rho0))
        plan.exec(sim)
        assert_parity(rho_of(sim, n), ref2)


def test_reset_in_circuit(Sim):
    c = W.random_circuit(5, 30, seed=77, kmax=2)
    c.ops.insert(12, W.Op("reset", (2,)))
    c.ops.append(W.Op("reset", (0,)))
    nm = W.synthetic_calibration(c, 77)
    with Sim(5) as sim:
        sim.run_circuit(c, nm)
        assert_parity(rho_of(sim, 5), dense.run(c, nm))


def test_mid_circuit_measurement(Sim):
    """tanq_measure: outcome probability from the diagonal, collapse P_b rho P_b / p_b."""
    n = 5
    c = W.random_circuit(n, 40, seed=88, kmax=2)
    nm = W.synthetic_calibration(c, 88)
    base = dense.run(c, nm)
    p1 = float(sum(dense.probs(base, n)[x] for x in range(2 ** n) if (x >> 3) & 1))
    ones = 0
    for seed in range(40):
        with Sim(n) as sim:
            sim.run_circuit(c, nm)
            b, pb = sim.measure(3, seed)
            ones += b
            assert abs(pb - (p1 if b else 1 - p1)) < 1e-12
            ref = np.ascontiguousarray(base.copy())
            P = np.diag([1.0 - b, float(b)]).astype(complex) / np.sqrt(pb)
            dense.apply_kraus(ref, n, (3,), [P])
            assert_parity(rho_of(sim, n), ref)
            assert abs(np.trace(rho_of(sim, n)) - 1) < 1e-12
    assert abs(ones - 40 * p1) <= 5 * np.sqrt(40 * p1 * (1 - p1)) + 1
    # GHZ: measuring one qubit collapses all three
    with Sim(3) as sim:
        sim.run_circuit(W.ghz3())
        b, pb = sim.measure(0, 123)
        assert abs(pb - 0.5) < 1e-12
        p = sim.probs()
        assert abs(p[7 if b else 0] - 1.0) < 1e-12


def test_qasm_front_end_on_gpu(Sim):
    """A QASM2 program lowered to the IBM basis, bound to a calibration and run (NEXT-4)."""
    from paper_2404_13184_b200 import QasmCircuit
    src = """OPENQASM 2.0;
include "qelib1.inc";
qreg q[4];
creg c[4];
h q[0];
cx q[0],q[1];
cp(pi/3) q[1],q[2];
u3(0.3,0.2,0.1) q[3];
swap q[2],q[3];
cz q[0],q[3];
measure q -> c;
"""
    qc = QasmCircuit(src, to_basis=True)
    circ = W.Circuit(qc.n, qc.ops)
    nm = W.synthetic_calibration(circ, 17)
    with Sim(qc.n) as sim:
        sim.run_circuit(qc, nm)
        assert_parity(rho_of(sim, qc.n), dense.run(circ, nm))



def test_mirror_mode_state_tracking(Sim):
    """Hermitian mirror mode: used only while rho is known Hermitian and ops preserve it."""
    n = 6
    rng = np.random.default_rng(31)
    c = W.random_circuit(n, 40, seed=31, kmax=3)
    nm = W.synthetic_calibration(c, 31)
    rho = W.random_density(rng, n, rank=5)
    ref = dense.run(c, nm, rho=np.ascontiguousarray(rho.copy()))
    with Sim(n) as sim:
        sim.set_state(dense.to_vec(rho))
        assert sim.check_hermitian()
        sim.run_circuit(c, nm)
        assert_parity(rho_of(sim, n), ref)
        # a non-Hermitian state is detected and handled without the mirror
        X = W.random_complex(rng, (2 ** n, 2 ** n)) * 0.01
        sim.set_state(dense.to_vec(X))
        assert not sim.check_hermitian()
        sim.run_circuit(c, nm)
        ref2 = dense.run(c, nm, rho=np.ascontiguousarray(X.copy()))
        assert np.abs(rho_of(sim, n) - ref2).max() < 1e-12
        # a non-Hermiticity-preserving superoperator in the middle of a circuit
        sim.reset()
        S = W.random_complex(rng, (16, 16)) * 0.2
        c2 = W.Circuit(n, c.ops[:20] + [W.Op("superop", (1, 4), mat=S)] + c.ops[20:])
        sim.run_circuit(c2, nm)
        assert_parity(rho_of(sim, n), dense.run(c2, nm))


def test_dist_handle_world1(Sim):
    """tanq_create_dist with world_size 1 (the torchrun N=1 path) matches the oracle."""
    c, nm = W.config_workload(4, n=6)
    with Sim(6, world_size=1, rank=0, device=0) as sim:
        sim.run_circuit(c, nm)
        assert_parity(rho_of(sim, 6), dense.run(c, nm))
        assert sim.info()["world_size"] == 1


def test_packed_layout_transitions(Sim):
    """Packed Hermitian layout bookkeeping: diagonal reads stay packed, X/Y expectations and
    get_state unpack, a non-Hermiticity-preserving op mid-plan unpacks inside a CUDA graph,
    and graph replays recapture when the starting layout differs."""
    from paper_2404_13184_b200.tanq import Plan
    rng = np.random.default_rng(77)
    n = 7
    c, nm = W.config_workload(3, n=n, depth=4)
    S = W.random_complex(rng, (16, 16)) * 0.2            # not Hermiticity-preserving
    c_bad = W.Circuit(n, c.ops[:25] + [W.Op("superop", (2, 5), mat=S)] + c.ops[25:])
    ref, ref_bad = dense.run(c, nm), dense.run(c_bad, nm)
    ro = dense.readout_of(nm)
    with Sim(n) as sim:
        # herm plan: probabilities (diagonal) straight from the packed layout, then an XY term
        sim.run_circuit(c, nm)
        np.testing.assert_allclose(sim.probs(ro), dense.probs(ref, n, ro), atol=ABS)
        for xm, zm in ((0b0000011, 0b0000001), (0b1010000, 0), (0, 0b1100110)):
            assert abs(sim.expect_pauli(xm, zm) - dense.expect_pauli(ref, n, xm, zm)) < ABS
        # continue from the (now unpacked) state with more packed ops, then read everything
        sim.run_circuit(c, nm)
        ref2 = dense.run(c, nm, rho=np.ascontiguousarray(ref.copy()))
        assert sim.check_hermitian()
        assert_parity(rho_of(sim, n), ref2)
        # graph replays of a plan whose middle op is not Hermiticity-preserving
        plan = Plan(sim, c_bad, nm, fuse=2, k_max=3, graph=True)
        for _ in range(3):                              # (rho is no longer Hermitian: its
            sim.reset()                                 #  diagonal has an imaginary part, so
            plan.exec(sim)                              #  compare the full state)
            assert_parity(rho_of(sim, n), ref_bad)
        with pytest.raises(Exception):
            sim.probs()                                 # E_STATE: |Im diag| >= 1e-6
        # a Hermitian plan replayed from a packed start and from an unpacked start
        plan2 = Plan(sim, c, nm, fuse=2, k_max=3, graph=True)
        sim.reset()
        plan2.exec(sim)                                 # ends packed
        plan2.exec(sim)                                 # starts packed
        assert_parity(rho_of(sim, n), ref2)             # get_state unpacks
        plan2.exec(sim)                                 # starts unpacked: recapture
        ref3 = dense.run(c, nm, rho=np.ascontiguousarray(ref2.copy()))
        assert_parity(rho_of(sim, n), ref3)


def test_run_circuit_plan_cache(Sim):
    """tanq_run_circuit caches plans by an exact key (ops, payloads, calibration, options):
    repeated runs replay the cached plan (as a CUDA graph from the second run), and any change
    of a matrix payload or calibration number plans afresh."""
    n = 6
    c = W.random_circuit(n, 50, seed=4242, kmax=3)
    nm = W.synthetic_calibration(c, 4242, depol=True, thermal=True, overrot=True)
    ref = dense.run(c, nm)
    with Sim(n) as sim:
        for it in range(4):
            sim.reset()
            st = sim.run_circuit(c, nm)
            assert_parity(rho_of(sim, n), ref)
            if it:
                assert st["plan_ms"] == 0.0
        # a different calibration value -> a different plan
        key = next(iter(nm.gates))
        nm.gates[key].depol_p *= 0.5
        ref2 = dense.run(c, nm)
        sim.reset()
        st = sim.run_circuit(c, nm)
        assert st["plan_ms"] > 0.0
        assert_parity(rho_of(sim, n), ref2)
        # a different user matrix payload (same shapes) -> a different plan
        i = next(j for j, o in enumerate(c.ops) if o.kind in ("u", "kraus"))
        op = c.ops[i]
        if op.kind == "u":
            op.mat = op.mat @ np.diag(np.exp(1j * np.arange(op.mat.shape[0])))
        else:
            op.kraus = [K * np.exp(0.3j) for K in op.kraus]
        ref3 = dense.run(c, nm)
        sim.reset()
        sim.run_circuit(c, nm)
        assert_parity(rho_of(sim, n), ref3)


def test_create_ex_on_torch_buffer(Sim):
    """tanq_create_ex: the state lives in a caller-owned torch tensor; after
    get_state (which unpacks) the tensor holds vec(rho) in the physical interleaved layout:
    element (r, c) at sum_q r_q 2^(2q) + c_q 2^(2q+1)."""
    import torch
    n = 6
    N = 2 ** n
    c = W.random_circuit(n, 40, seed=606, kmax=3)
    nm = W.synthetic_calibration(c, 606, depol=True, thermal=True, overrot=True)
    ref = dense.run(c, nm)
    buf = torch.empty(4 ** n, dtype=torch.complex128, device="cuda")
    with Sim(n, buffers=[buf]) as sim:
        torch.cuda.synchronize()
        assert abs(buf[0].item() - 1) == 0 and torch.count_nonzero(buf).item() == 1
        sim.run_circuit(c, nm)
        got = rho_of(sim, n)
        assert_parity(got, ref)
        sim.sync()
        raw = buf.cpu().numpy()
    r = np.arange(N)
    P_r = np.zeros(N, dtype=np.int64)
    for q in range(n):
        P_r |= ((r >> q) & 1) << (2 * q)
    phys = P_r[:, None] | (P_r[None, :] << 1)           # [row, col] -> physical index
    assert np.abs(raw[phys] - ref).max() <= 1e-10
