"""Shapes of the seeded synthetic workloads (SURVEY §8(d) recipe)."""
import workloads as W


def test_random_layered_shape():
    c = W.random_layered(14, 100)
    assert len(c.ops) == 7700                      # 14*5*100 1q + 7*100 CX
    assert sum(op.kind == "cx" for op in c.ops) == 700
    assert all(op.kind in ("rz", "sx", "cx") for op in c.ops)


def test_qpe16_shape():
    c = W.qpe_circuit(16)
    n_cx = sum(op.kind == "cx" for op in c.ops)
    assert 250 <= n_cx <= 280
    assert all(op.kind in ("rz", "sx", "cx", "x") for op in c.ops)


def test_qft10_shape():
    c = W.qft_circuit(10)
    assert sum(op.kind == "cx" for op in c.ops) == 45 * 2 + 5 * 3


def test_vqe18_paulis():
    c = W.vqe_circuit(18)
    assert len(c.paulis) == 69
    assert sum(op.kind == "cx" for op in c.ops) == 34


def test_calibration_determinism_and_ranges():
    c = W.random_layered(6, 3)
    a = W.synthetic_calibration(c, 7)
    b = W.synthetic_calibration(c, 7)
    assert a.gates == b.gates and a.qubits == b.qubits
    for qc in a.qubits:
        assert 50 <= qc.t1_us <= 150 and qc.t2_us <= 2 * qc.t1_us
    for (kind, qs), g in a.gates.items():
        assert kind != "rz"
        assert 0 <= g.depol_p <= 1
