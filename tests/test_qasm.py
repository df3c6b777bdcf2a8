"""OpenQASM 2.0 front-end (NEXT-4): parsing and basis lowering checked on the host (no GPU)
through the library's planner against the oracle, plus error reporting."""
import math

import numpy as np
import pytest

import workloads as W
from oracle import dense, statevector

GHZ = """OPENQASM 2.0;
include "qelib1.inc";
qreg q[3];
creg c[3];
h q[0];
cx q[0],q[1];
cx q[1],q[2];
measure q -> c;
"""


def _qasm_of(ops, n):
    lines = ["OPENQASM 2.0;", 'include "qelib1.inc";', f"qreg q[{n}];"]
    for op in ops:
        args = ",".join(f"q[{q}]" for q in op.qubits)
        if op.kind in ("rz", "rx", "ry", "cp"):
            lines.append(f"{op.kind}({op.theta!r}) {args};")
        else:
            lines.append(f"{op.kind} {args};")
    return "\n".join(lines) + "\n"


def test_ghz_parse_and_measures():
    from paper_2404_13184_b200 import QasmCircuit
    q = QasmCircuit(GHZ, to_basis=False)
    assert q.n == 3 and q.n_clbits == 3 and q.measures == [0, 1, 2]
    assert [o.kind for o in q.ops] == ["h", "cx", "cx"]
    rho = dense.run(W.Circuit(3, q.ops))
    psi = np.zeros(8)
    psi[0] = psi[7] = 1 / math.sqrt(2)
    np.testing.assert_allclose(rho, np.outer(psi, psi), atol=1e-15)


@pytest.mark.parametrize("seed", range(4))
def test_basis_lowering_preserves_the_state(seed):
    """Every logical gate lowered to {ID, SX, X, RZ, CX} gives the same rho."""
    from paper_2404_13184_b200 import QasmCircuit
    c = W.random_circuit(4, 30, seed=40 + seed, kmax=2, allow_matrix=False)
    src = _qasm_of(c.ops, 4)
    logical = QasmCircuit(src, to_basis=False)
    basis = QasmCircuit(src, to_basis=True)
    assert all(o.kind in ("id", "sx", "x", "rz", "cx") for o in basis.ops)
    assert len(basis.ops) >= len(logical.ops)
    psi = statevector.run(c)
    for q in (logical, basis):
        rho = dense.run(W.Circuit(4, q.ops))
        assert np.abs(rho - np.outer(psi, psi.conj())).max() < 1e-12


def test_expressions_registers_and_broadcast():
    from paper_2404_13184_b200 import QasmCircuit
    src = """OPENQASM 2.0;
include "qelib1.inc";
qreg a[2]; qreg b[1];
creg c[2];
rz(-pi/4 + 2*pi^2/pi) a[1];
u3(pi/2, 0.5, -(1.5)) b[0];
h a;            // broadcast over the register
cx a[0], b[0];
barrier a, b;
reset a[1];
measure a -> c;
"""
    q = QasmCircuit(src, to_basis=False)
    assert q.n == 3 and q.measures == [0, 1]
    assert abs(q.ops[0].theta - (-math.pi / 4 + 2 * math.pi)) < 1e-15
    kinds = [o.kind for o in q.ops]
    assert kinds.count("h") == 2 and kinds[-1] == "reset" and ("cx") in kinds
    assert q.ops[kinds.index("cx")].qubits == (0, 2)


@pytest.mark.parametrize("src,msg", [
    ("qreg q[2];", "OPENQASM"),
    ("OPENQASM 2.0;\nqreg q[2];\nfoo q[0];", "line 3"),
    ("OPENQASM 2.0;\nqreg q[2];\ncx q[0],q[0];", "repeated"),
    ("OPENQASM 2.0;\nqreg q[2];\nh q[5];", "out of range"),
    ("OPENQASM 2.0;\nqreg q[2];\ngate g a { h a; }", "not supported"),
    ("OPENQASM 2.0;\nqreg q[2];\nrz(pi/) q[0];", "line 3"),
])
def test_errors(src, msg):
    from paper_2404_13184_b200 import QasmCircuit, TanqError
    with pytest.raises(TanqError) as e:
        QasmCircuit(src)
    assert msg in str(e.value)
