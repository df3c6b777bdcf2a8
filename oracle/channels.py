"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Gate unitaries, Kraus channels and the per-gate noise binding, each written out
from its definition.  Citations: P:n = /root/reference/PAPER.md line n,
S:n = /root/reference/SPEC.md line n (conventions only).

Conventions (DESIGN.md readings):
  R2  a k-qubit matrix acting on qubits (q_0..q_{k-1}) uses local basis index
      sum_j b(q_j) 2^j  (q_0 = least significant); CX(q0=control, q1=target).
  R4  noise acts after the ideal gate.
  R5  order U -> over-rotation -> thermal -> depolarizing (order=0), or
      U -> over-rotation -> depolarizing -> thermal (order=1).
  R7  depolarizing on the gate's k qubits jointly: (1-p) rho + p I/d (x) Tr_Q rho.
  R8  thermal relaxation: amplitude damping gamma = 1-exp(-t/T1) then phase
      damping lambda = 1-exp(-2t(1/T2 - 1/(2 T1))), per qubit, over the gate
      duration; T2 <= 2 T1 ("decay probabilities as inputs").
  R9  RZ noiseless and zero-duration.
  R10 coherent over-rotation E = exp(-i eps A / 2) after the gate, A = X on 1q
      gates, A = Z(control) (x) X(target) on 2q gates.
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple

import numpy as np
import scipy.linalg

I2 = np.eye(2, dtype=complex)
PX = np.array([[0, 1], [1, 0]], dtype=complex)
PY = np.array([[0, -1j], [1j, 0]], dtype=complex)
PZ = np.array([[1, 0], [0, -1]], dtype=complex)


def _kron_local(mats: Sequence[np.ndarray]) -> np.ndarray:
    """Operator on local qubits 0..k-1 where mats[j] acts on local qubit j.

    With local index sum_j b_j 2^j, qubit k-1 is the most significant factor of
    the Kronecker product, so the product is mats[k-1] (x) ... (x) mats[0].
    """
    out = np.array([[1.0 + 0j]])
    for m in mats:
        out = np.kron(m, out)
    return out


def gate_unitary(kind: str, theta: float = 0.0) -> np.ndarray:
    """Textbook gate matrices (S:222 conventions)."""
    c, s = math.cos(theta / 2), math.sin(theta / 2)
    if kind == "id":
        return I2.copy()
    if kind == "x":
        return PX.copy()
    if kind == "y":
        return PY.copy()
    if kind == "z":
        return PZ.copy()
    if kind == "h":
        return np.array([[1, 1], [1, -1]], dtype=complex) / math.sqrt(2)
    if kind == "s":
        return np.diag([1, 1j])
    if kind == "sdg":
        return np.diag([1, -1j])
    if kind == "t":
        return np.diag([1, np.exp(1j * math.pi / 4)])
    if kind == "tdg":
        return np.diag([1, np.exp(-1j * math.pi / 4)])
    if kind == "sx":
        return 0.5 * np.array([[1 + 1j, 1 - 1j], [1 - 1j, 1 + 1j]])
    if kind == "rx":
        return np.array([[c, -1j * s], [-1j * s, c]])
    if kind == "ry":
        return np.array([[c, -s], [s, c]], dtype=complex)
    if kind == "rz":
        return np.diag([np.exp(-1j * theta / 2), np.exp(1j * theta / 2)])
    # two-qubit gates; local index = b(q0) + 2 b(q1); q0 = control for cx/cz/cp
    if kind == "cx":
        u = np.zeros((4, 4), dtype=complex)
        for i in range(4):
            ctrl, tgt = i & 1, (i >> 1) & 1
            j = ctrl | ((tgt ^ ctrl) << 1)
            u[j, i] = 1.0
        return u
    if kind == "cz":
        return np.diag([1, 1, 1, -1]).astype(complex)
    if kind == "cp":
        return np.diag([1, 1, 1, np.exp(1j * theta)])
    if kind == "swap":
        u = np.zeros((4, 4), dtype=complex)
        for i in range(4):
            j = ((i & 1) << 1) | ((i >> 1) & 1)
            u[j, i] = 1.0
        return u
    raise ValueError(f"unknown gate {kind}")


def overrotation_unitary(k: int, eps: float) -> np.ndarray:
    """R10: E = expm(-i eps A / 2); A = X (1q) or Z_control (x) X_target (2q)."""
    a = PX if k == 1 else _kron_local([PZ, PX])
    return scipy.linalg.expm(-0.5j * eps * a)


def amplitude_damping(gamma: float) -> List[np.ndarray]:
    """K0 = [[1,0],[0,sqrt(1-g)]], K1 = [[0,sqrt(g)],[0,0]]."""
    return [np.array([[1, 0], [0, math.sqrt(1 - gamma)]], dtype=complex),
            np.array([[0, math.sqrt(gamma)], [0, 0]], dtype=complex)]


def phase_damping(lam: float) -> List[np.ndarray]:
    """K0 = [[1,0],[0,sqrt(1-l)]], K1 = [[0,0],[0,sqrt(l)]]."""
    return [np.array([[1, 0], [0, math.sqrt(1 - lam)]], dtype=complex),
            np.array([[0, 0], [0, math.sqrt(lam)]], dtype=complex)]


def thermal_params(t1_us: float, t2_us: float, t_us: float) -> Tuple[float, float]:
    """R8: gamma = 1 - e^{-t/T1}, lambda = 1 - e^{-2t(1/T2 - 1/(2T1))}."""
    if t2_us > 2 * t1_us:
        raise ValueError("T2 > 2 T1")
    gamma = 1.0 - math.exp(-t_us / t1_us)
    lam = 1.0 - math.exp(-2.0 * t_us * (1.0 / t2_us - 1.0 / (2.0 * t1_us)))
    return gamma, lam


def gate_channel_sequence(op, noise) -> List[tuple]:
    """The channel list one circuit gate expands to, in application order.

    Each element is ('kraus', qubits, [K...]) or ('depol', qubits, p) or
    ('superop', qubits, S).  Noise binding follows readings R4-R10.
    """
    kind, qs = op.kind, tuple(op.qubits)
    k = len(qs)
    if kind == "u":
        return [("kraus", qs, [np.asarray(op.mat, dtype=complex)])]
    if kind == "kraus":
        return [("kraus", qs, [np.asarray(m, dtype=complex) for m in op.kraus])]
    if kind == "superop":
        return [("superop", qs, np.asarray(op.mat, dtype=complex))]
    if kind == "reset":  # reading R19: {|0><0|, |0><1|}, noiseless
        return [("kraus", qs, [np.array([[1, 0], [0, 0]], dtype=complex),
                               np.array([[0, 1], [0, 0]], dtype=complex)])]
    seq: List[tuple] = [("kraus", qs, [gate_unitary(kind, op.theta)])]
    if noise is None or kind == "rz":
        return seq
    cal = noise.gates.get((kind, qs))
    if cal is None:
        raise KeyError(f"missing calibration for {kind}{qs}")
    if cal.overrot_rad != 0.0:
        seq.append(("kraus", qs, [overrotation_unitary(k, cal.overrot_rad)]))
    thermal: List[tuple] = []
    t_us = cal.duration_ns * 1e-3
    if t_us > 0.0:
        for q in qs:
            qc = noise.qubits[q]
            if qc.t1_us > 0.0:
                g, l = thermal_params(qc.t1_us, qc.t2_us, t_us)
                thermal.append(("kraus", (q,), amplitude_damping(g)))
                thermal.append(("kraus", (q,), phase_damping(l)))
    depol = [("depol", qs, cal.depol_p)] if cal.depol_p != 0.0 else []
    if getattr(noise, "order", 0) == 0:
        seq += thermal + depol
    else:
        seq += depol + thermal
    return seq


def readout_matrix(p10: float, p01: float) -> np.ndarray:
    """Column-stochastic confusion M = [[1-P(1|0), P(0|1)], [P(1|0), 1-P(0|1)]] (R11)."""
    return np.array([[1 - p10, p01], [p10, 1 - p01]])


def noise_model_from_device(dev: dict):
    """Oracle-side reading of a device-calibration snapshot (SPEC S:365-370 schema; the
    paper's calibration-driven noise, Sec. 3.5): per qubit T1, T2 and readout
    P(0|1), P(1|0); per (gate, qubits) a depolarizing parameter from the reported gate error
    e as p = e d / (d - 1), d = 2^k (reading R6: e is the average infidelity of a
    d-dimensional depolarizing channel, F_avg = 1 - p (d - 1) / d), clamped to 1, and the
    gate duration for thermal relaxation; RZ noiseless (R9).  Written independently of the
    library's C++ parser."""
    import workloads as W  # data classes only
    n = int(dev["num_qubits"])
    qubits = [W.QubitCal(float(q["t1_us"]), float(q["t2_us"]), float(q["prob_meas1_prep0"]),
                         float(q["prob_meas0_prep1"])) for q in dev["qubits"]]
    nm = W.NoiseModel(n, qubits)
    for g in dev["gates"]:
        if g["name"] == "rz":
            continue
        qs = tuple(int(x) for x in g["qubits"])
        d = 2 ** len(qs)
        p = min(1.0, float(g["error"]) * d / (d - 1))
        nm.gates[(g["name"], qs)] = W.GateCal(p, float(g["duration_ns"]),
                                              float(g.get("overrot_rad", 0.0)))
    return nm
