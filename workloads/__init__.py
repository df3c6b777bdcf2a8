"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no gate matrices, no Kraus
operators, no superoperators).  It only emits plain data:

* circuits as lists of :class:`Op` (gate *names*, qubit indices, angles), in the
  IBM basis {ID, SX, X, RZ, CX} the paper transpiles to,
  or as the logical gates of the paper's GHZ worked example;
* device calibrations (:class:`NoiseModel`) whose value ranges are the synthetic
  recipe of DESIGN.md §"Input recipe" (the paper prints no calibration values,
  P:229);
* random complex matrices for the raw ``apply_gate`` / ``apply_channel`` /
  ``apply_superop`` entry points.

Both the oracle (``oracle/``) and the CUDA path (``paper_2404_13184_b200``)
consume these objects; neither side's arithmetic lives here.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

BASE_SEED = 240413184  # base seed 240413184 + config index

# Gate names understood by both sides.  'u' carries a user matrix, 'kraus' a
# user Kraus list, 'superop' a user superoperator (paper vec convention).
ONE_Q = ("id", "x", "y", "z", "h", "s", "sdg", "t", "tdg", "sx", "rx", "ry", "rz", "reset")
TWO_Q = ("cx", "cz", "cp", "swap")
MATRIX_KINDS = ("u", "kraus", "superop")


@dataclass
class Op:
    kind: str
    qubits: Tuple[int, ...]
    theta: float = 0.0
    mat: Optional[np.ndarray] = None          # 'u': 2^k x 2^k; 'superop': 4^k x 4^k
    kraus: Optional[List[np.ndarray]] = None  # 'kraus': list of 2^k x 2^k


@dataclass
class QubitCal:
    t1_us: float = 0.0        # <= 0 disables thermal relaxation on this qubit
    t2_us: float = 0.0
    p10: float = 0.0          # prob_meas1_prep0 = P(1|0)
    p01: float = 0.0          # prob_meas0_prep1 = P(0|1)


@dataclass
class GateCal:
    depol_p: float = 0.0      # depolarizing parameter p of E(rho) = (1-p) rho + p I/d
    duration_ns: float = 0.0  # thermal relaxation time of the gate
    overrot_rad: float = 0.0  # coherent over-rotation angle epsilon


@dataclass
class NoiseModel:
    n: int
    qubits: List[QubitCal]
    gates: Dict[Tuple[str, Tuple[int, ...]], GateCal] = field(default_factory=dict)
    order: int = 0            # 0: U, over-rot, thermal, depol ; 1: U, over-rot, depol, thermal


@dataclass
class Circuit:
    n: int
    ops: List[Op]
    name: str = ""
    # Observables for VQE-style workloads: list of (x_mask, z_mask)
    paulis: List[Tuple[int, int]] = field(default_factory=list)


# ----------------------------------------------------------------------------
# logical-gate -> IBM-basis rewriting (gate names and angles only)
# ----------------------------------------------------------------------------

def basis_h(q: int) -> List[Op]:
    return [Op("rz", (q,), math.pi / 2), Op("sx", (q,)), Op("rz", (q,), math.pi / 2)]


def basis_u3(q: int, theta: float, phi: float, lam: float) -> List[Op]:
    """U3(theta, phi, lam) ~ RZ(phi+pi) SX RZ(theta+pi) SX RZ(lam) (time order reversed)."""
    return [Op("rz", (q,), lam), Op("sx", (q,)), Op("rz", (q,), theta + math.pi),
            Op("sx", (q,)), Op("rz", (q,), phi + math.pi)]


def basis_cp(c: int, t: int, lam: float) -> List[Op]:
    return [Op("rz", (c,), lam / 2), Op("cx", (c, t)), Op("rz", (t,), -lam / 2),
            Op("cx", (c, t)), Op("rz", (t,), lam / 2)]


def basis_swap(a: int, b: int) -> List[Op]:
    return [Op("cx", (a, b)), Op("cx", (b, a)), Op("cx", (a, b))]


def lower_to_basis(ops: Sequence[Op]) -> List[Op]:
    out: List[Op] = []
    for op in ops:
        if op.kind == "h":
            out += basis_h(op.qubits[0])
        elif op.kind == "cp":
            out += basis_cp(op.qubits[0], op.qubits[1], op.theta)
        elif op.kind == "swap":
            out += basis_swap(*op.qubits)
        elif op.kind == "ry":
            out += basis_u3(op.qubits[0], op.theta, 0.0, 0.0)
        else:
            out.append(op)
    return out


# ----------------------------------------------------------------------------
# logical circuits
# ----------------------------------------------------------------------------

def qft_logical(qubits: Sequence[int], inverse: bool = False) -> List[Op]:
    """QFT on `qubits` (qubits[0] = LSB of the register integer), with final swaps."""
    m = len(qubits)
    ops: List[Op] = []
    for j in range(m - 1, -1, -1):
        ops.append(Op("h", (qubits[j],)))
        for k in range(j - 1, -1, -1):
            ops.append(Op("cp", (qubits[k], qubits[j]), math.pi / (2 ** (j - k))))
    for j in range(m // 2):
        ops.append(Op("swap", (qubits[j], qubits[m - 1 - j])))
    if inverse:
        inv = []
        for op in reversed(ops):
            inv.append(Op(op.kind, op.qubits, -op.theta))
        ops = inv
    return ops


def ghz3() -> Circuit:
    """Config 1: the paper's 3-qubit GHZ worked example: H(0); CX(0,1); CX(1,2)."""
    return Circuit(3, [Op("h", (0,)), Op("cx", (0, 1)), Op("cx", (1, 2))], name="ghz3")


def ghz3_noise(p1: float = 0.01, p2: float = 0.05, p10: float = 0.02,
               p01: float = 0.06) -> NoiseModel:
    nm = NoiseModel(3, [QubitCal(0.0, 0.0, p10, p01) for _ in range(3)])
    nm.gates[("h", (0,))] = GateCal(p1)
    nm.gates[("cx", (0, 1))] = GateCal(p2)
    nm.gates[("cx", (1, 2))] = GateCal(p2)
    return nm


def qft_circuit(n: int, x: Optional[int] = None, seed: int = BASE_SEED + 2,
                basis: bool = True) -> Circuit:
    """Config 2: X-prep of a seeded integer x, then QFT with final swaps."""
    rng = np.random.default_rng(seed)
    if x is None:
        x = int(rng.integers(0, 2 ** n))
    ops = [Op("x", (q,)) for q in range(n) if (x >> q) & 1]
    ops += qft_logical(list(range(n)))
    if basis:
        ops = lower_to_basis(ops)
    c = Circuit(n, ops, name=f"qft{n}")
    c.x = x  # type: ignore[attr-defined]
    return c


def random_layered(n: int, depth: int, seed: int = BASE_SEED + 3) -> Circuit:
    """Config 3: per layer RZ SX RZ SX RZ on every qubit, then CX on a random perfect matching."""
    rng = np.random.default_rng(seed)
    ops: List[Op] = []
    for _ in range(depth):
        for q in range(n):
            a, b, c = rng.uniform(0, 2 * math.pi, 3)
            ops += [Op("rz", (q,), a), Op("sx", (q,)), Op("rz", (q,), b), Op("sx", (q,)),
                    Op("rz", (q,), c)]
        perm = rng.permutation(n)
        for i in range(0, n - 1, 2):
            a, b = int(perm[i]), int(perm[i + 1])
            if rng.integers(0, 2):
                a, b = b, a
            ops.append(Op("cx", (a, b)))
    return Circuit(n, ops, name=f"random_layered_n{n}_d{depth}")


def qpe_circuit(n: int, m: Optional[int] = None, seed: int = BASE_SEED + 4,
                basis: bool = True) -> Circuit:
    """Config 4: QPE with n-1 counting qubits (0..n-2) and target n-1; phase phi = m / 2^(n-1)."""
    t = n - 1
    rng = np.random.default_rng(seed)
    if m is None:
        m = int(rng.integers(1, 2 ** t))
    phi = m / 2 ** t
    target = n - 1
    ops: List[Op] = [Op("x", (target,))]
    ops += [Op("h", (q,)) for q in range(t)]
    for j in range(t):
        ops.append(Op("cp", (j, target), 2 * math.pi * phi * (2 ** j)))
    ops += qft_logical(list(range(t)), inverse=True)
    if basis:
        ops = lower_to_basis(ops)
    c = Circuit(n, ops, name=f"qpe{n}")
    c.m = m  # type: ignore[attr-defined]
    return c


def vqe_paulis(n: int) -> List[Tuple[int, int]]:
    """H = sum_q (X_q X_q+1 + Y_q Y_q+1 + Z_q Z_q+1) + sum_q Z_q  ->  (x_mask, z_mask) list."""
    out = []
    for q in range(n - 1):
        pair = (1 << q) | (1 << (q + 1))
        out.append((pair, 0))        # XX
        out.append((pair, pair))     # YY
        out.append((0, pair))        # ZZ
    for q in range(n):
        out.append((0, 1 << q))      # Z
    return out


def vqe_circuit(n: int, layers: int = 2, seed: int = BASE_SEED + 5) -> Circuit:
    """Config 5: hardware-efficient ansatz, rotation layers + CX ladder (Table 1 VQE)."""
    rng = np.random.default_rng(seed)
    ops: List[Op] = []

    def rot_layer():
        for q in range(n):
            th, ph = rng.uniform(0, 2 * math.pi, 2)
            ops.extend(basis_u3(q, float(th), float(ph), 0.0))

    for _ in range(layers):
        rot_layer()
        for q in range(n - 1):
            ops.append(Op("cx", (q, q + 1)))
    rot_layer()
    return Circuit(n, ops, name=f"vqe{n}", paulis=vqe_paulis(n))


# ----------------------------------------------------------------------------
# synthetic device calibration (SURVEY §8(d) recipe; values invented)
# ----------------------------------------------------------------------------

def synthetic_calibration(circ: Circuit, seed: int, depol: bool = True, thermal: bool = True,
                          overrot: bool = False, readout: bool = True) -> NoiseModel:
    rng = np.random.default_rng(seed)
    n = circ.n
    qcal = []
    for _ in range(n):
        t1 = float(rng.uniform(50.0, 150.0))
        t2 = float(min(rng.uniform(0.4, 1.2) * t1, 2.0 * t1))
        p10 = float(rng.uniform(0.005, 0.03)) if readout else 0.0
        p01 = float(rng.uniform(0.01, 0.06)) if readout else 0.0
        qcal.append(QubitCal(t1 if thermal else 0.0, t2 if thermal else 0.0, p10, p01))
    nm = NoiseModel(n, qcal)
    keys = sorted({(op.kind, tuple(op.qubits)) for op in circ.ops
                   if op.kind not in ("rz", "reset") + MATRIX_KINDS})
    for kind, qs in keys:
        k = len(qs)
        if k == 1:
            err = float(rng.uniform(1e-4, 5e-4))
            dur = 35.5
        else:
            err = float(rng.uniform(5e-3, 2e-2))
            dur = float(rng.uniform(250.0, 550.0))
        d = 2 ** k
        # calibration "gate error" -> depolarizing parameter p = e*d/(d-1) (input recipe)
        p = min(1.0, err * d / (d - 1)) if depol else 0.0
        eps = float(rng.normal(0.0, 0.02)) if overrot else 0.0
        nm.gates[(kind, qs)] = GateCal(p, dur if thermal else 0.0, eps)
    return nm


# ----------------------------------------------------------------------------
# random matrices for the raw entry points
# ----------------------------------------------------------------------------

def random_complex(rng: np.random.Generator, shape) -> np.ndarray:
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def random_unitary(rng: np.random.Generator, d: int) -> np.ndarray:
    q, r = np.linalg.qr(random_complex(rng, (d, d)))
    return q * (np.diag(r) / np.abs(np.diag(r)))


def random_kraus(rng: np.random.Generator, d: int, m: int) -> List[np.ndarray]:
    """m Kraus operators of a random CPTP channel: columns of an isometry (md x d)."""
    v = random_unitary(rng, m * d)[:, :d]
    return [v[i * d:(i + 1) * d, :].copy() for i in range(m)]


def random_density(rng: np.random.Generator, n: int, rank: int = 3) -> np.ndarray:
    a = random_complex(rng, (2 ** n, rank))
    rho = a @ a.conj().T
    return rho / np.trace(rho)


def random_circuit(n: int, n_ops: int, seed: int, kmax: int = 2,
                   allow_matrix: bool = True) -> Circuit:
    """Mixed random circuit over named gates and (optionally) raw matrix ops."""
    rng = np.random.default_rng(seed)
    names1 = ["x", "sx", "rz", "h", "id", "y", "z", "s", "t", "rx", "ry"]
    names2 = ["cx", "cz", "cp", "swap"]
    ops: List[Op] = []
    for _ in range(n_ops):
        r = rng.random()
        if allow_matrix and r < 0.15:
            k = int(rng.integers(1, min(kmax, n) + 1))
            qs = tuple(int(x) for x in rng.choice(n, k, replace=False))
            sel = rng.integers(0, 3)
            if sel == 0:
                ops.append(Op("u", qs, mat=random_unitary(rng, 2 ** k)))
            elif sel == 1:
                ops.append(Op("kraus", qs, kraus=random_kraus(rng, 2 ** k, int(rng.integers(1, 4)))))
            else:
                # superop of a random channel is built by each side from this Kraus list
                ops.append(Op("kraus", qs, kraus=random_kraus(rng, 2 ** k, 2)))
        elif n >= 2 and r < 0.45:
            a, b = (int(x) for x in rng.choice(n, 2, replace=False))
            nm = names2[int(rng.integers(0, len(names2)))]
            ops.append(Op(nm, (a, b), float(rng.uniform(-math.pi, math.pi))))
        else:
            q = int(rng.integers(0, n))
            nm = names1[int(rng.integers(0, len(names1)))]
            ops.append(Op(nm, (q,), float(rng.uniform(-math.pi, math.pi))))
    return Circuit(n, ops, name=f"random_n{n}_{n_ops}")


def restrict(circ: Circuit, nm: Optional[NoiseModel], qubits: Sequence[int]):
    """The ops of `circ` acting inside `qubits` relabelled to 0..k-1 (qubits[j] -> j), with the
    matching slice of the noise model (relabelling only; no arithmetic of the method)."""
    loc = {q: j for j, q in enumerate(qubits)}
    ops = [Op(o.kind, tuple(loc[q] for q in o.qubits), o.theta, o.mat, o.kraus)
           for o in circ.ops if all(q in loc for q in o.qubits)]
    sub = Circuit(len(qubits), ops, name=f"{circ.name}|{tuple(qubits)}")
    if nm is None:
        return sub, None
    snm = NoiseModel(len(qubits), [nm.qubits[q] for q in qubits], order=nm.order)
    for (kind, qs), g in nm.gates.items():
        if all(q in loc for q in qs):
            snm.gates[(kind, tuple(loc[q] for q in qs))] = g
    return sub, snm


def cluster_product_workload(n: int, clusters: Sequence[Sequence[int]], layers: int, seed: int,
                             overrot: bool = True):
    """A noisy IBM-basis circuit whose gates never couple two clusters of qubits (interleaved in
    program order across clusters), so rho_out is the tensor product of the clusters' states.
    Returns (circuit, noise model, [(cluster qubits, sub-circuit, sub-noise model)]).  Used to pin
    the full-size GPU state element by element against per-cluster oracle runs."""
    rng = np.random.default_rng(seed)
    qs_all = sorted(q for c in clusters for q in c)
    assert qs_all == list(range(n)), "clusters must partition the register"
    ops: List[Op] = []
    for _ in range(layers):
        for cl in clusters:
            for q in cl:
                a, b = rng.uniform(0, 2 * math.pi, 2)
                ops += [Op("rz", (q,), a), Op("sx", (q,)), Op("rz", (q,), b)]
        for cl in clusters:
            perm = [int(x) for x in rng.permutation(list(cl))]
            for i in range(0, len(perm) - 1, 2):
                ops.append(Op("cx", (perm[i], perm[i + 1])))
            if len(perm) >= 3:
                ops.append(Op("cx", (perm[1], perm[2])))
    circ = Circuit(n, ops, name=f"clusters_n{n}_l{layers}")
    nm = synthetic_calibration(circ, seed, depol=True, thermal=True, overrot=overrot)
    return circ, nm, [(tuple(cl),) + restrict(circ, nm, cl) for cl in clusters]


# 16-qubit heavy-hex coupling of the Falcon r4P devices (ibmq_guadalupe), as pairs
GUADALUPE_COUPLING = [(0, 1), (1, 2), (1, 4), (2, 3), (3, 5), (4, 7), (5, 8), (6, 7), (7, 10),
                      (8, 9), (8, 11), (10, 12), (11, 14), (12, 13), (12, 15), (13, 14)]


def synthetic_device(n: int = 16, seed: int = BASE_SEED + 99, coupling=None,
                     name: str = "synthetic_guadalupe_like") -> dict:
    """A device-calibration snapshot in the JSON schema of SPEC S:365-370 with the synthetic
    calibration ranges of the input recipe: T1/T2, readout P(0|1)/P(1|0),
    per-gate error and duration for id/sx/x on every qubit, cx on both directions of every
    coupled pair, rz listed as noiseless.  Numbers only -- the error -> depolarizing
    conversion belongs to each side (library: tanq_device.cpp; oracle: channels.py)."""
    rng = np.random.default_rng(seed)
    coupling = list(coupling if coupling is not None else GUADALUPE_COUPLING)
    qubits = []
    for _ in range(n):
        t1 = float(rng.uniform(50.0, 150.0))
        t2 = float(min(rng.uniform(0.4, 1.2) * t1, 2.0 * t1))
        qubits.append({"t1_us": t1, "t2_us": t2, "frequency_ghz": float(rng.uniform(4.9, 5.3)),
                       "readout_length_ns": 5351.1,
                       "prob_meas0_prep1": float(rng.uniform(0.01, 0.06)),
                       "prob_meas1_prep0": float(rng.uniform(0.005, 0.03))})
    gates = []
    for q in range(n):
        for g in ("id", "sx", "x"):
            gates.append({"name": g, "qubits": [q], "error": float(rng.uniform(1e-4, 5e-4)),
                          "duration_ns": 35.5})
        gates.append({"name": "rz", "qubits": [q], "error": 0.0, "duration_ns": 0.0})
    for a, b in coupling:
        for c, t in ((a, b), (b, a)):
            gates.append({"name": "cx", "qubits": [c, t], "error": float(rng.uniform(5e-3, 2e-2)),
                          "duration_ns": float(rng.uniform(250.0, 550.0))})
    return {"name": name, "num_qubits": n, "qubits": qubits, "gates": gates,
            "coupling_map": [list(p) for p in coupling]}


CONFIGS = {
    1: "3-qubit GHZ + depolarizing gate noise + readout (paper worked example)",
    2: "10-qubit QFT, thermal relaxation + coherent over-rotation",
    3: "14-qubit random layered, depth 100, fusion up to k=3",
    4: "16-qubit QPE, calibrated device noise",
    5: "18-qubit VQE ansatz, Pauli-string expectations, 8 GPUs",
}


def config_workload(idx: int, n: Optional[int] = None, depth: Optional[int] = None):
    """(circuit, noise model) of BASELINE.json configs[idx-1]; n/depth override for scaled-down cases."""
    seed = BASE_SEED + idx
    if idx == 1:
        return ghz3(), ghz3_noise()
    if idx == 2:
        c = qft_circuit(n or 10, seed=seed)
        return c, synthetic_calibration(c, seed, depol=False, thermal=True, overrot=True,
                                        readout=False)
    if idx == 3:
        c = random_layered(n or 14, depth or 100, seed=seed)
        return c, synthetic_calibration(c, seed, depol=True, thermal=True, readout=False)
    if idx == 4:
        c = qpe_circuit(n or 16, seed=seed)
        return c, synthetic_calibration(c, seed, depol=True, thermal=True, readout=True)
    if idx == 5:
        c = vqe_circuit(n or 18, seed=seed)
        return c, synthetic_calibration(c, seed, depol=True, thermal=True, readout=True)
    raise ValueError(idx)
