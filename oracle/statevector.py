"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Brute-force state-vector simulator for noiseless pins: with no noise every G
is unitary and rho_out = |psi><psi| with psi = G_{m-1} ... G_0 |0..0>
(P:285-296 with pure rho_in).  Gates are applied by reshaping psi into an
n-axis tensor (axis n-1-q <-> qubit q) and contracting the target axes, a
different mechanism from both dense.c and kron_small.embed.
"""
from __future__ import annotations

import numpy as np

from . import channels


def apply(psi: np.ndarray, n: int, U: np.ndarray, qubits) -> np.ndarray:
    k = len(qubits)
    t = psi.reshape([2] * n)
    axes = [n - 1 - q for q in qubits]          # local qubit j -> tensor axis
    Ut = U.reshape([2] * (2 * k))               # row bits (b_{k-1}..b_0), col bits likewise
    # row index of U = sum_j b_j 2^j -> reshape axis (k-1-j) holds b_j
    in_axes_U = [2 * k - 1 - j for j in range(k)]
    moved = np.tensordot(Ut, t, axes=(in_axes_U, axes))
    # moved axes: U row axis i holds row bit (k-1-i), then the remaining psi axes in order
    rest = [a for a in range(n) if a not in axes]
    order = [None] * n
    for j in range(k):
        order[axes[j]] = k - 1 - j
    for i, a in enumerate(rest):
        order[a] = k + i
    return np.transpose(moved, order).reshape(-1)


def run(circuit) -> np.ndarray:
    n = circuit.n
    psi = np.zeros(2 ** n, dtype=complex)
    psi[0] = 1.0
    for op in circuit.ops:
        if op.kind in ("kraus", "superop"):
            raise ValueError("statevector oracle is noiseless-only")
        U = np.asarray(op.mat, dtype=complex) if op.kind == "u" else channels.gate_unitary(op.kind, op.theta)
        psi = apply(psi, n, U, op.qubits)
    return psi
