"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Independent tiny-n (n <= 5) cross-check of dense.c: every operator is expanded
to the full 2^n x 2^n matrix ("Kronecker product ... with the identity
matrix I for the other qubits") and applied as rho <- sum K_full rho K_full^dag.
Depolarizing goes through its Pauli-Kraus form (weights 1 - p(d^2-1)/d^2 on the
identity string and p/d^2 on each other string), not through the definition
dense.c uses, so the two implementations meet only at the mathematics.

`evolve_superop` additionally implements the paper's Eq. (sp) literally:
|rho(t)> = S |rho(t-1)> with the dense 4^n x 4^n S = sum conj(K) (x) K acting
on the column-stacked vec(rho), for n <= 3.
"""
from __future__ import annotations

import itertools
from typing import List, Sequence

import numpy as np

from . import channels

_PAULI = [channels.I2, channels.PX, channels.PY, channels.PZ]


def embed(op: np.ndarray, qubits: Sequence[int], n: int) -> np.ndarray:
    """G[a][b] = op[loc(a)][loc(b)] if a, b agree off the target qubits, else 0."""
    N = 2 ** n
    k = len(qubits)
    mask = sum(1 << q for q in qubits)
    G = np.zeros((N, N), dtype=complex)
    for a in range(N):
        for b in range(N):
            if (a & ~mask) != (b & ~mask):
                continue
            la = sum(((a >> q) & 1) << j for j, q in enumerate(qubits))
            lb = sum(((b >> q) & 1) << j for j, q in enumerate(qubits))
            G[a, b] = op[la, lb]
    assert op.shape == (2 ** k, 2 ** k)
    return G


def depol_pauli_kraus(k: int, p: float) -> List[np.ndarray]:
    d2 = 4 ** k
    out = []
    for idx in itertools.product(range(4), repeat=k):
        m = np.array([[1.0 + 0j]])
        for j in range(k):  # idx[j] acts on local qubit j (most significant factor last)
            m = np.kron(_PAULI[idx[j]], m)
        w = 1 - p * (d2 - 1) / d2 if all(i == 0 for i in idx) else p / d2
        out.append(np.sqrt(w) * m)
    return out


def kraus_list(seq_item, n):
    kind, qs, payload = seq_item
    if kind == "kraus":
        return [embed(K, qs, n) for K in payload]
    if kind == "depol":
        return [embed(K, qs, n) for K in depol_pauli_kraus(len(qs), payload)]
    raise ValueError(kind)


def evolve(circuit, noise=None, rho=None) -> np.ndarray:
    n = circuit.n
    assert n <= 5
    if rho is None:
        rho = np.zeros((2 ** n, 2 ** n), dtype=complex)
        rho[0, 0] = 1.0
    for op in circuit.ops:
        for item in channels.gate_channel_sequence(op, noise):
            if item[0] == "superop":
                rho = _apply_superop_full(rho, n, item[1], item[2])
                continue
            Ks = kraus_list(item, n)
            rho = sum(K @ rho @ K.conj().T for K in Ks)
    return rho


def _vec(rho):
    return rho.T.reshape(-1)


def _unvec(v, N):
    return v.reshape(N, N).T


def _full_superop_of_block(S: np.ndarray, qubits, n) -> np.ndarray:
    """Expand a 4^k block superoperator (local vec index r + c 2^k) to 4^n."""
    N = 2 ** n
    k = len(qubits)
    d = 2 ** k
    mask = sum(1 << q for q in qubits)
    F = np.zeros((N * N, N * N), dtype=complex)

    def loc(a):
        return sum(((a >> q) & 1) << j for j, q in enumerate(qubits))

    for r in range(N):
        for c in range(N):
            col = r + c * N
            for r2 in range(N):
                if (r2 & ~mask) != (r & ~mask):
                    continue
                for c2 in range(N):
                    if (c2 & ~mask) != (c & ~mask):
                        continue
                    F[r2 + c2 * N, col] = S[loc(r2) + loc(c2) * d, loc(r) + loc(c) * d]
    return F


def _apply_superop_full(rho, n, qubits, S):
    N = 2 ** n
    return _unvec(_full_superop_of_block(S, qubits, n) @ _vec(rho), N)


def evolve_superop(circuit, noise=None) -> np.ndarray:
    """Eq. (sp) literally: per channel S_full = sum conj(K_full) (x) K_full on vec(rho)."""
    n = circuit.n
    assert n <= 3
    N = 2 ** n
    v = np.zeros(N * N, dtype=complex)
    v[0] = 1.0
    for op in circuit.ops:
        for item in channels.gate_channel_sequence(op, noise):
            if item[0] == "superop":
                v = _full_superop_of_block(item[2], item[1], n) @ v
                continue
            S = sum(np.kron(K.conj(), K) for K in kraus_list(item, n))
            v = S @ v
    return _unvec(v, N)
