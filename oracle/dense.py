"""TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

ctypes driver for oracle/dense.c plus the circuit loop of Eq. (dmsim)
(P:291-296): rho_in = |0..0><0..0| (reading R1), then every circuit gate, in
program order and unfused, expands to its channel sequence
(channels.gate_channel_sequence) and each channel is applied to the dense rho.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

from . import channels

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dense.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile dense.c with gcc (plain C99 + OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu99", "-fopenmp", "-fPIC", "-shared",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i, u64, d = ctypes.c_int, ctypes.c_uint64, ctypes.c_double
        L.orc_apply_kraus.argtypes = [P, i, i, P, i, P]
        L.orc_apply_depolarizing.argtypes = [P, i, i, P, d]
        L.orc_apply_superop.argtypes = [P, i, i, P, P]
        L.orc_diag.argtypes = [P, i, P]
        L.orc_readout.argtypes = [P, i, P, P]
        L.orc_expect_pauli.argtypes = [P, i, u64, u64, P, P]
        L.orc_invariants.argtypes = [P, i, P]
        L.orc_init_ground.argtypes = [P, i]
        for f in (L.orc_apply_kraus, L.orc_apply_depolarizing, L.orc_apply_superop, L.orc_diag,
                  L.orc_readout, L.orc_expect_pauli, L.orc_invariants, L.orc_init_ground):
            f.restype = None
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _qubits(qs: Sequence[int]) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(qs, dtype=np.int32))


def ground(n: int) -> np.ndarray:
    rho = np.empty((2 ** n, 2 ** n), dtype=np.complex128)
    lib().orc_init_ground(_ptr(rho), n)
    return rho


def apply_kraus(rho: np.ndarray, n: int, qubits: Sequence[int], kraus) -> None:
    k = len(qubits)
    K = np.ascontiguousarray(np.stack([np.asarray(m, dtype=np.complex128) for m in kraus]))
    assert K.shape[1:] == (2 ** k, 2 ** k)
    q = _qubits(qubits)
    lib().orc_apply_kraus(_ptr(rho), n, k, _ptr(q), len(kraus), _ptr(K))


def apply_depolarizing(rho: np.ndarray, n: int, qubits: Sequence[int], p: float) -> None:
    q = _qubits(qubits)
    lib().orc_apply_depolarizing(_ptr(rho), n, len(qubits), _ptr(q), float(p))


def apply_superop(rho: np.ndarray, n: int, qubits: Sequence[int], S: np.ndarray) -> None:
    q = _qubits(qubits)
    S = np.ascontiguousarray(S, dtype=np.complex128)
    lib().orc_apply_superop(_ptr(rho), n, len(qubits), _ptr(q), _ptr(S))


def apply_channel_seq(rho: np.ndarray, n: int, seq) -> None:
    for kind, qs, payload in seq:
        if kind == "kraus":
            apply_kraus(rho, n, qs, payload)
        elif kind == "depol":
            apply_depolarizing(rho, n, qs, payload)
        elif kind == "superop":
            apply_superop(rho, n, qs, payload)
        else:
            raise ValueError(kind)


def run(circuit, noise=None, rho: Optional[np.ndarray] = None, ops=None) -> np.ndarray:
    """Eq. (dmsim): apply every gate's channel sequence in program order."""
    n = circuit.n
    if rho is None:
        rho = ground(n)
    for op in (circuit.ops if ops is None else ops):
        apply_channel_seq(rho, n, channels.gate_channel_sequence(op, noise))
    return rho


def probs(rho: np.ndarray, n: int, readout=None) -> np.ndarray:
    """Re diag(rho), then the readout confusion if `readout` = (p10[], p01[])."""
    p = np.empty(2 ** n)
    lib().orc_diag(_ptr(rho), n, _ptr(p))
    if readout is not None:
        p10 = np.ascontiguousarray(readout[0], dtype=np.float64)
        p01 = np.ascontiguousarray(readout[1], dtype=np.float64)
        lib().orc_readout(_ptr(p), n, _ptr(p10), _ptr(p01))
    return p


def readout_of(noise) -> Optional[tuple]:
    if noise is None:
        return None
    return (np.array([q.p10 for q in noise.qubits]), np.array([q.p01 for q in noise.qubits]))


def expect_pauli(rho: np.ndarray, n: int, x_mask: int, z_mask: int) -> complex:
    re, im = ctypes.c_double(), ctypes.c_double()
    lib().orc_expect_pauli(_ptr(rho), n, x_mask, z_mask, ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value)


def invariants(rho: np.ndarray, n: int) -> dict:
    out = np.zeros(5)
    lib().orc_invariants(_ptr(rho), n, _ptr(out))
    return {"trace": complex(out[0], out[1]), "herm": out[2], "min_diag": out[3],
            "max_im_diag": out[4]}


def to_vec(rho: np.ndarray) -> np.ndarray:
    """Column stacking vec(rho)[r + c 2^n] = rho[r][c]."""
    return np.ascontiguousarray(rho.T).reshape(-1)
