"""Closed-form pins of the library's C++ superoperator builder (SURVEY §4 layer 1; CPU).

The host binds every noisy gate to one Liouville superoperator (tanq_host.cpp bind_op: the
gate unitary, then coherent over-rotation, thermal relaxation and depolarizing noise in the
order of readings R4/R5, R7, R8, R10 of DESIGN.md §2).  A plan with fuse = 0 exports exactly
that superoperator (tanq_plan_get_op), so each channel and each composition order is compared
entry by entry (<= 1e-14) with the channel written out here from its definition, acting on
the 4^k matrix units E_l (vec index l = r + c 2^k) -- no library or oracle code.
"""
import math

import numpy as np
import pytest

import workloads as W

TOL = 1e-14
X = np.array([[0, 1], [1, 0]], dtype=complex)
Z = np.diag([1.0, -1.0]).astype(complex)


def cx_local():
    """CX in the local basis index b(q0) + 2 b(q1), q0 = control (tanq.h conventions)."""
    U = np.zeros((4, 4), dtype=complex)
    for i in range(4):
        U[i ^ 2 if i & 1 else i, i] = 1.0
    return U


def superop_of(channel, d):
    S = np.zeros((d * d, d * d), dtype=complex)
    for l in range(d * d):
        E = np.zeros((d, d), dtype=complex)
        E[l % d, l // d] = 1.0                      # vec index l = r + c d
        out = channel(E)
        S[:, l] = out.reshape(-1, order="F")        # column stacking
    return S


def unitary(U):
    return lambda r: U @ r @ U.conj().T


def depol(p, d):                                  # reading R7: on the gate's qubits jointly
    return lambda r: (1 - p) * r + p * np.trace(r) * np.eye(d) / d


def thermal(j, k, t1, t2, t):                     # reading R8 on local qubit j of k
    e1, e2 = math.exp(-t / t1), math.exp(-t / t2)
    d = 1 << k

    def ch(r):
        out = np.zeros_like(r)
        for a in range(d):
            for b in range(d):
                ra, rb = (a >> j) & 1, (b >> j) & 1
                if ra == rb == 0:
                    out[a, b] += r[a, b] + (1 - e1) * r[a | 1 << j, b | 1 << j]
                elif ra == rb == 1:
                    out[a, b] += e1 * r[a, b]
                else:
                    out[a, b] += e2 * r[a, b]
        return out
    return ch


def overrot(k, eps):                              # reading R10: exp(-i eps A / 2), A^2 = I
    A = X if k == 1 else np.kron(X, Z)            # 2q: Z on the control (local bit 0), X target
    return math.cos(eps / 2) * np.eye(1 << k) - 1j * math.sin(eps / 2) * A


def compose(*chs):
    def f(r):
        for ch in chs:
            r = ch(r)
        return r
    return f


def bound_superop(kind, qubits, n, qcal, gcal, order):
    from paper_2404_13184_b200.tanq import Plan
    nm = W.NoiseModel(n=n, qubits=qcal, gates={(kind, tuple(qubits)): gcal}, order=order)
    c = W.Circuit(n, [W.Op(kind, tuple(qubits))])
    qs, S = Plan(None, c, nm, fuse=0).op(0)
    assert tuple(qs) == tuple(qubits)
    return S


T1, T2, DUR = 80.0, 60.0, 400.0   # us, us, ns


@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("depol_p,thermal_on,eps", [
    (0.02, False, 0.0), (0.0, True, 0.0), (0.0, False, 0.07), (0.03, True, 0.05)])
def test_one_qubit_gate_channels(order, depol_p, thermal_on, eps):
    qcal = [W.QubitCal(t1_us=T1 if thermal_on else 0.0, t2_us=T2)]
    S = bound_superop("x", (0,), 1, qcal, W.GateCal(depol_p=depol_p, duration_ns=DUR,
                                                       overrot_rad=eps), order)
    chs = [unitary(X)]
    if eps:
        chs.append(unitary(overrot(1, eps)))
    noise = []
    if thermal_on:
        noise.append(thermal(0, 1, T1, T2, DUR * 1e-3))
    if depol_p:
        noise.append(depol(depol_p, 2))
    if order == 1:
        noise.reverse()          # order 1: depolarizing before thermal relaxation
    ref = superop_of(compose(*chs, *noise), 2)
    assert np.abs(S - ref).max() <= TOL


@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("depol_p,thermal_on,eps", [
    (0.04, False, 0.0), (0.0, True, 0.0), (0.0, False, 0.09), (0.05, True, 0.03)])
def test_two_qubit_gate_channels(order, depol_p, thermal_on, eps):
    t1 = [T1, 1.3 * T1]
    t2 = [T2, 0.9 * T2]
    qcal = [W.QubitCal(t1_us=t1[i] if thermal_on else 0.0, t2_us=t2[i]) for i in range(2)]
    S = bound_superop("cx", (0, 1), 2, qcal, W.GateCal(depol_p=depol_p, duration_ns=DUR,
                                                          overrot_rad=eps), order)
    chs = [unitary(cx_local())]
    if eps:
        chs.append(unitary(overrot(2, eps)))
    noise = []
    if thermal_on:
        noise.append(compose(thermal(0, 2, t1[0], t2[0], DUR * 1e-3),
                             thermal(1, 2, t1[1], t2[1], DUR * 1e-3)))
    if depol_p:
        noise.append(depol(depol_p, 4))
    if order == 1:
        noise.reverse()
    ref = superop_of(compose(*chs, *noise), 4)
    assert np.abs(S - ref).max() <= TOL


def test_reversed_qubit_order_relabels_the_superoperator():
    """cx on (1, 0): control is local qubit 0 = physical qubit 1; the exported superoperator is
    over qubits (1, 0) in that order, so it equals the (0, 1) one entry by entry."""
    qcal = [W.QubitCal(t1_us=T1, t2_us=T2), W.QubitCal(t1_us=T1, t2_us=T2)]
    g = W.GateCal(depol_p=0.02, duration_ns=DUR, overrot_rad=0.04)
    S01 = bound_superop("cx", (0, 1), 2, qcal, g, 0)
    S10 = bound_superop("cx", (1, 0), 2, qcal, g, 0)
    assert np.abs(S01 - S10).max() <= TOL


def test_rz_is_noiseless_and_kraus_is_sum():
    """RZ carries no noise; a user Kraus channel binds to sum_i conj(K_i) (x) K_i."""
    from paper_2404_13184_b200.tanq import Plan
    th = 0.37
    nm = W.NoiseModel(n=1, qubits=[W.QubitCal(t1_us=T1, t2_us=T2)],
                      gates={("rz", (0,)): W.GateCal(depol_p=0.5, duration_ns=DUR)})
    _, S = Plan(None, W.Circuit(1, [W.Op("rz", (0,), theta=th)]), nm, fuse=0).op(0)
    Rz = np.diag([np.exp(-0.5j * th), np.exp(0.5j * th)])
    assert np.abs(S - superop_of(unitary(Rz), 2)).max() <= TOL
    g = 0.3
    K = [np.array([[1, 0], [0, math.sqrt(1 - g)]], dtype=complex),
         np.array([[0, math.sqrt(g)], [0, 0]], dtype=complex)]
    _, S = Plan(None, W.Circuit(1, [W.Op("kraus", (0,), kraus=K)]), None, fuse=0).op(0)
    ref = superop_of(lambda r: sum(k @ r @ k.conj().T for k in K), 2)
    assert np.abs(S - ref).max() <= TOL
