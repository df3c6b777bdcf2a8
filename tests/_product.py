"""Tensor-product expectation for cluster workloads (workloads.cluster_product_workload).

A circuit whose gates never couple two clusters maps |0..0><0..0| to the tensor product of the
clusters' states: rho[r][c] = prod_cl rho_cl[r|cl][c|cl], where x|cl collects the bits of x at
the cluster's qubits (cluster qubit j -> bit j).  Each rho_cl is an oracle run on the relabelled
sub-circuit, so any entry of the full-size state has an exact oracle value.
"""
import numpy as np


def local_index(x: np.ndarray, qubits) -> np.ndarray:
    out = np.zeros_like(x)
    for j, q in enumerate(qubits):
        out |= ((x >> q) & 1) << j
    return out


def expected_columns(parts, n: int, cols: np.ndarray) -> np.ndarray:
    """parts = [(qubits, rho_cl)]; returns E[j, r] = rho[r][cols[j]] (the layout of
    sim.get_state(c * 2^n, 2^n) for one column c)."""
    N = 2 ** n
    r = np.arange(N, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    E = np.ones((len(cols), N), dtype=np.complex128)
    for qs, rho in parts:
        ri = local_index(r, qs)
        ci = local_index(cols, qs)
        E *= rho[ri[None, :], ci[:, None]]
    return E


def compare_column_blocks(sim, parts, n: int, starts, width: int):
    """max |delta|, sum |delta|^2, sum |ref|^2 over the column blocks [s, s + width), each read
    through the ABI with one tanq_get_state call."""
    N = 2 ** n
    worst, num, den = 0.0, 0.0, 0.0
    buf = np.empty(width * N, dtype=np.complex128)
    for s in sorted(int(x) for x in starts):
        got = sim.get_state(s * N, width * N, out=buf).reshape(width, N)
        E = expected_columns(parts, n, np.arange(s, s + width))
        d = got - E
        worst = max(worst, float(np.abs(d).max()))
        num += float(np.vdot(d, d).real)
        den += float(np.vdot(E, E).real)
    return worst, num, den
