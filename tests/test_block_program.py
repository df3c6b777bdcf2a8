"""Host-side program of the block-pipeline group kernel, checked on the CPU (-m "not gpu").

tanq_plan_block_program exports exactly what a launch would use; tests/_block_emu.py replays
its data movement in numpy (pieces, transposed loads, self-transposed blocks, offset tables,
fragment permutations) and the result must equal the plan op's superoperator applied by the
CPU oracle.  Also checks that the shared-memory placement makes the DMMA fragment accesses of
3-qubit groups above qubit 1 bank-conflict free (8 distinct 16 B banks per quarter warp).
"""
import os

import numpy as np
import pytest

import workloads as W
from oracle import dense

from _block_emu import emulate, lane_table, pair_swap, phys_of_rho


@pytest.fixture(scope="module")
def Plan():
    from paper_2404_13184_b200.tanq import Plan
    return Plan


def _cases():
    out = []
    for n, seed in ((6, 1), (6, 2), (7, 3)):
        c = W.random_circuit(n, 60, seed=5100 + seed, kmax=2, allow_matrix=True)
        out.append((f"random{n}_{seed}", c, W.synthetic_calibration(c, seed, depol=True,
                                                                    thermal=True, overrot=True)))
    c, nm = W.config_workload(4, n=7)
    out.append(("qpe7", c, nm))
    c, nm = W.config_workload(3, n=6, depth=6)
    out.append(("layered6", c, nm))
    return out


@pytest.mark.parametrize("name,circ,nm", _cases(), ids=[c[0] for c in _cases()])
@pytest.mark.parametrize("packed", [True, False])
def test_block_program_emulation_matches_oracle(Plan, name, circ, nm, packed):
    plan = Plan(None, circ, nm, fuse=2, k_max=3)
    ops = plan.ops()
    n = circ.n
    N = 2 ** n
    rng = np.random.default_rng(hash(name) % 1000 + packed)
    tested = 0
    for i, (qs, S) in enumerate(ops):
        prog = plan.block_program(i, packed=packed)
        if prog is None:
            continue
        prm, blob = prog
        assert prm.mirror == int(packed)
        rho = (W.random_density(rng, n, rank=4) if packed
               else W.random_complex(rng, (N, N)) * 0.1)
        a, P_r, P_c = phys_of_rho(rho, n)
        emulate(a, prm, blob)
        ref = np.ascontiguousarray(rho.copy())
        dense.apply_superop(ref, n, qs, S)
        aref, _, _ = phys_of_rho(ref, n)
        if packed:  # only the canonical element of each transpose pair is kept up to date
            P = np.arange(N * N)
            keep = np.array([p <= pair_swap(int(p)) for p in P])
            d = np.abs(a[keep] - aref[keep]).max()
        else:
            d = np.abs(a - aref).max()
        assert d < 1e-12, (name, i, qs, d)
        tested += 1
    assert tested >= 1


def _bank_degrees(prm, blob):
    """max lanes per 16 B bank over every quarter-warp of every fragment access."""
    u16 = blob.view(np.uint16)
    worst = []
    for q in range(prm.n_sub):
        g = prm.sub[q]
        if g.k != 2:
            continue
        rows = 32 if g.hadd >= 0 else 64
        if g.nnz:   # sparse sub-op: [nnz + 16 entries][rows] slots, one tuple per lane
            for e in range(int(g.nnz) + 16):
                for h in range(rows // 32):
                    T = np.array([int(u16[g.t_off + e * rows + h * 32 + l]) for l in range(32)])
                    for ph in range(4):
                        worst.append(np.bincount(T[8 * ph: 8 * ph + 8] % 8, minlength=8).max())
            continue
        for h in range(rows // 32):
            T = np.array([lane_table(u16, g.t_off, rows, h * 32 + l, 32)
                          for l in range(32)])               # [lane][32]
            for e in range(32):
                for ph in range(4):
                    banks = T[8 * ph: 8 * ph + 8, e] % 8
                    worst.append(np.bincount(banks, minlength=8).max())
    return max(worst) if worst else 1


def test_block_layout_bank_conflict_free(Plan):
    """QPE groups (3 qubits, all above qubit 1): in the rotation layout every B / D fragment
    quarter-warp hits 8 distinct banks; the TMA layout is accepted within one extra 2-way
    conflict of it (TANQ_BLOCK_TMA_SLACK=1), so at most 2 lanes share a bank there."""
    c, nm = W.config_workload(4, n=8)
    plan = Plan(None, c, nm, fuse=2, k_max=3)
    seen = 0
    for i, (qs, S) in enumerate(plan.ops()):
        if min(qs) < 2:
            continue
        prog = plan.block_program(i, packed=True)
        if prog is None:
            continue
        assert _bank_degrees(*prog) <= (2 if prog[0].tma else 1), (i, qs)
        seen += 1
    assert seen >= 3


K2_SNIPPET = r"""
import sys, numpy as np
sys.path.insert(0, %(root)r); sys.path.insert(0, %(tests)r)
import workloads as W
from oracle import dense
from paper_2404_13184_b200.tanq import Plan
from _block_emu import emulate, pair_swap, phys_of_rho
n = 7
rng = np.random.default_rng(3)
ops = [W.Op("kraus", (5, 6), kraus=W.random_kraus(rng, 4, 2)),
       W.Op("u", (1, 4), mat=W.random_unitary(rng, 4))]
plan = Plan(None, W.Circuit(n, ops), None, fuse=0, k_max=2)
seen = 0
for i, (qs, S) in enumerate(plan.ops()):
    for packed in (True, False):
        prog = plan.block_program(i, packed=packed)
        if prog is None:
            continue
        rho = W.random_density(rng, n, rank=3)
        a, _, _ = phys_of_rho(rho, n)
        emulate(a, *prog)
        ref = np.ascontiguousarray(rho.copy()); dense.apply_superop(ref, n, qs, S)
        aref, _, _ = phys_of_rho(ref, n)
        P = np.arange(4 ** n)
        keep = np.array([p <= pair_swap(int(p)) for p in P]) if packed else np.ones(4 ** n, bool)
        assert np.abs(a[keep] - aref[keep]).max() < 1e-12
        seen += 1
assert seen >= 2, seen
print("OK", seen)
"""


def test_block_program_standalone_k2():
    """Standalone k=2 ops with a target at physical position >= 6 run as a one-sub-op block
    program (2 group qubits + 3 free qubits per block; default, TANQ_BLOCK_K2=1)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, TANQ_BLOCK_K2="1")
    r = subprocess.run([sys.executable, "-c", K2_SNIPPET % {"root": os.path.dirname(here),
                                                             "tests": here}],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().startswith("OK"), r.stdout + r.stderr


def test_block_program_tma_layout_forced():
    """TANQ_BLOCK_TMA=1: every block program uses the TMA box layout (dims in the chosen
    order, 128 B swizzle, slot table for the cp.async path); the emulation must still match."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, TANQ_BLOCK_TMA="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        os.path.join(here, "test_block_program.py"), "-k",
                        "emulation_matches_oracle or standalone_k2"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("packed", [True, False])
def test_block_program_four_qubit_groups(Plan, packed):
    """k_max = 4: 4-qubit groups containing qubit 0 or 1 run as blocks (the group + the
    lowest free qubit); their host programs must replay to the oracle's result."""
    rng = np.random.default_rng(41 + packed)
    seen = 0
    for n, cfg in ((7, 3), (7, 4)):
        c, nm = W.config_workload(cfg, n=n, depth=4) if cfg == 3 else W.config_workload(cfg, n=n)
        plan = Plan(None, c, nm, fuse=2, k_max=4)
        N = 2 ** n
        for i, (qs, S) in enumerate(plan.ops()):
            if len(qs) != 4:
                continue
            prog = plan.block_program(i, packed=packed)
            assert prog is not None, qs                      # every 4-qubit group has 0 or 1
            rho = (W.random_density(rng, n, rank=3) if packed
                   else W.random_complex(rng, (N, N)) * 0.1)
            a, _, _ = phys_of_rho(rho, n)
            emulate(a, *prog)
            ref = np.ascontiguousarray(rho.copy())
            dense.apply_superop(ref, n, qs, S)
            aref, _, _ = phys_of_rho(ref, n)
            keep = (np.array([p <= pair_swap(int(p)) for p in range(N * N)]) if packed
                    else np.ones(N * N, bool))
            assert np.abs(a[keep] - aref[keep]).max() < 1e-12, (cfg, qs)
            seen += 1
    assert seen >= 2


SPARSE_SNIPPET = r"""
import os, sys, numpy as np
sys.path.insert(0, %(root)r); sys.path.insert(0, %(tests)r)
import workloads as W
from oracle import dense
from paper_2404_13184_b200.tanq import Plan
from _block_emu import emulate, pair_swap, phys_of_rho
rng = np.random.default_rng(5)
n = 7
c, nm = W.config_workload(4, n=n)
plan = Plan(None, c, nm, fuse=2, k_max=3)
seen = 0
for i, (qs, S) in enumerate(plan.ops()):
    for packed in (True, False):
        prog = plan.block_program(i, packed=packed)
        if prog is None or not any(prog[0].sub[j].nnz for j in range(prog[0].n_sub)):
            continue
        rho = W.random_density(rng, n, rank=3)
        a, _, _ = phys_of_rho(rho, n)
        emulate(a, *prog)
        ref = np.ascontiguousarray(rho.copy()); dense.apply_superop(ref, n, qs, S)
        aref, _, _ = phys_of_rho(ref, n)
        P = np.arange(4 ** n)
        keep = np.array([p <= pair_swap(int(p)) for p in P]) if packed else np.ones(4 ** n, bool)
        assert np.abs(a[keep] - aref[keep]).max() < 1e-12
        seen += 1
assert seen >= 4, seen
print("OK", seen)
"""


def test_block_program_sparse_subops():
    """TANQ_SPARSE_MAX=64 (read once per process: a subprocess): QPE's sparse noisy CX / CP
    superoperators become sparse DFMA sub-ops (value list, row starts, per-lane slot tables);
    the emulated program equals the oracle's superoperator on a random state."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TANQ_SPARSE_MAX="64")
    r = subprocess.run([sys.executable, "-c", SPARSE_SNIPPET % {
        "root": root, "tests": os.path.join(root, "tests")}], env=env, capture_output=True,
        text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert r.stdout.strip().splitlines()[-1].startswith("OK")


@pytest.mark.parametrize("packed", [True, False])
@pytest.mark.parametrize("case", ["qpe", "layered", "random"])
def test_block_groups_kmax5_circuit(Plan, case, packed):
    """k_max = 5 block groups (up to 5 qubits, at most 3 outside {0, 1}; each sub-op splits the
    block on its own warp-half bit, with a pair barrier where the split changes): the whole
    plan -- block programs through the emulator, other ops through the oracle -- must equal
    the oracle's run of the circuit."""
    n = 7
    if case == "qpe":
        c, nm = W.config_workload(4, n=n)
    elif case == "layered":
        c, nm = W.config_workload(3, n=n, depth=14)
    else:
        c = W.random_circuit(n, 70, seed=5300, kmax=2, allow_matrix=True)
        nm = W.synthetic_calibration(c, 3, depol=True, thermal=True, overrot=True)
    plan = Plan(None, c, nm, fuse=2, k_max=5)
    info = plan.info()
    assert info["n_k5"] > 0, info
    N = 2 ** n
    rho = dense.ground(n)
    a, P_r, P_c = phys_of_rho(rho, n)
    P = np.arange(N * N)
    noncanon = np.array([p > pair_swap(int(p)) for p in P])
    syncs = 0
    for i in range(info["ops_fused"]):
        prog = plan.block_program(i, packed=packed)
        if prog is not None:
            prm, blob = prog
            syncs += sum(int(prm.sub[j].sync) for j in range(prm.n_sub))
            emulate(a, prm, blob)
            continue
        if packed:   # restore the stale half before a full-layout op
            a[noncanon] = np.conj(a[np.array([pair_swap(int(p)) for p in P[noncanon]])])
        qs, S = plan.op(i)
        r = a[(P_r[:, None] | P_c[None, :]).reshape(-1)].reshape(N, N)
        r = np.ascontiguousarray(r)
        dense.apply_superop(r, n, qs, S)
        a[(P_r[:, None] | P_c[None, :]).reshape(-1)] = r.reshape(-1)
    if packed:
        a[noncanon] = np.conj(a[np.array([pair_swap(int(p)) for p in P[noncanon]])])
    got = a[(P_r[:, None] | P_c[None, :]).reshape(-1)].reshape(N, N)
    ref = dense.run(c, nm)
    assert np.abs(got - ref).max() < 1e-12
    assert syncs > 0   # some block group changed its warp-half bit between sub-ops


@pytest.mark.skipif(os.environ.get("TANQ_RBASIS") == "1", reason="nested run")
def test_block_programs_real_basis():
    """TANQ_RBASIS=1 (opt-in, read once per process: a nested pytest run): every group whose
    sub-ops preserve Hermiticity is transformed to the real basis (per-qubit pair tables,
    real R fragments, inverse transform before the store); the emulated programs must still
    equal the oracle, per op and over whole k_max = 5 plans."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TANQ_RBASIS="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", os.path.abspath(__file__),
                        "-k", "emulation_matches_oracle or kmax5 or four_qubit or standalone"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
