"""Host logic of the multi-GPU path on CPU (-m "not gpu"): world_size 2 and 4 over gloo.

Each rank holds one shard of vec(rho) in the engine's physical layout (row/col bits of qubit
q at 2q / 2q+1, top log2(G) bits = rank).  The ranks execute the schedule the library's
planner produces for that world size (tanq_plan_schedule: fused ops + global<->local bit
swaps) with a plain numpy mirror of the kernels, exchanging the swapped halves with gloo
send/recv exactly as the NCCL path does (pack the half {o : bit_b(o) != bit_{a-L}(rank)} in
run order, swap with partner rank ^ 2^{a-L}, unpack).  The gathered state must equal the
CPU oracle -- this pins the schedule, partner choice, half selection, run order and bit-map
bookkeeping of DESIGN.md A-6 without a GPU.
"""
import os
import socket

import numpy as np
import pytest

import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _insert_zeros(t, positions):
    for p in sorted(positions):
        lo = (1 << p) - 1
        t = ((t & ~lo) << 1) | (t & lo)
    return t


def _apply_op(shard, L, qubits, S, phys):
    k = len(qubits)
    rows = [phys[2 * q] for q in qubits]
    cols = [phys[2 * q + 1] for q in qubits]
    assert max(rows + cols) < L
    T = 1 << (L - 2 * k)
    base = _insert_zeros(np.arange(T, dtype=np.int64), rows + cols)
    d = 1 << k
    idx = np.empty((d * d, T), dtype=np.int64)
    for l in range(d * d):
        r, c = l & (d - 1), l >> k
        off = sum(((r >> j) & 1) << rows[j] for j in range(k)) + \
            sum(((c >> j) & 1) << cols[j] for j in range(k))
        idx[l] = base + off
    shard[idx] = S @ shard[idx]


def _half_offsets(L, b, v):
    e = np.arange(1 << (L - 1), dtype=np.int64)
    return ((e >> b) << (b + 1)) | (v << b) | (e & ((1 << b) - 1))


def _init_layout(n, g, parity):
    """The engine's initial layout (tanq_host.cpp init_layout): identity bit map; in the parity
    layout the top g qubits are half-global (row bit local above the pairs, global bit = r^c)."""
    phys = list(range(2 * n))
    par = 0
    if parity and n - g >= 5:  # smaller registers keep the bit layout
        F, L = n - g, 2 * n - g
        for i in range(g):
            h = F + i
            phys[2 * h], phys[2 * h + 1] = 2 * F + i, L + i
            par |= 1 << h
    return phys, par


def _parity_slot(j, s):
    """Leaving slot j of a shard with parity bit s: (ex, ey, ez) = (j >> 1, j & 1, ey ^ 1 ^ s)."""
    ex, ey = j >> 1, j & 1
    return ex, ey, ey ^ 1 ^ s


def _parity_remap(shard, L, x, y, z, s, exchange):
    """DESIGN.md §7 parity remap on one shard (parity bit s of the swapped global bit): the
    leaving half (ey ^ ez != s) goes to the partner in (octet, slot) order, the staying elements
    and the arriving ones land at bits (x, y, z) = (ey, ex, ex ^ s_sender)."""
    o = _insert_zeros(np.arange(1 << (L - 3), dtype=np.int64), [x, y, z])

    def at(bx, by, bz):
        return o | (bx << x) | (by << y) | (bz << z)
    send = np.stack([shard[at(*_parity_slot(j, s))] for j in range(4)], axis=1).reshape(-1)
    recv = exchange(send).reshape(-1, 4)
    new = shard.copy()
    for ex in (0, 1):
        for ey in (0, 1):
            ez = ey ^ s  # staying
            new[at(ey, ex, ex ^ s)] = shard[at(ex, ey, ez)]
    sp = s ^ 1
    for j in range(4):
        ex, ey, _ = _parity_slot(j, sp)
        new[at(ey, ex, ex ^ sp)] = recv[:, j]
    shard[:] = new


def _worker(rank, world, port, n, seed, out_path, layout):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["TANQ_LAYOUT"] = layout
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_13184_b200.tanq import Plan
    c = W.random_circuit(n, 40, seed=seed, kmax=3, allow_matrix=True)
    nm = W.synthetic_calibration(c, seed, depol=True, thermal=True)
    plan = Plan(None, c, nm, fuse=2, k_max=3, world_size=world)
    ops = plan.ops()
    sched = plan.schedule(world)
    g = world.bit_length() - 1
    L = 2 * n - g
    phys, par = _init_layout(n, g, layout == "parity")
    shard = np.zeros(1 << L, dtype=np.complex128)
    if rank == 0:
        shard[0] = 1.0
    n_swaps = 0

    def exchange(partner, arr):
        send = torch.from_numpy(np.ascontiguousarray(arr).view(np.float64))
        recv = torch.empty_like(send)
        reqs = [dist.isend(send, partner), dist.irecv(recv, partner)]
        for r in reqs:
            r.wait()
        return recv.numpy().view(np.complex128)

    for kind, x, y in sched:
        if kind == 0:
            qs, S = ops[x]
            _apply_op(shard, L, qs, S, phys)
        elif kind == 2:  # parity remap: half-global qubit x <-> fully local qubit y
            h, v = x, y
            bx, ba, by, bz = phys[2 * h], phys[2 * h + 1], phys[2 * v], phys[2 * v + 1]
            assert (par >> h) & 1 and not (par >> v) & 1 and ba >= L > max(bx, by, bz)
            gb = ba - L
            _parity_remap(shard, L, bx, by, bz, (rank >> gb) & 1,
                          lambda arr: exchange(rank ^ (1 << gb), arr))
            phys[2 * h], phys[2 * h + 1], phys[2 * v], phys[2 * v + 1] = by, bz, bx, ba
            par ^= (1 << h) | (1 << v)
            n_swaps += 1
        else:
            a, b = x, y
            gb = a - L
            partner = rank ^ (1 << gb)
            v = 1 - ((rank >> gb) & 1)
            off = _half_offsets(L, b, v)
            send = torch.from_numpy(np.ascontiguousarray(shard[off]).view(np.float64))
            recv = torch.empty_like(send)
            reqs = [dist.isend(send, partner), dist.irecv(recv, partner)]
            for r in reqs:
                r.wait()
            shard[off] = recv.numpy().view(np.complex128)
            ia, ib = phys.index(a), phys.index(b)
            phys[ia], phys[ib] = b, a
            n_swaps += 1
    gathered = [torch.zeros(2 * (1 << L), dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(shard.view(np.float64)))
    if rank == 0:
        full = np.concatenate([g.numpy().view(np.complex128) for g in gathered])
        N = 1 << n
        v = np.arange(N * N, dtype=np.int64)
        P = np.zeros_like(v)
        for q in range(n):
            P |= ((v >> q) & 1) << phys[2 * q]
            P |= ((v >> (n + q)) & 1) << phys[2 * q + 1]
            if (par >> q) & 1:  # parity layout: the global bit holds r ^ c
                P ^= ((v >> q) & 1) << phys[2 * q + 1]
        np.save(out_path, full[P])
        with open(out_path + ".swaps", "w") as f:
            f.write(str(n_swaps))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n,seed,layout", [
    (2, 4, 1, "bits"), (2, 5, 2, "bits"), (4, 5, 3, "bits"), (4, 4, 4, "bits"),
    (2, 6, 5, "parity"), (2, 7, 6, "parity"), (4, 7, 7, "parity"), (4, 8, 8, "parity"),
    (8, 8, 9, "parity")])
def test_distributed_schedule_matches_oracle(tmp_path, world, n, seed, layout):
    import torch.multiprocessing as mp
    from oracle import dense
    out = str(tmp_path / "vec.npy")
    mp.start_processes(_worker, args=(world, _free_port(), n, seed, out, layout), nprocs=world,
                       join=True, start_method="spawn")
    vec = np.load(out)
    c = W.random_circuit(n, 40, seed=seed, kmax=3, allow_matrix=True)
    nm = W.synthetic_calibration(c, seed, depol=True, thermal=True)
    ref = dense.to_vec(dense.run(c, nm))
    assert np.abs(vec - ref).max() < 1e-12
    assert int(open(out + ".swaps").read()) > 0       # the schedule really remapped


def test_schedule_makes_every_op_local():
    """Parity layout (the default): every remap trades a half-global qubit the next op targets
    for a fully local one it does not; every op then sees all its bits local."""
    from paper_2404_13184_b200.tanq import Plan
    for cfg, n, world in ((4, 16, 2), (4, 16, 8), (5, 18, 8), (3, 14, 4)):
        c, nm = W.config_workload(cfg, n=n)
        plan = Plan(None, c, nm, world_size=world)
        g = world.bit_length() - 1
        L = 2 * n - g
        phys, par = _init_layout(n, g, True)
        ops = plan.ops()
        seen = 0
        for kind, x, y in plan.schedule(world):
            if kind == 2:
                assert (par >> x) & 1 and not (par >> y) & 1
                assert x in ops[seen][0] and y not in ops[seen][0]
                bx, ba, by, bz = phys[2 * x], phys[2 * x + 1], phys[2 * y], phys[2 * y + 1]
                phys[2 * x], phys[2 * x + 1], phys[2 * y], phys[2 * y + 1] = by, bz, bx, ba
                par ^= (1 << x) | (1 << y)
            else:
                assert kind == 0 and x == seen
                seen += 1
                for q in ops[x][0]:
                    assert phys[2 * q] < L and phys[2 * q + 1] < L and not (par >> q) & 1
            # invariant: fully local qubits on aligned pairs below 2(n-g), row bits above
            for q in range(n):
                if (par >> q) & 1:
                    assert 2 * (n - g) <= phys[2 * q] < L <= phys[2 * q + 1]
                else:
                    assert phys[2 * q] // 2 == phys[2 * q + 1] // 2 < n - g
        assert seen == len(ops)


def test_schedule_makes_every_op_local_bits_layout():
    """The plain bit layout (TANQ_LAYOUT=bits, read once per process: a subprocess)."""
    import subprocess
    import sys
    code = ("import sys; sys.path[:0] = [%r, %r]; "
            "from test_dist_gloo import _bits_schedule_check as f; f()"
            % (ROOT, os.path.join(ROOT, "tests")))
    env = dict(os.environ, TANQ_LAYOUT="bits")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bits_schedule_check():
    from paper_2404_13184_b200.tanq import Plan
    for cfg, n, world in ((4, 16, 2), (4, 16, 8), (5, 18, 8), (3, 14, 4)):
        c, nm = W.config_workload(cfg, n=n)
        plan = Plan(None, c, nm, world_size=world)
        L = 2 * n - (world.bit_length() - 1)
        phys = list(range(2 * n))
        ops = plan.ops()
        seen = 0
        for kind, x, y in plan.schedule(world):
            if kind == 1:
                assert x >= L > y
                ia, ib = phys.index(x), phys.index(y)
                phys[ia], phys[ib] = y, x
            else:
                assert x == seen
                seen += 1
                for q in ops[x][0]:
                    assert phys[2 * q] < L and phys[2 * q + 1] < L
        assert seen == len(ops)
