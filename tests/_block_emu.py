"""numpy emulation of the block-pipeline kernel's data movement (tanq_block.cu) from the program
the host builds (tanq_plan_block_program): piece loads from in-place / transposed positions,
the in-shared-memory transposition fixups, self-transposed blocks, every sub-op's fragment
offset tables and A fragments, and the stores.  It checks the host-side program (placement,
tables, fragment permutations, packed-layout decisions) on the CPU; the arithmetic order is not
emulated (a complex matrix product stands in for the DMMA sequence).
"""
import numpy as np

M55 = 0x5555555555555555


def pair_swap(x: int) -> int:
    return ((x & M55) << 1) | ((x >> 1) & M55)


def pswap_bits(x: int, nbits: int) -> int:
    m = int("01" * (nbits // 2), 2)
    return ((x & m) << 1) | ((x >> 1) & m)


def insert_zeros(t: int, lo_masks) -> int:
    for m in lo_masks:
        t = ((t & ~m) << 1) | (t & m)
    return t


def phys_of_rho(rho: np.ndarray, n: int) -> np.ndarray:
    """a[P] with P's bit 2q = row bit q, bit 2q+1 = column bit q (initial interleaved layout)."""
    N = 2 ** n
    a = np.empty(N * N, dtype=np.complex128)
    r = np.arange(N)
    P_r = np.zeros(N, dtype=np.int64)
    for q in range(n):
        P_r |= ((r >> q) & 1) << (2 * q)
    P_c = P_r << 1
    a[(P_r[:, None] | P_c[None, :]).reshape(-1)] = rho.reshape(-1)
    return a, P_r, P_c


def lane_table(u16, t_off, rows, row, n):
    """the n offsets of table row `row` (layout [n / 8 chunks][rows][8 uint16])."""
    return np.array([u16[t_off + ((e >> 3) * rows + row) * 8 + (e & 7)] for e in range(n)],
                    dtype=np.int64)


def emulate(a: np.ndarray, prm, blob: np.ndarray, check=True):
    """Run the block program on the physical-order state a (in place)."""
    lo = [int(x) for x in prm.lo_mask]
    goff = [int(x) for x in prm.piece_goff]
    start = [int(x) for x in prm.piece_start]
    sbp = [int(x) for x in prm.start_by_pidx]
    mirror = bool(prm.mirror)
    dbl = blob.view(np.float64)
    u16 = blob.view(np.uint16)
    tma = bool(getattr(prm, "tma", 0))
    if tma:   # box order (dims as the tensor map lists them) + 128 B swizzle
        tab = u16[int(prm.slot_off):int(prm.slot_off) + 1024]
        assert sorted(int(x) for x in tab) == list(range(1024))
        # the slot table must be the box order of the tensor-map dims, swizzled: rebuild it
        pos_of = []            # physical position of block bit j
        for j in range(10):
            m = int(prm.lo_mask[j])
            pos_of.append((m + 1).bit_length() - 1)
        sb = [0, 1, 2] + [None] * 7
        nxt = 3
        for d in range(1, int(prm.tdims)):
            for b in range(int(prm.tbox[d])):
                j = pos_of.index(int(prm.tlo[d]) + b)
                sb[j] = nxt
                nxt += 1
        def slot(idx):
            s_ = sum(1 << sb[j] for j in range(10) if (idx >> j) & 1)
            return s_ ^ ((s_ >> 3) & 7)
        assert all(int(tab[i]) == slot(i) for i in range(1024))
    else:
        def slot(idx):
            return sbp[idx >> 4] + (idx & 15)
        assert sorted(start) == sorted(sbp)
    for i in range(int(prm.n_blocks)):
        if mirror and i > pair_swap(i):
            continue
        base = insert_zeros(i, lo)
        self_t = mirror and pair_swap(base) == base
        st = np.zeros(1032, dtype=np.complex128)
        trs = []
        for j in range(64):
            e0 = base + goff[j]
            em = pair_swap(e0)
            tr = mirror and not self_t and e0 > em
            src = em if tr else e0
            pidx = j if tma else [q for q in range(64) if sbp[q] == start[j]][0]
            for t in range(16):   # element t of the loaded piece -> its block slot
                tt = pswap_bits(t, 4) if tr else t
                st[slot(pidx * 16 + tt)] = np.conj(a[src + t]) if tr else a[src + t]
            trs.append((tr, src, pidx))
        if self_t:
            for idx in range(1024):
                idm = pswap_bits(idx, 10)
                if idx > idm:
                    st[slot(idx)] = np.conj(st[slot(idm)])
        rb_nq = int(getattr(prm, "rb_nq", 0))
        if rb_nq:   # real basis: forward transform of each group qubit's (10, 01) pairs
            RT = u16[int(prm.rb_off):int(prm.rb_off) + rb_nq * 512].reshape(rb_nq, 256, 2)
            for t in range(rb_nq):
                if check:
                    assert len(set(RT[t].reshape(-1).tolist())) == 512
                for o1, o2 in RT[t]:
                    x1, x2 = st[o1], st[o2]
                    st[o1], st[o2] = x1 + x2, 1j * (x2 - x1)
        for q in range(int(prm.n_sub)):
            g = prm.sub[q]
            for h in range(2):
                shared = g.hadd >= 0                        # per sub-op warp-half bit
                row0 = 0 if shared else h * 32             # table row of lane 0
                rows = 32 if shared else 64
                add = h * g.hadd if shared else 0          # slot offset of this half
                if g.k == 2 and g.nnz:   # sparse DFMA sub-op: lane = tuple
                    nnz = int(g.nnz)
                    sv = dbl[g.a_off:g.a_off + 2 * nnz].reshape(nnz, 2) @ np.array([1, 1j])
                    rs = [int(v) for v in u16[(g.a_off + 2 * nnz) * 4:(g.a_off + 2 * nnz) * 4 + 17]]
                    assert rs[0] == 0 and rs[16] == nnz and rs == sorted(rs)
                    rd, wr = [], []
                    for lane in range(32):
                        r = row0 + lane
                        tin = [add + int(u16[g.t_off + e * rows + r]) for e in range(nnz)]
                        tout = [add + int(u16[g.t_off + (nnz + i) * rows + r]) for i in range(16)]
                        x = {o: st[o] for o in tin}
                        y = np.zeros(16, dtype=np.complex128)
                        for i in range(16):
                            for e in range(rs[i], rs[i + 1]):
                                y[i] += sv[e] * x[tin[e]]
                        st[tout] = y
                        rd += tin
                        wr += tout
                    if check:   # the inputs are members of the lane's own 16-member tuple
                        assert len(set(wr)) == 512 and set(rd) <= set(wr)
                elif g.k == 2:
                    if rb_nq:   # real fragments [4 ks][32 lanes][2 mt]: R only
                        a_ = dbl[g.a_off:g.a_off + 256].reshape(4, 32, 2).transpose(2, 0, 1)
                        b_ = np.zeros_like(a_)
                        F = None
                    else:
                        F = dbl[g.a_off:g.a_off + 768].reshape(3, 4, 32, 2).transpose(0, 3, 1, 2)
                        a_ = F[0]
                        b_ = F[2] + F[0]
                    if check and F is not None:
                        assert np.allclose(F[1], -(a_ + b_), atol=1e-14, rtol=1e-14)
                        for mt in range(2):       # tiles the kernel skips are exactly zero
                            for ks in range(4):
                                if not (int(g.tmask) >> (mt * 4 + ks)) & 1 and F is not None:
                                    assert not F[:, mt, ks, :].any(), (q, mt, ks)
                    S = np.zeros((16, 16), dtype=np.complex128)
                    X = np.zeros((16, 32), dtype=np.complex128)
                    rd, wr = [], []
                    for lane in range(32):
                        T = add + lane_table(u16, g.t_off, rows, row0 + lane, 32)
                        c4, r4 = lane & 3, lane >> 2
                        for mt in range(2):
                            for ks in range(4):
                                S[mt * 8 + r4, ks * 4 + c4] = a_[mt, ks, lane] + 1j * b_[mt, ks, lane]
                        for ks in range(4):
                            for j in range(4):
                                X[ks * 4 + c4, 8 * j + r4] = st[T[ks * 4 + j]]
                                rd.append(int(T[ks * 4 + j]))
                    Y = S @ X
                    for lane in range(32):
                        T = add + lane_table(u16, g.t_off, rows, row0 + lane, 32)
                        c4, r4 = lane & 3, lane >> 2
                        for mt in range(2):
                            for j in range(4):
                                for c in range(2):
                                    off = int(T[16 + (mt * 4 + j) * 2 + c])
                                    st[off] = Y[8 * mt + r4, 8 * j + 2 * c4 + c]
                                    wr.append(off)
                    if check:
                        assert len(set(rd)) == 512 and set(rd) == set(wr)
                else:
                    S = (dbl[g.a_off:g.a_off + 32].reshape(16, 2) @ np.array([1, 1j])).reshape(4, 4)
                    rd = []
                    for lane in range(32):
                        T = add + lane_table(u16, g.t_off, rows, row0 + lane, 16)
                        for j in range(4):
                            offs = [int(T[j * 4 + m]) for m in range(4)]
                            rd += offs
                            st[offs] = S @ st[offs]
                    if check:
                        assert len(set(rd)) == 512
        if rb_nq:   # backward transform before the stores
            for t in range(rb_nq):
                for o1, o2 in RT[t]:
                    u1, u2 = st[o1], st[o2]
                    st[o1], st[o2] = (u1 + 1j * u2) / 2, (u1 - 1j * u2) / 2
        for j in range(64):
            tr, src, pidx = trs[j]
            for t in range(16):
                tt = pswap_bits(t, 4) if tr else t
                v = st[slot(pidx * 16 + tt)]
                a[src + t] = np.conj(v) if tr else v
    return a
