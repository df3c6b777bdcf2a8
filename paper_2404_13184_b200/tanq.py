"""Thin ctypes binding of libtanq.so (include/tanq.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module never
computes a state, a probability or a superoperator.  If libtanq.so is missing the import
fails loudly -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from typing import Iterable, List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtanq.so")

KIND = {"id": 0, "x": 1, "y": 2, "z": 3, "h": 4, "s": 5, "sdg": 6, "t": 7, "tdg": 8, "sx": 9,
        "rx": 10, "ry": 11, "rz": 12, "cx": 13, "cz": 14, "cp": 15, "swap": 16,
        "u": 17, "kraus": 18, "superop": 19, "reset": 20}
STATUS = {0: "OK", 1: "E_ARG", 2: "E_NOMEM", 3: "E_CUDA", 4: "E_NCCL", 5: "E_STATE",
          6: "E_UNSUPPORTED"}


class c64(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


class tanq_op(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("k", ctypes.c_int32), ("q", ctypes.c_int32 * 3),
                ("n_kraus", ctypes.c_int32), ("theta", ctypes.c_double),
                ("m", ctypes.c_void_p)]


class tanq_circuit(ctypes.Structure):
    _fields_ = [("n_ops", ctypes.c_uint64), ("ops", ctypes.POINTER(tanq_op))]


class tanq_qubit_cal(ctypes.Structure):
    _fields_ = [("t1_us", ctypes.c_double), ("t2_us", ctypes.c_double),
                ("p_meas1_prep0", ctypes.c_double), ("p_meas0_prep1", ctypes.c_double)]


class tanq_gate_cal(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("k", ctypes.c_int32), ("q", ctypes.c_int32 * 2),
                ("depol_p", ctypes.c_double), ("duration_ns", ctypes.c_double),
                ("overrot_rad", ctypes.c_double)]


class tanq_noise_model(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("order", ctypes.c_int32),
                ("qubits", ctypes.POINTER(tanq_qubit_cal)), ("n_gates", ctypes.c_uint64),
                ("gates", ctypes.POINTER(tanq_gate_cal))]


class tanq_readout(ctypes.Structure):
    _fields_ = [("p10", ctypes.c_void_p), ("p01", ctypes.c_void_p)]


class tanq_run_opts(ctypes.Structure):
    _fields_ = [("fuse", ctypes.c_int32), ("k_max", ctypes.c_int32),
                ("chunk_bytes", ctypes.c_uint64), ("flags", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class tanq_run_stats(ctypes.Structure):
    _fields_ = [("ops_in", ctypes.c_uint64), ("ops_fused", ctypes.c_uint64),
                ("gate_updates", ctypes.c_uint64), ("n_k", ctypes.c_uint64 * 6), ("n_remaps", ctypes.c_uint64),
                ("remap_bytes", ctypes.c_uint64), ("plan_ms", ctypes.c_double)]

    def as_dict(self):
        return {"ops_in": self.ops_in, "ops_fused": self.ops_fused,
                "gate_updates": self.gate_updates,
                "n_k1": self.n_k[1], "n_k2": self.n_k[2], "n_k3": self.n_k[3],
                "n_k4": self.n_k[4], "n_k5": self.n_k[5],
                "n_remaps": self.n_remaps, "remap_bytes": self.remap_bytes,
                "plan_ms": self.plan_ms}


class tanq_block_sub(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("a_off", ctypes.c_int32), ("t_off", ctypes.c_int32),
                ("tmask", ctypes.c_int32), ("nnz", ctypes.c_int32), ("hadd", ctypes.c_int32),
                ("sync", ctypes.c_int32)]


class tanq_block_params(ctypes.Structure):
    """Mirror of tanq::BlockParams (csrc/tanq_internal.h) for tanq_plan_block_program."""
    _fields_ = [("blob", ctypes.c_void_p), ("blob_bytes", ctypes.c_int32),
                ("n_sub", ctypes.c_int32), ("pairs", ctypes.c_int32), ("mirror", ctypes.c_uint32),
                ("tp_lo", ctypes.c_uint64), ("tp_m", ctypes.c_uint64),
                ("dbg", ctypes.c_uint32), ("half_add", ctypes.c_int32),
                ("n_blocks", ctypes.c_uint64), ("lo_mask", ctypes.c_uint64 * 10),
                ("piece_goff", ctypes.c_uint64 * 64), ("piece_start", ctypes.c_uint16 * 64),
                ("start_by_pidx", ctypes.c_uint16 * 64), ("sub", tanq_block_sub * 12),
                ("tma", ctypes.c_uint32), ("tdims", ctypes.c_int32), ("tlo", ctypes.c_int32 * 5),
                ("tbits", ctypes.c_int32 * 5), ("tbox", ctypes.c_int32 * 5),
                ("hi_blk", ctypes.c_int32), ("slot_off", ctypes.c_int32),
                ("rb_nq", ctypes.c_int32), ("rb_off", ctypes.c_int32)]


class tanq_info(ctypes.Structure):
    _fields_ = [("n_qubits", ctypes.c_int32), ("n_shards", ctypes.c_int32),
                ("world_size", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("local_bits", ctypes.c_int32), ("rowpos", ctypes.c_int32 * 32),
                ("colpos", ctypes.c_int32 * 32), ("shard_bytes", ctypes.c_uint64),
                ("parity_qubits", ctypes.c_uint64)]


class tanq_kernel_prof(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_uint64),
                ("total_ms", ctypes.c_double), ("bytes", ctypes.c_double),
                ("flops", ctypes.c_double), ("hw_flops", ctypes.c_double)]


# exported symbols and their signatures (mirrors include/tanq.h)
_P, _I, _U64, _D = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_double
SIGNATURES = {
    "tanq_create": ([_I, _I, ctypes.POINTER(_P)], _I),
    "tanq_create_dist": ([_I, _I, _I, _I, _P, ctypes.POINTER(_P)], _I),
    "tanq_create_ex": ([_I, _I, ctypes.POINTER(_P), ctypes.POINTER(_I), ctypes.c_size_t,
                        ctypes.POINTER(_P)], _I),
    "tanq_nccl_unique_id": ([_P, ctypes.c_size_t], _I),
    "tanq_destroy": ([_P], _I),
    "tanq_reset": ([_P], _I),
    "tanq_info_get": ([_P, ctypes.POINTER(tanq_info)], _I),
    "tanq_set_stream": ([_P, _I, _P], _I),
    "tanq_apply_gate": ([_P, _I, _P, _P], _I),
    "tanq_apply_channel": ([_P, _I, _P, _I, _P, _I], _I),
    "tanq_apply_superop": ([_P, _I, _P, _P], _I),
    "tanq_run_circuit": ([_P, ctypes.POINTER(tanq_circuit), ctypes.POINTER(tanq_noise_model),
                          ctypes.POINTER(tanq_run_opts), ctypes.POINTER(tanq_run_stats)], _I),
    "tanq_plan_create": ([_P, ctypes.POINTER(tanq_circuit), ctypes.POINTER(tanq_noise_model),
                          ctypes.POINTER(tanq_run_opts), ctypes.POINTER(_P)], _I),
    "tanq_plan_exec": ([_P, _P, ctypes.POINTER(tanq_run_stats)], _I),
    "tanq_plan_destroy": ([_P], _I),
    "tanq_plan_create_host": ([_I, _I, ctypes.POINTER(tanq_circuit),
                               ctypes.POINTER(tanq_noise_model), ctypes.POINTER(tanq_run_opts),
                               ctypes.POINTER(_P)], _I),
    "tanq_plan_info": ([_P, ctypes.POINTER(tanq_run_stats)], _I),
    "tanq_plan_get_op": ([_P, _U64, _P, _P, _P], _I),
    "tanq_plan_schedule": ([_P, _I, _P, _U64, ctypes.POINTER(_U64)], _I),
    "tanq_plan_block_program": ([_P, _U64, _I, _P, ctypes.c_size_t, _P, ctypes.c_size_t,
                                 ctypes.POINTER(_I), ctypes.POINTER(ctypes.c_size_t)], _I),
    "tanq_probs": ([_P, ctypes.POINTER(tanq_readout), _P], _I),
    "tanq_expect_pauli": ([_P, _U64, _U64, _P, _P], _I),
    "tanq_sample": ([_P, ctypes.POINTER(tanq_readout), _U64, _U64, _P], _I),
    "tanq_measure": ([_P, _I, _U64, ctypes.POINTER(_I), ctypes.POINTER(_D)], _I),
    "tanq_qasm_parse": ([ctypes.c_char_p, _I, ctypes.POINTER(_P)], _I),
    "tanq_qasm_circuit": ([_P, ctypes.POINTER(tanq_circuit), ctypes.POINTER(_I), ctypes.POINTER(_I)], _I),
    "tanq_qasm_measures": ([_P, _P], _I),
    "tanq_qasm_free": ([_P], _I),
    "tanq_check_hermitian": ([_P, _D, ctypes.POINTER(_I)], _I),
    "tanq_device_parse": ([ctypes.c_char_p, ctypes.POINTER(_P)], _I),
    "tanq_device_noise": ([_P, ctypes.POINTER(tanq_noise_model), ctypes.POINTER(_I)], _I),
    "tanq_device_coupling": ([_P, _P, _U64, ctypes.POINTER(_U64)], _I),
    "tanq_device_name": ([_P], ctypes.c_char_p),
    "tanq_device_free": ([_P], _I),
    "tanq_get_state": ([_P, _U64, _U64, _P], _I),
    "tanq_set_state": ([_P, _U64, _U64, _P], _I),
    "tanq_sync": ([_P], _I),
    "tanq_last_error": ([], ctypes.c_char_p),
    "tanq_profile_read": ([_P, ctypes.POINTER(tanq_kernel_prof), _I, ctypes.POINTER(_I)], _I),
    "tanq_profile_reset": ([_P], _I),
    "tanq_launch_count": ([_P], _U64),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libtanq.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


class TanqError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib().tanq_last_error().decode()
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(st: int, where: str):
    if st != 0:
        raise TanqError(st, where)


def _c64_array(m) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(m, dtype=np.complex128))


# ----------------------------------------------------------------------------------
# marshalling of circuits / noise models (duck-typed: .n, .ops[kind, qubits, theta, mat,
# kraus]; NoiseModel with .qubits[t1_us, t2_us, p10, p01], .gates{(kind, qubits): cal})
# ----------------------------------------------------------------------------------
class CCircuit:
    def __init__(self, ops: Sequence):
        self.keep: List[np.ndarray] = []
        arr = (tanq_op * max(1, len(ops)))()
        for i, op in enumerate(ops):
            o = arr[i]
            o.kind = KIND[op.kind]
            o.k = len(op.qubits)
            for j, q in enumerate(op.qubits):
                o.q[j] = int(q)
            o.theta = float(getattr(op, "theta", 0.0) or 0.0)
            o.n_kraus = 0
            o.m = None
            if op.kind in ("u", "superop"):
                m = _c64_array(op.mat)
                self.keep.append(m)
                o.m = m.ctypes.data
            elif op.kind == "kraus":
                m = _c64_array(np.stack([np.asarray(K) for K in op.kraus]))
                self.keep.append(m)
                o.m = m.ctypes.data
                o.n_kraus = len(op.kraus)
        self.arr = arr
        self.c = tanq_circuit(len(ops), ctypes.cast(arr, ctypes.POINTER(tanq_op)))


class CNoise:
    def __init__(self, nm):
        qa = (tanq_qubit_cal * nm.n)()
        for q, qc in enumerate(nm.qubits):
            qa[q].t1_us, qa[q].t2_us = qc.t1_us, qc.t2_us
            qa[q].p_meas1_prep0, qa[q].p_meas0_prep1 = qc.p10, qc.p01
        items = list(nm.gates.items())
        ga = (tanq_gate_cal * max(1, len(items)))()
        for i, ((kind, qs), g) in enumerate(items):
            ga[i].kind = KIND[kind]
            ga[i].k = len(qs)
            ga[i].q[0] = qs[0]
            ga[i].q[1] = qs[1] if len(qs) > 1 else -1
            ga[i].depol_p, ga[i].duration_ns, ga[i].overrot_rad = g.depol_p, g.duration_ns, g.overrot_rad
        self.qa, self.ga = qa, ga
        self.c = tanq_noise_model(nm.n, int(getattr(nm, "order", 0)),
                                  ctypes.cast(qa, ctypes.POINTER(tanq_qubit_cal)), len(items),
                                  ctypes.cast(ga, ctypes.POINTER(tanq_gate_cal)))


class CReadout:
    def __init__(self, p10, p01):
        self.p10 = np.ascontiguousarray(p10, dtype=np.float64)
        self.p01 = np.ascontiguousarray(p01, dtype=np.float64)
        self.c = tanq_readout(self.p10.ctypes.data, self.p01.ctypes.data)

    @staticmethod
    def of(nm) -> Optional["CReadout"]:
        if nm is None:
            return None
        return CReadout([q.p10 for q in nm.qubits], [q.p01 for q in nm.qubits])


class Plan:
    """tanq_plan_create / tanq_plan_exec: host steps A-1..A-4 done once, executed many times.

    sim=None plans on the host only (tanq_plan_create_host) for an n-qubit register split
    over world_size shards."""

    def __init__(self, sim, circuit, noise=None, *, fuse=2, k_max=3, profile=False,
                 world_size: int = 1, graph: bool = False, mirror: bool = True):
        cc = CCircuit(circuit.ops)
        cn = _noise_of(noise)
        opts = tanq_run_opts(fuse, k_max, 0,
                             (1 if profile else 0) | (2 if graph else 0) | (0 if mirror else 4), 0)
        h = ctypes.c_void_p()
        nmp = ctypes.byref(cn.c) if cn is not None else None
        if sim is None:
            _check(lib().tanq_plan_create_host(circuit.n, world_size, ctypes.byref(cc.c), nmp,
                                               ctypes.byref(opts), ctypes.byref(h)),
                   "tanq_plan_create_host")
        else:
            _check(lib().tanq_plan_create(sim.h, ctypes.byref(cc.c), nmp, ctypes.byref(opts),
                                          ctypes.byref(h)), "tanq_plan_create")
        self.h = h
        nb = 0
        if isinstance(cn, CNoise):
            nb = ctypes.sizeof(cn.qa) + ctypes.sizeof(cn.ga)
        elif cn is not None:
            nb = cn.c.n * ctypes.sizeof(tanq_qubit_cal) + cn.c.n_gates * ctypes.sizeof(tanq_gate_cal)
        self.h2d_bytes = ctypes.sizeof(cc.arr) + sum(a.nbytes for a in cc.keep) + nb

    def exec(self, sim: "Simulator") -> dict:
        st = tanq_run_stats()
        _check(lib().tanq_plan_exec(sim.h, self.h, ctypes.byref(st)), "tanq_plan_exec")
        return st.as_dict()

    def info(self) -> dict:
        st = tanq_run_stats()
        _check(lib().tanq_plan_info(self.h, ctypes.byref(st)), "tanq_plan_info")
        return st.as_dict()

    def schedule(self, world_size: int):
        """[(0, op_index, 0) | (1, a_global_bit, b_local_bit)] as executed on world_size shards."""
        n = ctypes.c_uint64()
        _check(lib().tanq_plan_schedule(self.h, world_size, None, 0, ctypes.byref(n)),
               "tanq_plan_schedule")
        items = np.zeros(3 * max(1, n.value), dtype=np.int32)
        _check(lib().tanq_plan_schedule(self.h, world_size, items.ctypes.data, n.value,
                                        ctypes.byref(n)), "tanq_plan_schedule")
        return [tuple(int(v) for v in items[3 * i:3 * i + 3]) for i in range(n.value)]

    def op(self, i: int):
        """(qubits tuple, S ndarray 4^k x 4^k) of fused op i (a group: its sub-ops' product)."""
        k = ctypes.c_int()
        q = (ctypes.c_int * 8)()
        _check(lib().tanq_plan_get_op(self.h, i, ctypes.byref(k), q, None), "tanq_plan_get_op")
        S = np.empty((4 ** k.value, 4 ** k.value), dtype=np.complex128)
        _check(lib().tanq_plan_get_op(self.h, i, ctypes.byref(k), q, S.ctypes.data),
               "tanq_plan_get_op")
        return tuple(q[:k.value]), S

    def ops(self):
        """[(qubits tuple, S ndarray 4^k x 4^k)] of the fused plan."""
        return [self.op(i) for i in range(self.info()["ops_fused"])]

    def block_program(self, i: int, packed: bool = True):
        """(params, blob bytes) of the block-pipeline kernel for op i, or None."""
        prm = tanq_block_params()
        kind, nbytes = ctypes.c_int(), ctypes.c_size_t()
        _check(lib().tanq_plan_block_program(self.h, i, int(packed), ctypes.byref(prm),
                                             ctypes.sizeof(prm), None, 0, ctypes.byref(kind),
                                             ctypes.byref(nbytes)), "tanq_plan_block_program")
        if kind.value != 2:
            return None
        blob = np.zeros(nbytes.value, dtype=np.uint8)
        _check(lib().tanq_plan_block_program(self.h, i, int(packed), ctypes.byref(prm),
                                             ctypes.sizeof(prm), blob.ctypes.data, blob.size,
                                             ctypes.byref(kind), ctypes.byref(nbytes)),
               "tanq_plan_block_program")
        return prm, blob

    def close(self):
        if self.h:
            lib().tanq_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class QasmOp:
    __slots__ = ("kind", "qubits", "theta", "mat", "kraus")

    def __init__(self, kind, qubits, theta):
        self.kind, self.qubits, self.theta, self.mat, self.kraus = kind, qubits, theta, None, None

    def __repr__(self):
        return f"QasmOp({self.kind}, {self.qubits}, {self.theta:.6g})"


class QasmCircuit:
    """tanq_qasm_parse: OpenQASM 2.0 subset -> circuit (optionally lowered to the IBM basis).
    `.ops` mirrors the library's op list (kind names, qubits, angles) for inspection; runs use
    the library-owned C array directly."""

    def __init__(self, text: str, to_basis: bool = True):
        h = ctypes.c_void_p()
        _check(lib().tanq_qasm_parse(text.encode(), int(to_basis), ctypes.byref(h)), "tanq_qasm_parse")
        self.h = h
        c = tanq_circuit()
        nq, nc = ctypes.c_int(), ctypes.c_int()
        _check(lib().tanq_qasm_circuit(h, ctypes.byref(c), ctypes.byref(nq), ctypes.byref(nc)),
               "tanq_qasm_circuit")
        self.c, self.n, self.n_clbits = c, nq.value, nc.value
        names = {v: k for k, v in KIND.items()}
        self.ops = [QasmOp(names[c.ops[i].kind], tuple(c.ops[i].q[:c.ops[i].k]), c.ops[i].theta)
                    for i in range(c.n_ops)]
        meas = (ctypes.c_int32 * max(1, self.n_clbits))()
        _check(lib().tanq_qasm_measures(h, meas), "tanq_qasm_measures")
        self.measures = list(meas[:self.n_clbits])

    def close(self):
        if self.h:
            lib().tanq_qasm_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Device:
    """tanq_device_parse: a device-calibration JSON (T1, T2, readout, gate error and length;
    SPEC S:365-370 schema) -> the library's noise model.  Pass it wherever a noise model is
    accepted; `.readout()` gives the per-qubit readout confusion for probs / sample."""

    def __init__(self, text: str):
        h = ctypes.c_void_p()
        _check(lib().tanq_device_parse(text.encode(), ctypes.byref(h)), "tanq_device_parse")
        self.h = h
        self.c = tanq_noise_model()
        n = ctypes.c_int()
        _check(lib().tanq_device_noise(h, ctypes.byref(self.c), ctypes.byref(n)),
               "tanq_device_noise")
        self.n = n.value
        self.name = lib().tanq_device_name(h).decode()
        cnt = ctypes.c_uint64()
        _check(lib().tanq_device_coupling(h, None, 0, ctypes.byref(cnt)), "tanq_device_coupling")
        pairs = np.zeros(2 * max(1, cnt.value), dtype=np.int32)
        _check(lib().tanq_device_coupling(h, pairs.ctypes.data, cnt.value, ctypes.byref(cnt)),
               "tanq_device_coupling")
        self.coupling = [tuple(int(x) for x in pairs[2 * i:2 * i + 2]) for i in range(cnt.value)]

    def gates(self):
        """[(kind name, qubits, depol_p, duration_ns, overrot_rad)] as bound by the library."""
        names = {v: k for k, v in KIND.items()}
        out = []
        for i in range(self.c.n_gates):
            g = self.c.gates[i]
            out.append((names[g.kind], tuple(g.q[:g.k]), g.depol_p, g.duration_ns, g.overrot_rad))
        return out

    def readout(self) -> "CReadout":
        return CReadout([self.c.qubits[q].p_meas1_prep0 for q in range(self.n)],
                        [self.c.qubits[q].p_meas0_prep1 for q in range(self.n)])

    def close(self):
        if self.h:
            lib().tanq_device_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _noise_of(noise):
    if noise is None:
        return None
    return noise if isinstance(noise, Device) else CNoise(noise)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().tanq_nccl_unique_id(buf, 128), "tanq_nccl_unique_id")
    return buf.raw


class Simulator:
    """One handle of libtanq (tanq_create / tanq_create_dist)."""

    def __init__(self, n_qubits: int, n_shards: int = 1, *, world_size: int = 0, rank: int = 0,
                 device: int = 0, nccl_uid: Optional[bytes] = None, buffers=None):
        self.n = n_qubits
        h = ctypes.c_void_p()
        if buffers is not None:
            # caller-owned device buffers (tanq_create_ex), e.g. torch tensors: anything with
            # data_ptr(), nbytes and a .device.index; kept referenced for the handle's lifetime
            self._buffers = list(buffers)
            ptrs = (ctypes.c_void_p * len(self._buffers))(*[b.data_ptr() for b in self._buffers])
            devs = (ctypes.c_int * len(self._buffers))(*[int(b.device.index or 0)
                                                         for b in self._buffers])
            nbytes = min(int(b.nbytes) for b in self._buffers)
            _check(lib().tanq_create_ex(n_qubits, len(self._buffers), ptrs, devs, nbytes,
                                        ctypes.byref(h)), "tanq_create_ex")
        elif world_size:
            uid = ctypes.create_string_buffer(nccl_uid, 128) if nccl_uid else None
            _check(lib().tanq_create_dist(n_qubits, world_size, rank, device, uid,
                                          ctypes.byref(h)), "tanq_create_dist")
        else:
            _check(lib().tanq_create(n_qubits, n_shards, ctypes.byref(h)), "tanq_create")
        self.h = h

    def close(self):
        if self.h:
            lib().tanq_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- state ----------------------------------------------------------------------
    def reset(self):
        _check(lib().tanq_reset(self.h), "tanq_reset")

    def info(self) -> dict:
        i = tanq_info()
        _check(lib().tanq_info_get(self.h, ctypes.byref(i)), "tanq_info_get")
        return {"n_qubits": i.n_qubits, "n_shards": i.n_shards, "world_size": i.world_size,
                "rank": i.rank, "local_bits": i.local_bits,
                "rowpos": list(i.rowpos[:i.n_qubits]), "colpos": list(i.colpos[:i.n_qubits]),
                "shard_bytes": i.shard_bytes, "parity_qubits": i.parity_qubits}

    def set_stream(self, stream_ptr: int, shard: int = 0):
        _check(lib().tanq_set_stream(self.h, shard, ctypes.c_void_p(stream_ptr)), "tanq_set_stream")

    def get_state(self, first: int = 0, count: Optional[int] = None, out: Optional[np.ndarray] = None):
        total = 4 ** self.n
        if count is None:
            count = total - first
        if out is None:
            out = np.empty(count, dtype=np.complex128)
        _check(lib().tanq_get_state(self.h, first, count, out.ctypes.data), "tanq_get_state")
        return out

    def set_state(self, vec: np.ndarray, first: int = 0):
        v = _c64_array(vec).reshape(-1)
        _check(lib().tanq_set_state(self.h, first, v.size, v.ctypes.data), "tanq_set_state")

    def check_hermitian(self, tol: float = 1e-13) -> bool:
        r = ctypes.c_int()
        _check(lib().tanq_check_hermitian(self.h, tol, ctypes.byref(r)), "tanq_check_hermitian")
        return bool(r.value)

    def sync(self):
        _check(lib().tanq_sync(self.h), "tanq_sync")

    # -- operations -----------------------------------------------------------------
    def apply_gate(self, qubits: Sequence[int], U):
        q = np.ascontiguousarray(qubits, dtype=np.int32)
        m = _c64_array(U)
        _check(lib().tanq_apply_gate(self.h, len(q), q.ctypes.data, m.ctypes.data), "tanq_apply_gate")

    def apply_channel(self, qubits: Sequence[int], kraus, check_cptp: bool = False):
        q = np.ascontiguousarray(qubits, dtype=np.int32)
        m = _c64_array(np.stack([np.asarray(K) for K in kraus]))
        _check(lib().tanq_apply_channel(self.h, len(q), q.ctypes.data, len(kraus), m.ctypes.data,
                                        int(check_cptp)), "tanq_apply_channel")

    def apply_superop(self, qubits: Sequence[int], S):
        q = np.ascontiguousarray(qubits, dtype=np.int32)
        m = _c64_array(S)
        _check(lib().tanq_apply_superop(self.h, len(q), q.ctypes.data, m.ctypes.data),
               "tanq_apply_superop")

    def run_circuit(self, circuit, noise=None, *, fuse: int = 2, k_max: int = 3,
                    profile: bool = False, prepared=None, mirror: bool = True) -> dict:
        if isinstance(circuit, QasmCircuit):
            class _C:  # the library-owned op array
                c = circuit.c
            cc = _C()
        else:
            cc = prepared[0] if prepared else CCircuit(circuit.ops)
        cn = prepared[1] if prepared else _noise_of(noise)
        opts = tanq_run_opts(fuse, k_max, 0, (1 if profile else 0) | (0 if mirror else 4), 0)
        st = tanq_run_stats()
        _check(lib().tanq_run_circuit(self.h, ctypes.byref(cc.c),
                                      ctypes.byref(cn.c) if cn is not None else None,
                                      ctypes.byref(opts), ctypes.byref(st)), "tanq_run_circuit")
        return st.as_dict()

    def plan(self, circuit, noise=None, *, fuse: int = 2, k_max: int = 3,
             profile: bool = False, graph: bool = False, mirror: bool = True) -> "Plan":
        return Plan(self, circuit, noise, fuse=fuse, k_max=k_max, profile=profile, graph=graph,
                    mirror=mirror)

    @staticmethod
    def prepare(circuit, noise=None):
        return (CCircuit(circuit.ops), _noise_of(noise))

    # -- reductions -----------------------------------------------------------------
    def probs(self, readout=None) -> np.ndarray:
        out = np.empty(2 ** self.n)
        ro = readout if (readout is None or isinstance(readout, CReadout)) else CReadout(*readout)
        _check(lib().tanq_probs(self.h, ctypes.byref(ro.c) if ro else None, out.ctypes.data),
               "tanq_probs")
        return out

    def expect_pauli(self, x_mask: int, z_mask: int) -> complex:
        re, im = ctypes.c_double(), ctypes.c_double()
        _check(lib().tanq_expect_pauli(self.h, x_mask, z_mask, ctypes.byref(re), ctypes.byref(im)),
               "tanq_expect_pauli")
        return complex(re.value, im.value)

    def sample(self, shots: int, seed: int, readout=None) -> np.ndarray:
        out = np.empty(shots, dtype=np.uint64)
        ro = readout if (readout is None or isinstance(readout, CReadout)) else CReadout(*readout)
        _check(lib().tanq_sample(self.h, ctypes.byref(ro.c) if ro else None, seed, shots,
                                 out.ctypes.data), "tanq_sample")
        return out

    def measure(self, qubit: int, seed: int):
        """Mid-circuit projective measurement: returns (outcome, probability of that outcome)."""
        b, p = ctypes.c_int(), ctypes.c_double()
        _check(lib().tanq_measure(self.h, qubit, seed, ctypes.byref(b), ctypes.byref(p)),
               "tanq_measure")
        return b.value, p.value

    # -- instrumentation --------------------------------------------------------------
    def profile(self) -> List[dict]:
        arr = (tanq_kernel_prof * 8)()
        n = ctypes.c_int()
        _check(lib().tanq_profile_read(self.h, arr, 8, ctypes.byref(n)), "tanq_profile_read")
        return [{"name": arr[i].name.decode(), "launches": arr[i].launches,
                 "total_ms": arr[i].total_ms, "bytes": arr[i].bytes, "flops": arr[i].flops,
                 "hw_flops": arr[i].hw_flops}
                for i in range(n.value)]

    def profile_reset(self):
        _check(lib().tanq_profile_reset(self.h), "tanq_profile_reset")

    def launch_count(self) -> int:
        return int(lib().tanq_launch_count(self.h))
