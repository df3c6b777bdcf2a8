"""Device-calibration front end (NEXT-4; Sec. 3.5; schema SPEC S:365-370).

CPU: the C++ parser (tanq_device_parse) binds the same noise model the oracle derives
independently from the JSON (channels.noise_model_from_device), and rejects malformed
snapshots naming the JSON path.  GPU: a QASM circuit on the synthetic 16-qubit heavy-hex
device, lowered to the IBM basis, run under the parsed noise, equals the oracle.
"""
import json
import os

import numpy as np
import pytest

import workloads as W
from oracle import channels, dense

GOLD = os.path.join(os.path.dirname(__file__), "golden", "device_guadalupe_like.json")


def _dev():
    return json.load(open(GOLD))


def test_device_binding_matches_oracle_reading():
    from paper_2404_13184_b200 import Device
    raw = _dev()
    d = Device(json.dumps(raw))
    ref = channels.noise_model_from_device(raw)
    assert d.n == 16 and d.name == raw["name"]
    assert d.coupling == [tuple(p) for p in raw["coupling_map"]]
    got = {(k, q): (p, t, e) for k, q, p, t, e in d.gates()}
    assert set(got) == set(ref.gates)                       # RZ entries dropped (noiseless)
    for key, g in ref.gates.items():
        assert got[key] == pytest.approx((g.depol_p, g.duration_ns, g.overrot_rad), abs=0, rel=1e-15)
    ro = d.readout()
    np.testing.assert_array_equal(ro.p10, [q.p10 for q in ref.qubits])
    np.testing.assert_array_equal(ro.p01, [q.p01 for q in ref.qubits])


def test_device_error_conversion_closed_form():
    """Reading R6: e = 0.0075 on a 1q gate -> p = 0.015; on a cx -> p = 0.01; e = 0.9 on cx
    -> p = 1.2 clamped to 1."""
    from paper_2404_13184_b200 import Device
    dev = {"name": "t", "num_qubits": 2,
           "qubits": [{"t1_us": 100, "t2_us": 80, "prob_meas0_prep1": 0.02,
                       "prob_meas1_prep0": 0.01}] * 2,
           "gates": [{"name": "sx", "qubits": [0], "error": 0.0075, "duration_ns": 35.5},
                     {"name": "cx", "qubits": [0, 1], "error": 0.0075, "duration_ns": 300},
                     {"name": "cx", "qubits": [1, 0], "error": 0.9, "duration_ns": 300,
                      "overrot_rad": 0.01}]}
    g = {(k, q): (p, e) for k, q, p, t, e in Device(json.dumps(dev)).gates()}
    assert g[("sx", (0,))][0] == pytest.approx(0.015, rel=1e-15)
    assert g[("cx", (0, 1))][0] == pytest.approx(0.01, rel=1e-15)
    assert g[("cx", (1, 0))] == (1.0, 0.01)


@pytest.mark.parametrize("mutate,where", [
    (lambda d: d.pop("qubits"), "$.qubits"),
    (lambda d: d["qubits"][3].update(t2_us=2.5 * d["qubits"][3]["t1_us"]), "$.qubits[3]"),
    (lambda d: d["qubits"][5].pop("prob_meas0_prep1"), "$.qubits[5].prob_meas0_prep1"),
    (lambda d: d["gates"][7].update(name="cz"), "$.gates[7].name"),
    (lambda d: d["gates"][70].update(qubits=[3]), "$.gates[70].qubits"),
    (lambda d: d["gates"][2].update(error=1.5), "$.gates[2].error"),
    (lambda d: d.update(num_qubits=15), "$.qubits"),
    (lambda d: d["coupling_map"].append([1, 99]), "$.coupling_map[16]"),
])
def test_device_schema_errors(mutate, where):
    from paper_2404_13184_b200 import Device, TanqError
    d = _dev()
    mutate(d)
    with pytest.raises(TanqError) as e:
        Device(json.dumps(d))
    assert e.value.status == 1 and where in str(e.value), str(e.value)


def test_device_malformed_json():
    from paper_2404_13184_b200 import Device, TanqError
    for bad in ('{"name": "x", ', '[1, 2]', '{"name": "x"} trailing', ''):
        with pytest.raises(TanqError):
            Device(bad)


@pytest.mark.gpu
def test_qasm_on_device_noise_vs_oracle():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from __graft_entry__ import build
    build()
    from paper_2404_13184_b200 import Device, QasmCircuit, Simulator
    raw = _dev()
    dev = Device(json.dumps(raw))
    # 7 qubits of the device along coupled pairs; QFT-like entangler lowered to {rz, sx, x, cx}
    src = """OPENQASM 2.0;
include "qelib1.inc";
qreg q[16];
creg c[7];
h q[0]; h q[1]; x q[4];
cx q[0],q[1]; cp(pi/4) q[1],q[2]; cx q[1],q[4];
u3(0.4,0.1,-0.3) q[2]; cx q[2],q[3]; cx q[4],q[7];
rz(0.3) q[7]; sx q[3]; cx q[3],q[5]; cx q[7],q[6]; h q[6];
"""
    qc = QasmCircuit(src, to_basis=True)
    # compact to the used qubits so the oracle stays small; calibrations follow the qubits
    used = sorted({q for o in qc.ops for q in o.qubits})
    full = W.Circuit(16, [W.Op(o.kind, tuple(o.qubits), o.theta) for o in qc.ops])
    nm16 = channels.noise_model_from_device(raw)
    sub, snm = W.restrict(full, nm16, used)
    ref = dense.run(sub, snm)
    # the library side: the same compact circuit with the device's calibration rows remapped
    dsub = dict(raw)
    loc = {q: j for j, q in enumerate(used)}
    dsub["num_qubits"] = len(used)
    dsub["qubits"] = [raw["qubits"][q] for q in used]
    dsub["gates"] = [dict(g, qubits=[loc[q] for q in g["qubits"]]) for g in raw["gates"]
                     if all(q in loc for q in g["qubits"])]
    dsub["coupling_map"] = [[loc[a], loc[b]] for a, b in raw["coupling_map"]
                            if a in loc and b in loc]
    dev_sub = Device(json.dumps(dsub))
    n = len(used)
    with Simulator(n) as sim:
        sim.run_circuit(sub, dev_sub)
        got = sim.get_state().reshape(2 ** n, 2 ** n).T
        p = sim.probs(dev_sub.readout())
    d = got - ref
    assert np.abs(d).max() <= 1e-10 and np.linalg.norm(d) / np.linalg.norm(ref) <= 1e-12
    ro = (np.array([q.p10 for q in snm.qubits]), np.array([q.p01 for q in snm.qubits]))
    np.testing.assert_allclose(p, dense.probs(ref, n, ro), atol=1e-10, rtol=0)
