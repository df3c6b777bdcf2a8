"""C-ABI library checks that need no GPU (-m "not gpu")."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tanq.h")


def _built_lib():
    from paper_2404_13184_b200 import build
    return build.build()


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tanq_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared_functions()
    for required in ("tanq_create", "tanq_create_dist", "tanq_destroy", "tanq_apply_gate",
                     "tanq_apply_channel", "tanq_apply_superop", "tanq_run_circuit",
                     "tanq_probs", "tanq_expect_pauli", "tanq_sample", "tanq_get_state",
                     "tanq_sync", "tanq_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol():
    path = _built_lib()
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tanq_\w+)", out))
    missing = [f for f in _declared_functions() if f not in exported]
    assert not missing, missing
    L = ctypes.CDLL(path)
    for f in _declared_functions():
        getattr(L, f)


def test_binding_signatures_cover_header():
    from paper_2404_13184_b200 import tanq
    assert set(tanq.SIGNATURES) == set(_declared_functions())


def test_kernels_are_sm100a_and_use_dmma():
    path = _built_lib()
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", path], capture_output=True,
                                       text=True).stdout
    assert "DMMA.8x8x4" in sass           # K3 on the FP64 tensor pipe
    assert "DFMA" in sass                 # K1/K2 register FMA streams


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2404_13184_b200 import Simulator, TanqError
    with pytest.raises(TanqError) as e:
        Simulator(3)
    assert e.value.status == 6


def test_argument_errors_without_device():
    from paper_2404_13184_b200 import tanq
    L = tanq.lib()
    h = ctypes.c_void_p()
    assert L.tanq_create(0, 1, ctypes.byref(h)) == 1
    assert L.tanq_create(3, 3, ctypes.byref(h)) == 1
    assert L.tanq_create_dist(3, 2, 5, 0, None, ctypes.byref(h)) == 1
    assert b"rank" in L.tanq_last_error()
