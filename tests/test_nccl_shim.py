"""CPU self-test of the NCCL test shim used by tests/test_gpu_dist.py (-m "not gpu"): the shim
is test infrastructure standing in for NCCL when several ranks share one GPU, so it is checked
on its own -- all-reduce sum / max and grouped pairwise exchanges larger than one mailbox,
2, 4 and 8 forked ranks, host buffers (-DSHIM_HOST_TEST)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM = os.path.join(ROOT, "tests", "nccl_shim")


@pytest.fixture(scope="module")
def selftest(tmp_path_factory):
    if not shutil.which("g++") or not os.path.exists("/usr/local/cuda/include/cuda_runtime.h"):
        pytest.skip("g++ / CUDA headers not available")
    exe = str(tmp_path_factory.mktemp("shim") / "shim_selftest")
    r = subprocess.run(["g++", "-O2", "-std=c++17", "-DSHIM_HOST_TEST", "-I/usr/local/cuda/include",
                        os.path.join(SHIM, "shim_selftest.cpp"), os.path.join(SHIM, "nccl_shim.cpp"),
                        "-o", exe, "-lpthread"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_shim_collectives(selftest, ranks):
    r = subprocess.run([selftest, str(ranks)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr
