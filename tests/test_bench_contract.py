"""bench.py contract checks that need no GPU (-m "not gpu").

* `--impl reference` (the oracle arm) prints one JSON line with the keys the driver reads.
* Our arm fails loudly without a GPU: there is no CPU fallback on the product path.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, timeout=600):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout)


def test_reference_arm_json_line():
    r = _bench("--impl", "reference", "--config", "3", "--n", "7", "--steps", "3", "--warmup", "3",
               "--ref-budget", "0.5")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["steps"] == 3 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["n_qubits"] == 7 and "workload" in d["config"]
    assert d["config"]["gate_updates"] > 0 and "fusion" in d["config"]


def test_reference_arm_never_loads_the_product_library():
    """The reference arm (the CPU oracle) must not load libtanq.so: it reads the fused-update
    count from workloads/plan_counts.json."""
    snippet = (
        "import sys, runpy\n"
        f"sys.path.insert(0, {ROOT!r})\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--config', '3', '--n', '7', '--steps', "
        "'3', '--warmup', '3', '--ref-budget', '0.3']\n"
        "try:\n    runpy.run_path(%r, run_name='__main__')\nexcept SystemExit:\n    pass\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('LIBTANQ' if 'libtanq' in maps else 'CLEAN', 'ORACLE' if 'liboracle' in maps else '')\n"
    ) % os.path.join(ROOT, "bench.py")
    r = subprocess.run([sys.executable, "-c", snippet], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    last = r.stdout.strip().splitlines()[-1]
    assert last.startswith("CLEAN ORACLE"), r.stdout[-2000:]


def test_plan_counts_table_matches_planner():
    """workloads/plan_counts.json (read by the reference arm) equals the live host planner."""
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    import plan_counts
    table = json.load(open(os.path.join(ROOT, "workloads", "plan_counts.json")))
    assert plan_counts.compute() == table


def test_warmup_floor():
    r = _bench("--impl", "reference", "--config", "1", "--warmup", "2")
    assert r.returncode != 0 and "warmup" in r.stderr


def test_our_arm_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = _bench("--config", "1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", timeout=300)
    assert r.returncode != 0
    assert not any(ln.startswith("{") for ln in r.stdout.splitlines())
