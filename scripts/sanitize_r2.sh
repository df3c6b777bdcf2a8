#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over the round-2 paths at small n:
# parity-layout shards (packed kernels with a shard transpose descriptor, parity remap kernels),
# k_max = 5 block groups (per-sub-op warp split + pair barriers), and the opt-in real-basis
# and sparse sub-op programs.  Usage (GPU box): bash scripts/sanitize_r2.sh > out.txt 2>&1
cd "$(dirname "$0")/.."
SNIP='
import numpy as np, sys, os
sys.path.insert(0, ".")
import workloads as W
from paper_2404_13184_b200 import Simulator
mode = os.environ["SAN_CASE"]
n = 7
if mode == "shards":
    c = W.random_circuit(n, 40, seed=311, kmax=3)
    nm = W.synthetic_calibration(c, n, depol=True, thermal=True, overrot=True)
    for shards in (2, 4):
        with Simulator(n, shards) as sim:
            st = sim.run_circuit(c, nm, fuse=2, k_max=3)
            p = sim.probs(); e = sim.expect_pauli(0b11 << (n - 2), 0); s = sim.get_state()
            assert st["n_remaps"] > 0
else:
    c, nm = W.config_workload(4, n=n)
    for kmax in ((5,) if mode == "kmax5" else (3, 5)):
        with Simulator(n) as sim:
            sim.run_circuit(c, nm, fuse=2, k_max=kmax)
            p = sim.probs(); s = sim.get_state()
print("ran", flush=True)
'
TOOLS=${TOOLS:-racecheck synccheck memcheck}
for tool in $TOOLS; do
  for v in "shards 1 0 0" "shards 0 0 0" "kmax5 1 0 0" "kmax5 0 0 0" "rbasis 1 1 0" "sparse 1 0 64"; do
    set -- $v
    echo "=== $tool case=$1 TANQ_MIRROR=$2 TANQ_RBASIS=$3 TANQ_SPARSE_MAX=$4 TANQ_GRID_CAP=2"
    SAN_CASE=$1 TANQ_MIRROR=$2 TANQ_RBASIS=$3 TANQ_SPARSE_MAX=$4 TANQ_GRID_CAP=2 timeout 900 \
      /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
      python -c "$SNIP" > /tmp/san.$$ 2>&1
    grep -E 'Race reported|access at|Error|Invalid|SUMMARY|^ran' /tmp/san.$$ | sed -E 's/\+0x[0-9a-f]+//' | sort | uniq -c | head -20
  done
done
