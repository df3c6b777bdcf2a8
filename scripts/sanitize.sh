#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over every forced kernel variant at small n
# (the shared-memory tiles, named barriers of self-transposed blocks and packed placement).
# Usage (GPU box): bash scripts/sanitize.sh > gpurun_out/sanitize.txt 2>&1
cd "$(dirname "$0")/.."
SNIP='
import numpy as np, sys
sys.path.insert(0, ".")
import workloads as W
from paper_2404_13184_b200 import Simulator
for n in (6, 7):  # n = 6, 7: L = 12, 14 -> the block kernel runs too (TANQ_BLOCK=1)
    c = W.random_circuit(n, 40, seed=300 + n, kmax=3)
    nm = W.synthetic_calibration(c, n, depol=True, thermal=True, overrot=True)
    for kmax in (3, 4):
        with Simulator(n) as sim:
            sim.run_circuit(c, nm, fuse=2, k_max=kmax)
            p = sim.probs()
            s = sim.get_state()
print("ran", flush=True)
'
TOOLS=${TOOLS:-racecheck synccheck memcheck}
for tool in $TOOLS; do
  for v in "block auto 1" "block auto 0" "blocktma auto 1" "blocktma auto 0" "warp direct 1" "q1 tile 1" "o1 auto 1" "auto auto 1" "auto auto 0" "warp tile 0"; do
    set -- $v
    echo "=== $tool TANQ_GROUP=$1 TANQ_K2PATH=$2 TANQ_MIRROR=$3 TANQ_GRID_CAP=2"
    BLK=0; TMA=auto; [ "$1" = block ] && BLK=1 && TMA=0; [ "$1" = blocktma ] && BLK=1 && TMA=1
    TANQ_BLOCK=$BLK TANQ_BLOCK_TMA=$TMA TANQ_GROUP=$1 TANQ_K2PATH=$2 TANQ_MIRROR=$3 TANQ_GRID_CAP=2 timeout 900 \
      /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
      python -c "$SNIP" > /tmp/san.$$ 2>&1
    grep -E 'Race reported|access at|Error|Invalid|SUMMARY|^ran' /tmp/san.$$ | sed -E 's/\+0x[0-9a-f]+//' | sort | uniq -c | head -20
  done
done
