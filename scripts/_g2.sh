set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python - <<'PY' > gpurun_out/g2_smoke.log 2>&1
import numpy as np, sys, time
sys.path.insert(0, ".")
import workloads as W
from oracle import dense
from paper_2404_13184_b200 import Simulator
for n in (6, 7, 8):
    c, nm = W.config_workload(4, n=n)
    ref = dense.run(c, nm)
    for mirror in (True, False):
        with Simulator(n) as sim:
            st = sim.run_circuit(c, nm, mirror=mirror)
            got = sim.get_state().reshape(2**n, 2**n).T
        print(n, mirror, st["n_k3"], np.abs(got - ref).max(), flush=True)
PY
cat gpurun_out/g2_smoke.log
timeout 1200 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q > gpurun_out/g2_tests.log 2>&1; tail -15 gpurun_out/g2_tests.log
for B in 0 1; do TANQ_BLOCK=$B timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g2_kbench_block$B.jsonl 2>&1; done
for D in 1 2; do TANQ_BLOCK=1 TANQ_DBG=$D timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g2_kbench_block1_dbg$D.jsonl 2>&1; done
tail -8 gpurun_out/g2_kbench_*.jsonl
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g2_bench_c4.json 2> gpurun_out/g2_bench_c4.err; tail -c 1500 gpurun_out/g2_bench_c4.json; tail -5 gpurun_out/g2_bench_c4.err
