set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
cat > /tmp/smk.py <<'PY'
import numpy as np, sys
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
for C in ws bulk; do TANQ_BLOCK_COPY=$C timeout 300 python /tmp/smk.py > gpurun_out/g6_smoke_$C.log 2>&1; echo $C; cat gpurun_out/g6_smoke_$C.log | tail -8; done
for C in ws bulk; do
  TANQ_BLOCK_COPY=$C timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g6_kbench_$C.jsonl 2>&1
  for D in 1 2; do TANQ_BLOCK_COPY=$C TANQ_DBG=$D timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g6_kbench_${C}_dbg$D.jsonl 2>&1; done
done
for f in gpurun_out/g6_kbench_*.jsonl; do echo $f; python -c "
import json
print([round(json.loads(l)['ms'],1) for l in open('$f') if l.startswith('{')])" 2>&1 | tail -2; done
for C in ws bulk; do TANQ_BLOCK_COPY=$C timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g6_bench_$C.json 2> gpurun_out/g6_bench_$C.err; python -c "import json; d=json.load(open('gpurun_out/g6_bench_$C.json')); print('$C', d['value'], d['ms_per_step'], {k:round(v['avg_ms'],2) for k,v in d['kernels'].items()})" 2>&1 | tail -1; done
