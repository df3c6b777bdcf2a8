set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
TANQ_BLOCK_ACC=2 timeout 300 python scripts/_smk.py > gpurun_out/g13_smoke.log 2>&1; tail -3 gpurun_out/g13_smoke.log
for A in 0 2; do
  TANQ_BLOCK_ACC=$A timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g13_kbench_$A.jsonl 2>&1
  TANQ_BLOCK_ACC=$A TANQ_DBG=2 timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g13_kbench_${A}_dbg2.jsonl 2>&1
  TANQ_BLOCK_ACC=$A timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g13_bench_$A.json 2>&1
done
for f in gpurun_out/g13_kbench_*.jsonl; do echo $f; python -c "
import json
print([round(json.loads(l)['ms'],1) for l in open('$f') if l.startswith('{')])" 2>&1 | tail -1; done
for f in gpurun_out/g13_bench_*.json; do python -c "import json; d=json.loads([l for l in open('$f') if l.startswith('{')][-1]); print('$f', round(d['value'],1), {k:round(v['avg_ms'],2) for k,v in d['kernels'].items()})" 2>&1 | tail -1; done
