set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
TANQ_BLOCK_COPY=u timeout 300 python /root/repo/scripts/_smk.py > gpurun_out/g7_smoke.log 2>&1; tail -6 gpurun_out/g7_smoke.log
for C in u bulk; do
  TANQ_BLOCK_COPY=$C timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g7_kbench_$C.jsonl 2>&1
  for D in 1 2; do TANQ_BLOCK_COPY=$C TANQ_DBG=$D timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g7_kbench_${C}_dbg$D.jsonl 2>&1; done
done
for f in gpurun_out/g7_kbench_*.jsonl; do echo $f; python -c "
import json
print([round(json.loads(l)['ms'],1) for l in open('$f') if l.startswith('{')])" 2>&1 | tail -2; done
for C in u bulk; do TANQ_BLOCK_COPY=$C timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g7_bench_$C.json 2> gpurun_out/g7_bench_$C.err; python -c "import json; d=json.load(open('gpurun_out/g7_bench_$C.json')); print('$C', d['value'], d['ms_per_step'], {k:round(v['avg_ms'],2) for k,v in d['kernels'].items()})" 2>&1 | tail -1; done
