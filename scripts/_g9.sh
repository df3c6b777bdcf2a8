set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for M in 1 auto; do TANQ_BLOCK_TMA=$M timeout 300 python scripts/_smk.py > gpurun_out/g9_smoke_$M.log 2>&1; echo "tma=$M"; tail -6 gpurun_out/g9_smoke_$M.log; done
TANQ_BLOCK_TMA=1 timeout 1500 python -m pytest tests/test_gpu_headline.py -x -q > gpurun_out/g9_tests_tma1.log 2>&1; tail -3 gpurun_out/g9_tests_tma1.log
for M in 1 auto 0; do
  TANQ_BLOCK_TMA=$M timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g9_kbench_$M.jsonl 2>&1
  TANQ_BLOCK_TMA=$M TANQ_DBG=1 timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g9_kbench_${M}_dbg1.jsonl 2>&1
  TANQ_BLOCK_TMA=$M timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g9_bench_$M.json 2> gpurun_out/g9_bench_$M.err
done
for f in gpurun_out/g9_kbench_*.jsonl; do echo $f; python -c "
import json
print([round(json.loads(l)['ms'],1) for l in open('$f') if l.startswith('{')])" 2>&1 | tail -1; done
for f in gpurun_out/g9_bench_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['ms_per_step'],1), {k:round(v['avg_ms'],2) for k,v in d['kernels'].items()})" 2>&1 | tail -1; done
