set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
TANQ_BLOCK_TMA=auto timeout 300 python scripts/_smk.py > gpurun_out/g10_smoke.log 2>&1; tail -3 gpurun_out/g10_smoke.log
for S in 0 1 2; do TANQ_BLOCK_TMA_SLACK=$S timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g10_bench_s$S.json 2> gpurun_out/g10_bench_s$S.err; done
for f in gpurun_out/g10_bench_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['ms_per_step'],1), {k:round(v['avg_ms'],2) for k,v in d['kernels'].items()})" 2>&1 | tail -1; done
