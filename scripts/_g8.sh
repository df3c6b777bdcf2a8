set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
for V in "bulk 0" "bs 0" "bulk 1" "bs 1"; do set -- $V
  TANQ_BLOCK_COPY=$1 TANQ_BLOCK_ACC=$2 timeout 300 python scripts/_smk.py > gpurun_out/g8_smoke_$1_$2.log 2>&1; echo "$1 $2"; tail -2 gpurun_out/g8_smoke_$1_$2.log
  TANQ_BLOCK_COPY=$1 TANQ_BLOCK_ACC=$2 timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g8_kbench_$1_$2.jsonl 2>&1
  TANQ_BLOCK_COPY=$1 TANQ_BLOCK_ACC=$2 TANQ_DBG=2 timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g8_kbench_$1_$2_dbg2.jsonl 2>&1
  TANQ_BLOCK_COPY=$1 TANQ_BLOCK_ACC=$2 TANQ_DBG=1 timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g8_kbench_$1_$2_dbg1.jsonl 2>&1
  TANQ_BLOCK_COPY=$1 TANQ_BLOCK_ACC=$2 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g8_bench_$1_$2.json 2> gpurun_out/g8_bench_$1_$2.err
done
for f in gpurun_out/g8_kbench_*.jsonl; do echo $f; python -c "
import json
print([round(json.loads(l)['ms'],1) for l in open('$f') if l.startswith('{')])" 2>&1 | tail -1; done
for f in gpurun_out/g8_bench_*.json; do python -c "import json; d=json.load(open('$f')); print('$f', round(d['value'],1), round(d['ms_per_step'],1), {k:round(v['avg_ms'],2) for k,v in d['kernels'].items()})" 2>&1 | tail -1; done
