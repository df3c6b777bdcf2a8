set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_headline.py -x -q -k "qpe or cluster or many_tiles" > gpurun_out/g4_tests.log 2>&1; tail -3 gpurun_out/g4_tests.log
for C in bulk ldg; do
  TANQ_BLOCK_COPY=$C timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g4_kbench_$C.jsonl 2>&1
  for D in 1 2; do TANQ_BLOCK_COPY=$C TANQ_DBG=$D timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g4_kbench_${C}_dbg$D.jsonl 2>&1; done
done
for f in gpurun_out/g4_kbench_*.jsonl; do echo $f; cut -c1-110 $f; done
TANQ_BLOCK_COPY=ldg timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_kernel -s 1 -c 1 -o gpurun_out/g4_ldg2 python scripts/prof_group.py --n 14 --pairs 5,13:13,12 > gpurun_out/g4_ncu2.log 2>&1
for C in bulk ldg; do TANQ_BLOCK_COPY=$C timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g4_bench_$C.json 2> gpurun_out/g4_bench_$C.err; python -c "import json; d=json.load(open('gpurun_out/g4_bench_$C.json')); print('$C', d['value'], d['ms_per_step'], d['kernels'])"; done
