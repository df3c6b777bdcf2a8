set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_headline.py -x -q -k "qpe or cluster" > gpurun_out/g3_tests.log 2>&1; tail -3 gpurun_out/g3_tests.log
TANQ_BLOCK=1 timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g3_kbench_block1.jsonl 2>&1
TANQ_BLOCK=1 TANQ_DBG=2 timeout 600 python scripts/kbench.py --n 16 --groups-only --reps 5 > gpurun_out/g3_kbench_block1_dbg2.jsonl 2>&1
cat gpurun_out/g3_kbench_block1.jsonl gpurun_out/g3_kbench_block1_dbg2.jsonl | cut -c1-120
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_kernel -s 1 -c 1 -o gpurun_out/g3_block2 python scripts/prof_group.py --n 14 --pairs 5,13:13,12 > gpurun_out/g3_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_kernel -s 1 -c 1 -o gpurun_out/g3_block4 python scripts/prof_group.py --n 14 --pairs 11,12:12,13:11,13:12,11 > gpurun_out/g3_ncu4.log 2>&1
tail -3 gpurun_out/g3_ncu2.log gpurun_out/g3_ncu4.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g3_bench_c4.json 2> gpurun_out/g3_bench_c4.err; tail -c 600 gpurun_out/g3_bench_c4.json
