# round-2 evidence session
set -x
mkdir -p gpurun_out
nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.build()"
timeout 2700 python -m pytest tests -m gpu -x -q --durations=20 > gpurun_out/g11_tests.log 2>&1; tail -25 gpurun_out/g11_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g11_smoke.log 2>&1; tail -2 gpurun_out/g11_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/g11_bench_c4.json 2> gpurun_out/g11_bench_c4.err; tail -c 400 gpurun_out/g11_bench_c4.json
TANQ_BLOCK_K2=1 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g11_bench_c4_k2blk.json 2>&1
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g11_bench_c3.json 2>&1
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g11_bench_c2.json 2>&1
timeout 900 python bench.py --config 5 --n 16 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/g11_bench_c5.json 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g11_bench_ref.json 2>&1
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --config 4 --n 12 > gpurun_out/g11_bench_gpus2_shim.json 2>&1
timeout 900 python bench.py --gpus 2 --remap p2p --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g11_bench_gpus2_p2p.json 2>&1
timeout 900 python bench.py --shards 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/g11_bench_2vshards.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/g11_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --whole-n 0 > gpurun_out/g11_ncu_bench.log 2>&1
python scripts/launch_table.py gpurun_out/g11_launches_c4.csv gpurun_out/g11_launches_c4.md "ncu launch list, bench.py config 4 (QPE-16), round 2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:block_kernel -s 2 -c 2 -o gpurun_out/g11_block python scripts/prof_driver.py --config 4 --n 14 > gpurun_out/g11_ncu_block.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_kernel_tma -s 1 -c 1 -o gpurun_out/g11_block_tma python scripts/prof_group.py --n 14 --pairs 2,9:3,9 > gpurun_out/g11_ncu_tma.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_kernel -s 1 -c 1 -o gpurun_out/g11_block_rot python scripts/prof_group.py --n 14 --pairs 5,13:13,12 > gpurun_out/g11_ncu_rot.log 2>&1
TOOLS="racecheck synccheck memcheck" bash scripts/sanitize.sh > gpurun_out/g11_sanitize.txt 2>&1; grep -c 'SUMMARY' gpurun_out/g11_sanitize.txt
ls gpurun_out | grep g11
