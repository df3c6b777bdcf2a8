set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g23_build.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/g23_tests.log 2>&1; tail -3 gpurun_out/g23_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g23_smoke.log 2>&1
python bench.py > gpurun_out/g23_bench_c4.json 2> gpurun_out/g23_bench_c4.err
python bench.py --config 3 --no-cpu-baseline > gpurun_out/g23_bench_c3.json 2>&1
python bench.py --config 3 --kmax 4 --no-cpu-baseline > gpurun_out/g23_bench_c3_k4.json 2>&1
python bench.py --config 2 --no-cpu-baseline > gpurun_out/g23_bench_c2.json 2>&1
python bench.py --config 4 --shards 4 --no-cpu-baseline > gpurun_out/g23_bench_4vs.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g23_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g23_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:block_kernel -s 4 -c 2 -o gpurun_out/g23_block python scripts/prof_driver.py --config 4 --n 14 > gpurun_out/g23_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:parity_swap -s 0 -c 1 -o gpurun_out/g23_parity python bench.py --config 4 --qubits 12 --shards 2 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/g23_ncu2.log 2>&1
ls gpurun_out | grep g23
