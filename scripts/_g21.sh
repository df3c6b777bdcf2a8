set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g21_build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g21_smoke.log 2>&1
python bench.py > gpurun_out/g21_bench_c4.json 2> gpurun_out/g21_bench_c4.err
python bench.py --impl reference > gpurun_out/g21_bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g21_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/g21_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:block_kernel -s 4 -c 2 -o gpurun_out/g21_block python scripts/prof_driver.py --config 4 --n 14 > gpurun_out/g21_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:parity_swap -s 0 -c 1 -o gpurun_out/g21_parity python bench.py --config 4 --qubits 12 --shards 2 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/g21_ncu2.log 2>&1
ls gpurun_out | grep g21
