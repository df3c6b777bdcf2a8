# Round-end measurement on one B200 (run through gpurun from the repo root).
set -x
python -c "import __graft_entry__ as g; g.build()"
python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.log 2>&1; tail -2 gpurun_out/f_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1
python bench.py > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err
python bench.py --config 3 > gpurun_out/f_bench_c3.json 2>&1
python bench.py --config 2 > gpurun_out/f_bench_c2.json 2>&1
python scripts/suite.py > gpurun_out/f_suite.jsonl 2>&1
python bench.py --impl reference > gpurun_out/f_bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/f_ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:group_kernel -s 3 -c 1 -o gpurun_out/f_group python scripts/prof_driver.py --config 4 --n 14 > gpurun_out/f_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gate2 -s 1 -c 1 -o gpurun_out/f_k2 python scripts/prof_k3.py --n 14 --qubits 0,1 > gpurun_out/f_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gate_kernel -s 1 -c 1 -o gpurun_out/f_k1 python scripts/prof_k3.py --n 14 --qubits 5 > gpurun_out/f_ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tile_kernel -s 1 -c 1 -o gpurun_out/f_tile python scripts/prof_driver.py --config 4 --n 14 > gpurun_out/f_ncu4.log 2>&1
ls gpurun_out/
