set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g18_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_variants.py -x -q -k "64" > gpurun_out/g18_tests.log 2>&1; tail -3 gpurun_out/g18_tests.log
python bench.py --config 3 --no-cpu-baseline > gpurun_out/g18_bench_c3_k3.json 2>&1
python bench.py --config 3 --kmax 4 --no-cpu-baseline > gpurun_out/g18_bench_c3_k4.json 2>&1
python bench.py --kmax 4 --no-cpu-baseline --steps 5 > gpurun_out/g18_bench_c4_k4.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_kernel_tma -s 4 -c 1 -o gpurun_out/g18_tma python scripts/prof_driver.py --config 4 --n 14 > gpurun_out/g18_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_kernel -s 2 -c 2 -o gpurun_out/g18_blk_c3 python scripts/prof_driver.py --config 3 --n 14 > gpurun_out/g18_ncu2.log 2>&1
ls gpurun_out
