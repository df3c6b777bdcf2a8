set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g19_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_headline.py -x -q -k "kmax5 or many_tiles" > gpurun_out/g19_tests.log 2>&1; tail -3 gpurun_out/g19_tests.log
python bench.py --config 3 --kmax 5 --no-cpu-baseline > gpurun_out/g19_bench_c3_k5.json 2>&1
python bench.py --config 3 --kmax 4 --no-cpu-baseline > gpurun_out/g19_bench_c3_k4.json 2>&1
python bench.py --kmax 5 --no-cpu-baseline --steps 5 > gpurun_out/g19_bench_c4_k5.json 2>&1
TANQ_BLOCK_ACC=2 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/g19_bench_c4_acc2.json 2>&1
python bench.py --config 2 --kmax 5 --no-cpu-baseline > gpurun_out/g19_bench_c2_k5.json 2>&1
