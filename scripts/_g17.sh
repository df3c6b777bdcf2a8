set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g17_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_variants.py -x -q > gpurun_out/g17_tests.log 2>&1; tail -3 gpurun_out/g17_tests.log
TANQ_SPARSE_MAX=0 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/g17_bench_dense.json 2>&1
python bench.py --no-cpu-baseline --steps 5 > gpurun_out/g17_bench_sparse.json 2>&1
python bench.py --no-cpu-baseline --steps 5 --kmax 4 > gpurun_out/g17_bench_sparse_k4.json 2>&1
python bench.py --config 2 --no-cpu-baseline > gpurun_out/g17_bench_c2.json 2>&1
python bench.py --config 5 --no-cpu-baseline > gpurun_out/g17_bench_c5.json 2>&1
