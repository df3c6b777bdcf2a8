set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g20_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py -x -q > gpurun_out/g20_tests.log 2>&1; tail -3 gpurun_out/g20_tests.log
python bench.py --no-cpu-baseline --steps 5 > gpurun_out/g20_bench_c4_rb.json 2>&1
TANQ_RBASIS=0 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/g20_bench_c4_norb.json 2>&1
python bench.py --kmax 5 --no-cpu-baseline --steps 5 > gpurun_out/g20_bench_c4_k5.json 2>&1
python bench.py --kmax 4 --no-cpu-baseline --steps 5 > gpurun_out/g20_bench_c4_k4.json 2>&1
python bench.py --config 3 --no-cpu-baseline > gpurun_out/g20_bench_c3_k3.json 2>&1
python bench.py --config 3 --kmax 4 --no-cpu-baseline > gpurun_out/g20_bench_c3_k4.json 2>&1
python bench.py --config 3 --kmax 5 --no-cpu-baseline > gpurun_out/g20_bench_c3_k5.json 2>&1
TANQ_RBASIS=0 python bench.py --config 3 --kmax 4 --no-cpu-baseline > gpurun_out/g20_bench_c3_k4_norb.json 2>&1
