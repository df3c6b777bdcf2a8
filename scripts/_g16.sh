set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g16_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "shards or config4" > gpurun_out/g16_tests.log 2>&1; tail -3 gpurun_out/g16_tests.log
timeout 1200 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/g16_dist.log 2>&1; tail -3 gpurun_out/g16_dist.log
python bench.py --config 4 --shards 2 --no-cpu-baseline > gpurun_out/g16_bench_2vs.json 2>&1
python bench.py --config 4 --shards 4 --no-cpu-baseline > gpurun_out/g16_bench_4vs.json 2>&1
