set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g15_build.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/g15_tests.log 2>&1; tail -3 gpurun_out/g15_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g15_smoke.log 2>&1
python bench.py > gpurun_out/g15_bench_c4.json 2> gpurun_out/g15_bench_c4.err
python bench.py --config 4 --shards 2 --no-cpu-baseline > gpurun_out/g15_bench_2vs.json 2>&1
python bench.py --config 3 --no-cpu-baseline > gpurun_out/g15_bench_c3.json 2>&1
