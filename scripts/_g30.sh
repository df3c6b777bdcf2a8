set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g30_build.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/g30_tests.log 2>&1; tail -3 gpurun_out/g30_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g30_smoke.log 2>&1
python bench.py --gpus 8 --config 5 --qubits 12 --steps 3 --warmup 3 > gpurun_out/g30_gpus8_c5.json 2>&1
