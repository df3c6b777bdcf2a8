set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g31_build.log 2>&1
python -m pytest tests/test_gpu_parity.py -x -q -k "parity_packed" > gpurun_out/g31_tests.log 2>&1; tail -3 gpurun_out/g31_tests.log
