set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g28_build.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g28_smoke.log 2>&1
python bench.py > gpurun_out/g28_bench_c4.json 2> gpurun_out/g28_bench_c4.err
python bench.py --config 3 --no-cpu-baseline > gpurun_out/g28_bench_c3.json 2>&1
python bench.py --config 3 --kmax 4 --no-cpu-baseline > gpurun_out/g28_bench_c3_k4.json 2>&1
python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g28_bench_c2.json 2>&1
python bench.py --config 5 --qubits 16 --no-cpu-baseline > gpurun_out/g28_bench_c5.json 2>&1
python bench.py --config 4 --shards 2 --no-cpu-baseline > gpurun_out/g28_bench_2vs.json 2>&1
python bench.py --impl reference > gpurun_out/g28_bench_ref.json 2>&1
