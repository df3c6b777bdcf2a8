set -x
mkdir -p gpurun_out
nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/g1_tests.log 2>&1; tail -25 gpurun_out/g1_tests.log
python bench.py --steps 5 --warmup 3 > gpurun_out/g1_bench_c4.json 2> gpurun_out/g1_bench_c4.err; tail -c 3000 gpurun_out/g1_bench_c4.json
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pipes microbench/pipes.cu && /tmp/pipes > gpurun_out/g1_pipes.txt 2>&1; cat gpurun_out/g1_pipes.txt
bash scripts/sanitize.sh > gpurun_out/g1_sanitize.txt 2>&1; tail -60 gpurun_out/g1_sanitize.txt
