set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests/test_gpu_headline.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_device.py -x -q -m gpu > gpurun_out/g12_tests.log 2>&1; tail -3 gpurun_out/g12_tests.log
TOOLS=racecheck bash scripts/sanitize.sh > gpurun_out/g12_racecheck.txt 2>&1; grep -A8 'blocktma auto 1\|=== racecheck TANQ_GROUP=blocktma TANQ_K2PATH=auto TANQ_MIRROR=1' gpurun_out/g12_racecheck.txt | head -30
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/g12_bench_c4.json 2>&1; python -c "import json; d=json.loads([l for l in open('gpurun_out/g12_bench_c4.json') if l.startswith('{')][-1]); print(d['value'], d['e2e']['value'], d['kernels'])"
timeout 900 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g12_bench_c2.json 2>&1; python -c "import json; d=json.loads([l for l in open('gpurun_out/g12_bench_c2.json') if l.startswith('{')][-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'])"
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --config 4 --n 12 > gpurun_out/g12_bench_gpus2_shim.json 2>&1; tail -c 600 gpurun_out/g12_bench_gpus2_shim.json
