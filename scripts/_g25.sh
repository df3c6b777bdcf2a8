set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g25_build.log 2>&1
TANQ_GRAPH_DEBUG=1 python scripts/e2e_probe.py --config 2 > gpurun_out/g25_probe_new.log 2>&1
(cd abtest/old && python scripts/e2e_probe.py --config 2) > gpurun_out/g25_probe_old.log 2>&1
TANQ_BLOCK_TMA=1 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/g25_bench_tma1.json 2>&1
python bench.py --no-cpu-baseline --steps 5 > gpurun_out/g25_bench_default.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:block_kernel_tma -s 2 -c 1 -o gpurun_out/g25_tma python scripts/prof_driver.py --config 4 --n 14 > gpurun_out/g25_ncu1.log 2>&1
SAN_CASE=shards TANQ_MIRROR=1 timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 20 python -c "import sys; print(sys.version)" > gpurun_out/g25_san_probe1.log 2>&1
TOOLS=racecheck bash -x scripts/sanitize_r2.sh > gpurun_out/g25_san_racecheck.txt 2>&1
