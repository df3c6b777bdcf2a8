set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g22_build.log 2>&1
for r in 1 2; do
python bench.py --no-cpu-baseline --steps 5 > gpurun_out/g22_new_$r.json 2>&1
(cd abtest/old && python bench.py --no-cpu-baseline --steps 5) > gpurun_out/g22_old_$r.json 2>&1
done
python bench.py --config 4 --shards 2 --no-cpu-baseline > gpurun_out/g22_2vs.json 2>&1
python bench.py --gpus 2 --steps 3 --warmup 3 --qubits 12 > gpurun_out/g22_gpus2_shim.json 2>&1
