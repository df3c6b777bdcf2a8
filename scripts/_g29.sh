set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g29_build.log 2>&1
python bench.py --gpus 4 --qubits 12 --steps 3 --warmup 3 > gpurun_out/g29_gpus4.json 2>&1
python bench.py --gpus 8 --qubits 12 --steps 3 --warmup 3 > gpurun_out/g29_gpus8.json 2>&1
python bench.py --gpus 8 --config 5 --qubits 12 --steps 3 --warmup 3 > gpurun_out/g29_gpus8_c5.json 2>&1
