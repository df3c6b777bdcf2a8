set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g32_build.log 2>&1
python bench.py --config 3 --kmax 4 --no-cpu-baseline > gpurun_out/g32_c3_k4.json 2>&1
python bench.py --config 3 --kmax 5 --no-cpu-baseline > gpurun_out/g32_c3_k5.json 2>&1
TANQ_BLOCK_GROUP_MAX=8 python bench.py --config 3 --kmax 5 --no-cpu-baseline > gpurun_out/g32_c3_k5_g8.json 2>&1
TANQ_BLOCK_GROUP_MAX=4 python bench.py --config 3 --kmax 5 --no-cpu-baseline > gpurun_out/g32_c3_k5_g4.json 2>&1
TANQ_FWD_MERGE=0 python bench.py --config 3 --kmax 4 --no-cpu-baseline > gpurun_out/g32_c3_k4_nofwd.json 2>&1
