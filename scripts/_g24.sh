set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g24_build.log 2>&1
bash scripts/sanitize_r2.sh > gpurun_out/g24_sanitize_r2.txt 2>&1
python bench.py --gpus 2 --remap p2p --no-cpu-baseline > gpurun_out/g24_bench_p2p.json 2>&1
nproc > gpurun_out/g24_nproc.txt; free -g >> gpurun_out/g24_nproc.txt
python scripts/fullsize_parity.py --config 4 --n 16 > gpurun_out/g24_fullsize_qpe16.jsonl 2> gpurun_out/g24_fullsize_qpe16.err
