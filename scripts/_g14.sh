set -x
mkdir -p gpurun_out
nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.build()"
TOOLS=racecheck bash scripts/sanitize.sh > gpurun_out/g14_racecheck.txt 2>&1; grep -A3 'blocktma' gpurun_out/g14_racecheck.txt | head -20
timeout 1800 python scripts/fullsize_parity.py --config 4 --n 14 > gpurun_out/g14_qpe14_full.json 2>&1; tail -2 gpurun_out/g14_qpe14_full.json
timeout 1200 python scripts/fullsize_parity.py --config 3 --n 12 --depth 100 > gpurun_out/g14_c3_n12_d100.json 2>&1; tail -2 gpurun_out/g14_c3_n12_d100.json
TANQ_FULLSIZE=1 timeout 3000 python -m pytest tests/test_gpu_headline.py -q -k "qpe16_prefix or cluster_product_vs_oracle" --durations=5 > gpurun_out/g14_fullsize.log 2>&1; tail -12 gpurun_out/g14_fullsize.log
