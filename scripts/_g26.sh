set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g26_build.log 2>&1
python scripts/fullsize_parity.py --config 4 --n 15 > gpurun_out/g26_fullsize_qpe15.jsonl 2> gpurun_out/g26_fullsize_qpe15.err
