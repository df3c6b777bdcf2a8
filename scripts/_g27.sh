set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/g27_build.log 2>&1
python scripts/fullsize_parity.py --config 4 --n 16 --prefix 160 > gpurun_out/g27_fullsize_qpe16_p160.jsonl 2> gpurun_out/g27_fullsize_qpe16_p160.err
