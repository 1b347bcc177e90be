timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu11.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu11.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench11.json 2> gpurun_out/bench11.err; echo bench=$?
tail -1 gpurun_out/bench11.json | cut -c1-400
