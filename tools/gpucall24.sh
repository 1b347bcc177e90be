timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu24.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu24.log
python bench.py --no-cpu-baseline > gpurun_out/bench24.json 2>gpurun_out/bench24.err; echo bench=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench24.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e'], d['roofline']['frac'])"
