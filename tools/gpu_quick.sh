timeout 1100 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pt.txt; cat gpurun_out/pt.txt
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $BENCHARGS 2>&1 | tail -1 > gpurun_out/b.json
python -c "
import json; d=json.load(open('gpurun_out/b.json')); print(d['ms_per_step'], {k:(round(v.get('ms_per_launch') or 0,4),round(v.get('frac') or 0,3)) for k,v in d['kernels'].items() if isinstance(v,dict) and v.get('ms_per_launch')})"
