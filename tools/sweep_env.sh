# usage: VAR=SSCG_K2_GROUPS VALS="2 4 8" bash tools/sweep_env.sh
for g in $VALS; do
  env $VAR=$g timeout 150 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/b_g$g.json
  python -c "
import json; d=json.load(open('gpurun_out/b_g$g.json')); print('$VAR=$g', round(d['ms_per_step'],4), {k:round(v.get('ms_per_launch') or 0,4) for k,v in d['kernels'].items() if isinstance(v,dict) and v.get('ms_per_launch')})"
done
