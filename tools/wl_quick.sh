# quick per-kernel numbers for a list of workloads: WL="cfg5|cfg4 --s 4|..." bash tools/wl_quick.sh
IFS='|'
for a in $WL; do
  IFS=' '
  timeout 150 python bench.py --workload $a --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "
import json,sys
t=sys.stdin.read()
try:
    d=json.loads(t); print('$a', round(d['ms_per_step'],4), {k:(round(v.get('ms_per_launch') or 0,4), round(v.get('frac') or 0,3)) for k,v in d['kernels'].items() if isinstance(v,dict) and v.get('ms_per_launch')})
except Exception: print('$a FAILED', t[-300:])"
  IFS='|'
done
