#!/bin/bash
# usage: tools/sweep.sh N "ENV1" "ENV2" ...   -> prints per-variant K1/K2/K5 and ms/step
N=$1; shift
for v in "$@"; do
  env $v python bench.py --n $N --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/sw.json 2>/tmp/sw.err || { echo "$v FAILED"; tail -2 /tmp/sw.err; continue; }
  python - "$v" <<'PY'
import json, sys
d = json.loads(open('/tmp/sw.json').read().strip().splitlines()[-1])
k = d['kernels']
print("%-40s ms/step %.4f | K1 %.4f ms %.3f | K2 %.4f ms %.3f | K5 %.4f ms %.3f | K4 %.1f us" % (sys.argv[1], d['ms_per_step'],
      k['basis']['ms_per_launch'], k['basis']['frac'], k['gram']['ms_per_launch'], k['gram']['frac'],
      k['update']['ms_per_launch'], k['update']['frac'], k['fgs']['us_per_launch']))
PY
done
