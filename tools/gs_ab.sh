#!/bin/bash
# Same-box A/B of a K2R variant knob at cfg 5 (default SSCG_K2_IL; e.g.
# SSCG_GRAM_SPACE, R27): bench lines interleaved, then a launch list of each
# (ncu, serialised).   bash tools/gs_ab.sh [KNOB]
KNOB=${1:-SSCG_K2_IL}
mkdir -p gpurun_out
for rep in 1 2; do
  for m in 1 0; do
    env $KNOB=$m python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${KNOB}_${m}_$rep.json 2>gpurun_out/ab_${KNOB}_${m}_$rep.err
  done
done
for m in 1 0; do
  env $KNOB=$m ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ab_${KNOB}_launches_$m.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "== $KNOB=$m"; python tools/launch_table.py gpurun_out/ab_${KNOB}_launches_$m.csv
done
for f in gpurun_out/ab_${KNOB}_?_?.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f', round(d['ms_per_step'],4), {k:round(v.get('ms_per_launch') or 0,4) for k,v in d['kernels'].items() if isinstance(v,dict) and v.get('ms_per_launch')}, d['clocks']['sm_mhz'])"; done
