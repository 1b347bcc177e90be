#!/bin/bash
# Same-box A/B of the w_{s-1} fold modes (SSCG_WL_FOLD = 0 / 1 / 2) at cfg 5:
# the bench line of each (event-timed) and a launch list (ncu, serialised).
mkdir -p gpurun_out
for m in 0 1 2; do
  SSCG_WL_FOLD=$m python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_bench_$m.json 2>gpurun_out/ab_bench_$m.err
done
for m in 0 1 2; do
  SSCG_WL_FOLD=$m ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/ab_launches_$m.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "== SSCG_WL_FOLD=$m"; python tools/launch_table.py gpurun_out/ab_launches_$m.csv
done
for m in 0 1 2; do python -c "
import json; d=json.loads(open('gpurun_out/ab_bench_$m.json').read().strip().splitlines()[-1])
print('fold $m', round(d['ms_per_step'],4), {k:(round(v.get('ms_per_launch') or 0,4),round(v.get('frac') or 0,3)) for k,v in d['kernels'].items() if isinstance(v,dict) and v.get('ms_per_launch')}, d['clocks']['sm_mhz'])"; done
