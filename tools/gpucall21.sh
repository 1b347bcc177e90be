timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu21.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu21.log
for v in "SSCG_K2_DUAL=1 --s 32" "SSCG_K2_DUAL=0 --s 32" "SSCG_K2_DUAL=1 --s 24" "SSCG_K2_DUAL=0 --s 24"; do
  e=${v%% *}; a=${v#* }
  env $e timeout 300 python bench.py --workload cfg4 $a --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/w.json 2>/tmp/w.err || { echo "$v FAILED"; tail -3 /tmp/w.err; continue; }
  python - "$v" <<'PY'
import json, sys
d = json.loads(open('/tmp/w.json').read().strip().splitlines()[-1])
k = d['kernels']
print("%-28s GDOF/s %.3f ms/step %.4f | K1 %.3f | K2 %.3f (%.3f ms) | K5 %.3f" % (sys.argv[1], d['value'], d['ms_per_step'], k['basis']['frac'], k['gram']['frac'], k['gram']['ms_per_launch'], k['update']['frac']))
PY
done
