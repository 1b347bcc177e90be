timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu23.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu23.log
for v in "SSCG_PDL=1 --workload cfg2" "SSCG_PDL=0 --workload cfg2" "SSCG_PDL=1 --workload cfg5" "SSCG_PDL=0 --workload cfg5" "SSCG_PDL=1 --workload cfg3"; do
  e=${v%% *}; a=${v#* }
  env $e timeout 300 python bench.py $a --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/w.json 2>/tmp/w.err || { echo "$v FAILED"; tail -3 /tmp/w.err; continue; }
  python - "$v" <<'PY'
import json, sys
d = json.loads(open('/tmp/w.json').read().strip().splitlines()[-1])
k = d['kernels']
print("%-28s GDOF/s %.3f ms/step %.4f | K1 %.3f | K2 %.3f (%.4f ms) | K5 %.3f" % (sys.argv[1], d['value'], d['ms_per_step'], k['basis']['frac'], k['gram']['frac'], k['gram']['ms_per_launch'], k['update']['frac']))
PY
done
