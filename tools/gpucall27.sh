timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu27.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu27.log | grep -v "^$" | tail -6
for w in "--workload cfg4" "--workload cfg4 --s 32" "--workload cfg3" "--workload cfg2"; do
  timeout 300 python bench.py $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/w.json 2>/tmp/w.err || { echo "$w FAILED"; tail -3 /tmp/w.err; continue; }
  tail -1 /tmp/w.json >> gpurun_out/workloads27.jsonl
  python - "$w" <<'PY'
import json, sys
d = json.loads(open('/tmp/w.json').read().strip().splitlines()[-1])
k = d['kernels']
print("%-28s GDOF/s %.3f ms/step %.4f path %.3f | K1 %.3f | K2 %.3f | K5 %.3f" % (sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['path_frac'], k['basis']['frac'], k['gram']['frac'], k['update']['frac']))
PY
done
