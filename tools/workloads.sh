for w in "--workload cfg1" "--workload cfg2" "--workload cfg3" "--workload cfg4 --s 4" "--workload cfg4 --s 8" "--workload cfg4" "--workload cfg4 --s 24" "--workload cfg4 --s 32" "--workload cfg4 --n 384 --strong" "--workload cfg5 --nu 20"; do
  timeout 400 python bench.py $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/w.json 2>/tmp/w.err || { echo "$w FAILED"; tail -3 /tmp/w.err; continue; }
  tail -1 /tmp/w.json >> gpurun_out/workloads_final.jsonl
  python - "$w" <<'PY'
import json, sys
d = json.loads(open('/tmp/w.json').read().strip().splitlines()[-1])
k = d['kernels']
f = lambda n: "%.3f" % k[n]['frac'] if n in k and k[n].get('frac') else "-"   # KS (cfg 1): one launch
p64 = k.get('gram', {}).get('fp64_pipe')
print("%-34s GDOF/s %7.3f ms/step %8.4f path %.3f | K1 %s | K1 single %s | K2 %s (FP64 pipe %s) | K5 %s | K4 %.1f us" % (sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['path_frac'], f('basis'), f('basis_single'), f('gram'), ("%.3f %s" % (p64['frac'], p64['kernel'])) if p64 else "-", f('update'), k['fgs']['us_per_launch']))
PY
done
