# usage: LIBS="a b c" [ARGS="--workload cfg4"] bash tools/sweep_libs.sh   (variant builds libsscg_<v>.so; "base" = libsscg.so)
for v in $LIBS; do
  if [ "$v" = base ]; then L=paper_2512_09642_b200/libsscg.so; else L=paper_2512_09642_b200/libsscg_$v.so; fi
  SSCG_LIB=$PWD/$L timeout 150 python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --no-e2e $ARGS 2>&1 | tail -1 > gpurun_out/b_$v.json
  python -c "
import json; d=json.load(open('gpurun_out/b_$v.json')); print('$v', round(d['ms_per_step'],4), {k:round(v.get('ms_per_launch') or 0,4) for k,v in d['kernels'].items() if isinstance(v,dict) and v.get('ms_per_launch')})" || tail -3 gpurun_out/b_$v.json
done
