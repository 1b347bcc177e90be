C="python bench.py --workload cfg4 --s 32 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$C > gpurun_out/plain16.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k2_gram|k1t' -s 70 -c 3 -o gpurun_out/prof_cfg4 $C > gpurun_out/ncu16.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu16.log
