C="python bench.py --workload cfg4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$C > gpurun_out/plain18.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1t' -s 40 -c 1 -o gpurun_out/prof_k1t4 $C > gpurun_out/ncu18.log 2>&1; echo ncu=$?
