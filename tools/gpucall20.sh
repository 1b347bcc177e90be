C="python bench.py --workload cfg4 --s 32 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$C > gpurun_out/plain20.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k2_gram' -s 2 -c 1 -o gpurun_out/prof_k2s32 $C > gpurun_out/ncu20.log 2>&1; echo ncu=$?
