./tools/membw > gpurun_out/membw.txt 2>&1; cat gpurun_out/membw.txt
C="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$C > gpurun_out/plain13.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k2_gram|k5_update|k4_fgs|k1f' -s 12 -c 4 -o gpurun_out/prof_all $C > gpurun_out/ncu_all.log 2>&1; echo ncu=$?
