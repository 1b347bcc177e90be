C="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1_lap_vec' -s 20 -c 1 -o gpurun_out/prof_k1 $C > gpurun_out/ncu_k1.log 2>&1; echo k1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k2_gram' -s 1 -c 1 -o gpurun_out/prof_k2 $C > gpurun_out/ncu_k2.log 2>&1; echo k2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k5_update' -s 1 -c 1 -o gpurun_out/prof_k5 $C > gpurun_out/ncu_k5.log 2>&1; echo k5=$?
