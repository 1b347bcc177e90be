C="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$C > gpurun_out/plain10.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1f' -s 10 -c 1 -o gpurun_out/prof_k1f $C > gpurun_out/ncu_k1f.log 2>&1; echo k1f=$?
