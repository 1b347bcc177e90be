C="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$C > gpurun_out/plain25.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches25.csv $C > gpurun_out/ncu25a.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k1f' -s 10 -c 1 -o gpurun_out/prof25_k1f $C > gpurun_out/ncu25b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k2_gram' -s 3 -c 1 -o gpurun_out/prof25_k2 $C > gpurun_out/ncu25c.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k5_update' -s 3 -c 1 -o gpurun_out/prof25_k5 $C > gpurun_out/ncu25d.log 2>&1; echo ncu=$?
