# ncu --set full of chosen kernels at other workloads (after a plain run of each command)
set -x
C4="python bench.py --workload cfg4 --s 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
C32="python bench.py --workload cfg4 --s 32 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
C2="python bench.py --workload cfg2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
TAG=${1:-rXX}
$C4 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2r -s 3 -c 1 -o gpurun_out/prof_${TAG}_cfg4s4_k2r $C4 > /dev/null 2>&1
$C32 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2r -s 3 -c 1 -o gpurun_out/prof_${TAG}_cfg4s32_k2r $C32 > /dev/null 2>&1
$C2 > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2r|k1t" -s 40 -c 2 -o gpurun_out/prof_${TAG}_cfg2 $C2 > /dev/null 2>&1
$C2 > /dev/null 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_cfg2.csv $C2 > /dev/null 2>&1
ls gpurun_out
