#!/bin/bash
# Evidence for profiles/ (run on a B200 through gpurun; see B200_PROFILING.md):
#   bash tools/profile_round.sh <tag>
# 1. the bench line, 2. the per-launch device times of the same command under
# ncu (shares, not absolutes), 3. one `ncu --set full` capture per hot kernel,
# 4. the HBM read/write mix ceilings.  Each ncu run follows a plain run of the
# same command that exited 0.
set -e
TAG=${1:-rXX}
ONLY=${2:-all}
mkdir -p gpurun_out
C="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
[ "$ONLY" = all ] && python bench.py > gpurun_out/bench_$TAG.json
$C > gpurun_out/plain_$TAG.log 2>&1
[ "$ONLY" = all ] && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $C > /dev/null 2>&1
# skip the warm-up launches: K1M runs 5x per outer (s = 16), K2R/K5 once (10 outer iterations in this command)
for ks in "k1m 8" "k2r 3" "k5_update 3"; do
  set -- $ks
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 -o gpurun_out/prof_${TAG}_$1 $C > /dev/null 2>&1
done
[ "$ONLY" = all ] && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/membw tools/membw.cu && /tmp/membw > gpurun_out/membw_$TAG.txt
# then, here: python tools/launch_shares.py gpurun_out/launches_$TAG.csv > profiles/${TAG}_launches448_shares.txt
#             python tools/ncu_raw_summary.py profiles/${TAG}_ncu_full_448.json gpurun_out/prof_${TAG}_*.ncu-rep > profiles/${TAG}_ncu_full_448.txt
