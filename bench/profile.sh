#!/bin/bash
# ncu evidence for the dominant kernel (run under gpurun, one GPU).  Usage: bench/profile.sh <tag>
# 1) plain run of the same command (must exit 0 before ncu is used),
# 2) launch list with per-kernel device time (cold-cache, serialised: compare shares),
# 3) one --set full capture of k2_dp_batched.
set -e
TAG=${1:-r01}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-valley"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_dp_batched -s 3 -c 1 \
    -o gpurun_out/${TAG}_k2 $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
