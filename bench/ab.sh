#!/bin/bash
# A/B on one box: ab/libheddle_head.so (previous commit) vs the working tree's library, interleaved.
# Usage: bench/ab.sh <tag> <N gpus> [configs]
TAG=${1:-ab}; N=${2:-1}; CFGS=${3:-"large tp_sweep paper_6.2"}
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29519 --nproc-per-node $N"
for rep in 1 2; do
  for lib in head new; do
    if [ $lib = head ]; then export HEDDLE_PLACE_LIB=$PWD/ab/libheddle_head.so; else unset HEDDLE_PLACE_LIB; fi
    for cfg in $CFGS; do
      timeout 300 python bench/configs.py --only $cfg --reps 5 --kernel layered 2>&1 | grep '^{' | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/${TAG}.jsonl
    done
    if [ $N -gt 1 ]; then
      timeout 300 $T bench.py --gpus $N --workload large --steps 5 2>&1 | grep '^{' | sed "s/^{/{\"lib\": \"$lib\", \"config\": \"split$N\", /" >> gpurun_out/${TAG}.jsonl
    fi
  done
done
echo done
