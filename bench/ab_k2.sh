#!/bin/bash
# A/B of one BASELINE config over libraries in ab/, interleaved, 3 reps.
# Usage: [CFG=batched] [ALGO=scan] bench/ab_k2.sh <tag> <lib names: ab/libheddle_<name>.so, "new" = working tree>...
TAG=$1; shift
CFG=${CFG:-batched}; ALGO=${ALGO:-scan}
mkdir -p gpurun_out
for rep in 1 2 3; do
  for lib in "$@"; do
    if [ $lib = new ]; then unset HEDDLE_PLACE_LIB; else export HEDDLE_PLACE_LIB=$PWD/ab/libheddle_$lib.so; fi
    timeout 300 python bench/configs.py --only $CFG --algo $ALGO --reps 10 2>&1 | grep '^{' | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/${TAG}.jsonl
  done
done
echo done
