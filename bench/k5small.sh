#!/bin/bash
# K5 on the latency-bound configs: chunk size x resident CTAs per SM.  Usage: bench/k5small.sh <tag>
TAG=${1:-k5small}
mkdir -p gpurun_out
for cfg in tp_sweep paper_6.2; do
  for kc in 64 128 256; do
    for ctas in 1 2 3; do
      HEDDLE_PLACE_K5_KC=$kc HEDDLE_PLACE_K5_CTAS=$ctas timeout 300 python bench/configs.py --only $cfg --reps 5 --kernel layered 2>&1 | grep '^{' | sed "s/^{/{\"kc\": $kc, \"ctas\": $ctas, /" >> gpurun_out/${TAG}.jsonl
    done
  done
done
echo done
