#!/bin/bash
# large instance on 1 GPU: bigger chunks / fewer CTAs.  Usage: bench/k5big.sh <tag>
TAG=${1:-k5big}
mkdir -p gpurun_out
for rep in 1 2; do
  for s in 0:0 4096:2 8192:2 4096:1 8192:1; do
    kc=${s%%:*}; ctas=${s##*:}
    if [ $kc = 0 ]; then unset HEDDLE_PLACE_K5_KC HEDDLE_PLACE_K5_CTAS; else export HEDDLE_PLACE_K5_KC=$kc HEDDLE_PLACE_K5_CTAS=$ctas; fi
    timeout 300 python bench/configs.py --only large --reps 3 --kernel layered 2>&1 | grep '^{' | sed "s/^{/{\"kc\": $kc, \"ctas\": $ctas, /" >> gpurun_out/${TAG}.jsonl
  done
done
echo done
