#!/bin/bash
# A/B of the paper-call-shape latency lines (bench.latency_lines: rollout / TP sweep / §6.2, device
# time from a CUDA graph) and the batched valley config over libraries in ab/, interleaved.
# Usage: bench/ab_latency.sh <tag> <lib names: ab/libheddle_<name>.so, "new" = working tree>...
TAG=$1; shift
mkdir -p gpurun_out
for rep in 1 2 3; do
  for lib in "$@"; do
    if [ $lib = new ]; then unset HEDDLE_PLACE_LIB; else export HEDDLE_PLACE_LIB=$PWD/ab/libheddle_$lib.so; fi
    timeout 300 python -c "
import json, torch, bench
r = bench.latency_lines(torch.device('cuda:0'))
print(json.dumps({'lib': '$lib', 'rep': $rep, 'latency': r}))" 2>&1 | grep '^{' >> gpurun_out/${TAG}.jsonl
    timeout 300 python bench/configs.py --only batched --algo valley --reps 5 2>&1 | grep '^{' | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/${TAG}.jsonl
  done
done
echo done
