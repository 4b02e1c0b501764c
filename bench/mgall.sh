#!/bin/bash
# K5 (kc, CTAs/SM) for the large instance at 1, 2 and 4 GPUs (one box).  Usage: bench/mgall.sh <tag>
TAG=${1:-mgall}
mkdir -p gpurun_out
run() {  # N kc ctas
  if [ $1 = 1 ]; then
    HEDDLE_PLACE_K5_KC=$2 HEDDLE_PLACE_K5_CTAS=$3 timeout 300 python bench.py --workload large --steps 5 --no-cpu-baseline 2>&1 | grep '^{' | sed "s/^{/{\"kc\": $2, \"ctas\": $3, /" >> gpurun_out/${TAG}.jsonl
  else
    HEDDLE_PLACE_K5_KC=$2 HEDDLE_PLACE_K5_CTAS=$3 timeout 300 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29529 --nproc-per-node $1 bench.py --gpus $1 --workload large --steps 5 2>&1 | grep '^{' | sed "s/^{/{\"kc\": $2, \"ctas\": $3, /" >> gpurun_out/${TAG}.jsonl
  fi
}
for rep in 1 2; do
  run 1 2048 3; run 1 2048 2; run 1 4096 2
  run 2 1024 3; run 2 1024 2; run 2 2048 2
  run 4 1024 2; run 4 2048 2; run 4 1024 1
done
echo done
