#!/bin/bash
# split large instance on N GPUs: K5 chunk size x resident CTAs.  Usage: bench/mg4sweep.sh <tag> <N>
TAG=${1:-mg4sw}; N=${2:-4}
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29525 --nproc-per-node $N"
for kc in 512 1024 2048; do
  for ctas in 2 3; do
    HEDDLE_PLACE_K5_KC=$kc HEDDLE_PLACE_K5_CTAS=$ctas timeout 300 $T bench.py --gpus $N --workload large --steps 5 2>&1 | grep '^{' | sed "s/^{/{\"kc\": $kc, \"ctas\": $ctas, /" >> gpurun_out/${TAG}.jsonl
  done
done
echo done
