#!/bin/bash
# split mode (configs[4]) on N GPUs after a K5 change: bit-identity check, then bench lines.  Usage: bench/mg2k5.sh <tag> <N>
TAG=${1:-mgk5}; N=${2:-2}
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29517 --nproc-per-node $N"
timeout 600 $T tests/mgpu_split_check.py > gpurun_out/${TAG}_check.log 2>&1; echo "check rc=$?" >> gpurun_out/${TAG}_check.log
for kd in 0 256; do
  [ "$kd" = 0 ] && unset HEDDLE_PLACE_K5_KD || export HEDDLE_PLACE_K5_KD=$kd
  timeout 300 $T bench.py --gpus $N --workload large --steps 5 2>&1 | grep '^{' | sed "s/^{/{\"kd\": $kd, /" >> gpurun_out/${TAG}.jsonl
done
unset HEDDLE_PLACE_K5_KD
timeout 300 python bench.py --workload large --steps 5 --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/${TAG}.jsonl
echo done
