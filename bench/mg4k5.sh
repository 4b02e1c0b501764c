#!/bin/bash
# 4-GPU evidence after the K5 rework: split bit-identity, split and sharded bench lines.  Usage: bench/mg4k5.sh <tag>
TAG=${1:-mg4}
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29521"
timeout 600 $T --nproc-per-node 4 tests/mgpu_split_check.py > gpurun_out/${TAG}_check4.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_check4.log
timeout 300 python bench.py --workload large --steps 5 --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/${TAG}.jsonl
timeout 300 $T --nproc-per-node 2 bench.py --gpus 2 --workload large --steps 5 2>&1 | grep '^{' >> gpurun_out/${TAG}.jsonl
timeout 300 $T --nproc-per-node 4 bench.py --gpus 4 --workload large --steps 5 2>&1 | grep '^{' >> gpurun_out/${TAG}.jsonl
HEDDLE_PLACE_EXCHANGE=nccl timeout 300 $T --nproc-per-node 4 bench.py --gpus 4 --workload large --steps 5 2>&1 | grep '^{' | sed 's/^{/{"exchange": "nccl", /' >> gpurun_out/${TAG}.jsonl
timeout 300 $T --nproc-per-node 2 bench.py --gpus 2 --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/${TAG}.jsonl
timeout 300 $T --nproc-per-node 4 bench.py --gpus 4 --no-cpu-baseline 2>&1 | grep '^{' >> gpurun_out/${TAG}.jsonl
echo done
