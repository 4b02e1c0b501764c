#!/bin/bash
# A/B of ab/libheddle_head.so vs the working tree on the large instance at 1/2/4 GPUs and the
# latency-bound configs; then the 4-GPU split bit-identity check.  Usage: bench/abmg.sh <tag>
TAG=${1:-abmg}
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29531"
for rep in 1 2; do
  for lib in head new; do
    if [ $lib = head ]; then export HEDDLE_PLACE_LIB=$PWD/ab/libheddle_head.so; else unset HEDDLE_PLACE_LIB; fi
    for cfg in tp_sweep paper_6.2; do
      timeout 300 python bench/configs.py --only $cfg --reps 5 --kernel layered 2>&1 | grep '^{' | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/${TAG}.jsonl
    done
    timeout 300 python bench.py --workload large --steps 5 --no-cpu-baseline 2>&1 | grep '^{' | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/${TAG}.jsonl
    for N in 2 4; do
      timeout 300 $T --nproc-per-node $N bench.py --gpus $N --workload large --steps 5 2>&1 | grep '^{' | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/${TAG}.jsonl
    done
  done
done
unset HEDDLE_PLACE_LIB
timeout 600 $T --nproc-per-node 4 tests/mgpu_split_check.py > gpurun_out/${TAG}_check4.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_check4.log
timeout 600 python -m pytest tests/test_gpu_k5_trace.py tests/test_gpu_parity.py -m gpu -x -q -k "k5 or layered or split or large or tp_sweep" > gpurun_out/${TAG}_pytest.log 2>&1
echo done
