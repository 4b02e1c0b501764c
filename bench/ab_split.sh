#!/bin/bash
# A/B of ab/libheddle_head.so vs the working tree on configs[4]: 1 GPU and the N-GPU split (fused
# exchange), interleaved, 2 rounds.  Usage: gpurun --gpus N -- 'bash bench/ab_split.sh <tag> N'
TAG=${1:-absplit}; N=${2:-4}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29541"
for rep in 1 2; do
  for lib in head new; do
    if [ $lib = head ]; then export HEDDLE_PLACE_LIB=$PWD/ab/libheddle_head.so; else unset HEDDLE_PLACE_LIB; fi
    timeout 300 python bench.py --workload large --steps 5 --no-cpu-baseline --no-valley 2>&1 | grep '^{' | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/${TAG}.jsonl
    timeout 300 $T --nproc-per-node $N bench.py --gpus $N --workload large --steps 5 --no-valley 2>&1 | grep '^{' | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/${TAG}.jsonl
  done
done
unset HEDDLE_PLACE_LIB
echo done
