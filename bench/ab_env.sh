#!/bin/bash
# A/B of an environment switch on configs[4] (1 GPU and the N-GPU split) and the TP sweep, interleaved,
# 2 rounds.  Usage: gpurun --gpus N -- 'bash bench/ab_env.sh <tag> N VAR val_a val_b'
TAG=$1; N=$2; VAR=$3; A=$4; B=$5
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29591"
for rep in 1 2; do
  for v in $A $B; do
    export $VAR=$v
    timeout 300 python bench.py --workload large --steps 5 --no-cpu-baseline --no-valley 2>&1 | grep '^{' | sed "s/^{/{\"$VAR\": \"$v\", /" >> gpurun_out/${TAG}.jsonl
    timeout 120 python bench/configs.py --only tp_sweep --reps 5 2>&1 | grep '^{' | sed "s/^{/{\"$VAR\": \"$v\", /" >> gpurun_out/${TAG}.jsonl
    if [ $N -gt 1 ]; then
      timeout 300 $T --nproc-per-node $N bench.py --gpus $N --workload large --steps 5 --no-valley 2>&1 | grep '^{' | sed "s/^{/{\"$VAR\": \"$v\", /" >> gpurun_out/${TAG}.jsonl
    fi
  done
done
echo done
