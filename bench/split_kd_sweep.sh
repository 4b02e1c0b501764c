#!/bin/bash
# configs[4] split over N GPUs: large off-diagonal chunks (HEDDLE_PLACE_K5_KC) with small diagonal
# chunks (HEDDLE_PLACE_K5_KD), 2 rounds.  Usage: gpurun --gpus N -- 'bash bench/split_kd_sweep.sh <tag> N'
TAG=${1:-kdsweep}; N=${2:-4}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29553 --nproc-per-node $N"
for rep in 1 2; do
for cfg in "0 0" "2048 512" "4096 512" "4096 1024" "2048 256"; do
  set -- $cfg
  if [ $1 = 0 ]; then unset HEDDLE_PLACE_K5_KC HEDDLE_PLACE_K5_KD; else export HEDDLE_PLACE_K5_KC=$1 HEDDLE_PLACE_K5_KD=$2; fi
  timeout 300 $T bench.py --gpus $N --workload large --steps 5 --no-valley 2>/dev/null | grep '^{' | sed "s/^{/{\"kc\": $1, \"kd\": $2, /" >> gpurun_out/${TAG}.jsonl
done
done
echo done
