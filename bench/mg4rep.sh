#!/bin/bash
# split large instance on N GPUs: repeated, interleaved K5 (kc, CTAs/SM) settings.  Usage: bench/mg4rep.sh <tag> <N> "kc:ctas ..."
TAG=${1:-mg4rep}; N=${2:-4}; SETS=${3:-"512:3 1024:2 1024:3 768:3"}
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29527 --nproc-per-node $N"
for rep in 1 2; do
  for s in $SETS; do
    kc=${s%%:*}; ctas=${s##*:}
    HEDDLE_PLACE_K5_KC=$kc HEDDLE_PLACE_K5_CTAS=$ctas timeout 300 $T bench.py --gpus $N --workload large --steps 5 2>&1 | grep '^{' | sed "s/^{/{\"kc\": $kc, \"ctas\": $ctas, \"rep\": $rep, /" >> gpurun_out/${TAG}.jsonl
  done
done
echo done
