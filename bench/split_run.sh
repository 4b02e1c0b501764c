#!/bin/bash
# Multi-GPU evidence on one box with N GPUs: the split-mode parity test (golden + bit-identical
# across ranks and to 1 GPU), the configs[4] split bench with the fused NVLink exchange and with the
# NCCL all-gather baseline, the sharded configs[3] bench, and the 1-GPU large-instance line on the
# same box.
#   gpurun --gpus N -- 'bash bench/split_run.sh N tag'
N=${1:-2}; tag=${2:-r02}
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29561 --nproc-per-node $N"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_split${N}_build.log 2>&1
timeout 600 $T tests/mgpu_split_check.py > gpurun_out/${tag}_split${N}_check.log 2>&1; echo "check=$?" >> gpurun_out/${tag}_split${N}_status.txt
# the configs[4] split line with the fused exchange (no ncu here: ncu is never run on a multi-rank
# command; NVLink byte counters are unavailable on this pool)
timeout 300 $T bench.py --gpus $N --workload large --steps 5 --no-valley > gpurun_out/${tag}_split${N}_fused.out 2>gpurun_out/${tag}_split${N}_fused.err
grep '^{' gpurun_out/${tag}_split${N}_fused.out >> gpurun_out/${tag}_split${N}.jsonl
HEDDLE_PLACE_EXCHANGE=nccl timeout 300 $T bench.py --gpus $N --workload large --steps 5 --no-valley 2>gpurun_out/${tag}_split${N}_nccl.err | grep '^{' >> gpurun_out/${tag}_split${N}.jsonl
timeout 300 $T bench.py --gpus $N --steps 10 --no-valley --no-cpu-baseline --no-latency 2>gpurun_out/${tag}_shard${N}.err | grep '^{' >> gpurun_out/${tag}_split${N}.jsonl
timeout 300 python bench.py --workload large --steps 5 --no-valley --no-cpu-baseline 2>gpurun_out/${tag}_large1.err | grep '^{' >> gpurun_out/${tag}_split${N}.jsonl
echo done >> gpurun_out/${tag}_split${N}_status.txt
