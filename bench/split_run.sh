#!/bin/bash
# Multi-GPU evidence on one box with N GPUs: the split-mode parity test (golden + bit-identical
# across ranks and to 1 GPU), the configs[4] split bench with the fused NVLink exchange and with the
# NCCL all-gather baseline (NVML NVLink byte counters in the line), the sharded configs[3] bench,
# and the 1-GPU large-instance line on the same box.
#   gpurun --gpus N -- 'bash bench/split_run.sh N tag'
N=${1:-2}; tag=${2:-r02}
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29561 --nproc-per-node $N"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_split${N}_build.log 2>&1
timeout 600 $T tests/mgpu_split_check.py > gpurun_out/${tag}_split${N}_check.log 2>&1; echo "check=$?" >> gpurun_out/${tag}_split${N}_status.txt
# then NVLink bytes of one K5 launch in split mode, from ncu on rank 0 only (nvltx / nvlrx counters;
# NVML's NVLink throughput counters read N/A on this pool: profiles/r02_nvlink_probe.json), right
# after the same command line exited 0 without ncu
timeout 300 $T bench.py --gpus $N --workload large --steps 5 --no-valley > gpurun_out/${tag}_split${N}_fused.out 2>gpurun_out/${tag}_split${N}_fused.err && \
timeout 600 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29571 --nproc-per-node $N \
    --no-python bash bench/rank0_ncu.sh ${tag}_split${N} python bench.py --gpus $N --workload large --steps 5 \
    --no-valley > gpurun_out/${tag}_split${N}_ncu.log 2>&1; echo "ncu=$?" >> gpurun_out/${tag}_split${N}_status.txt
grep '^{' gpurun_out/${tag}_split${N}_fused.out >> gpurun_out/${tag}_split${N}.jsonl
HEDDLE_PLACE_EXCHANGE=nccl timeout 300 $T bench.py --gpus $N --workload large --steps 5 --no-valley 2>gpurun_out/${tag}_split${N}_nccl.err | grep '^{' >> gpurun_out/${tag}_split${N}.jsonl
timeout 300 $T bench.py --gpus $N --steps 10 --no-valley --no-cpu-baseline --no-latency 2>gpurun_out/${tag}_shard${N}.err | grep '^{' >> gpurun_out/${tag}_split${N}.jsonl
timeout 300 python bench.py --workload large --steps 5 --no-valley --no-cpu-baseline 2>gpurun_out/${tag}_large1.err | grep '^{' >> gpurun_out/${tag}_split${N}.jsonl
echo done >> gpurun_out/${tag}_split${N}_status.txt
