mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29511"
python bench.py --workload large --steps 5 --no-cpu-baseline > gpurun_out/mg1_large1.log 2>&1
$T --nproc-per-node 2 bench.py --gpus 2 --workload large --steps 5 > gpurun_out/mg1_large2.log 2>&1
$T --nproc-per-node 4 bench.py --gpus 4 --workload large --steps 5 > gpurun_out/mg1_large4.log 2>&1
HEDDLE_PLACE_TRACE=1 $T --nproc-per-node 4 bench.py --gpus 4 --workload large --steps 2 --warmup 3 > gpurun_out/mg1_large4_trace.log 2>&1
HEDDLE_PLACE_TRACE=1 python bench.py --workload large --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/mg1_large1_trace.log 2>&1
$T --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/mg1_b2.log 2>&1
$T --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/mg1_b4.log 2>&1
$T --nproc-per-node 4 tests/mgpu_split_check.py > gpurun_out/mg1_splitcheck4.log 2>&1
echo done
