mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29515"
timeout 300 python bench/configs.py --only large --reps 3 2>&1 | grep '^{' >> gpurun_out/mg5_large1.jsonl
HEDDLE_PLACE_K5_KC=1024 timeout 300 python bench/configs.py --only large --reps 3 2>&1 | grep '^{' | sed "s/^{/{\"kc\": 1024, /" >> gpurun_out/mg5_large1.jsonl
for kc in 512 1024; do
  HEDDLE_PLACE_K5_KC=$kc timeout 300 $T --nproc-per-node 4 bench.py --gpus 4 --workload large --steps 3 2>&1 | grep '^{' | sed "s/^{/{\"kc\": $kc, /" >> gpurun_out/mg5_large4.jsonl
done
timeout 300 python bench/configs.py --only tp_sweep --reps 3 2>&1 | grep '^{' >> gpurun_out/mg5_large1.jsonl
echo done
