# K5 tile-size / residency sweep on the large instance (1 GPU and 4-GPU split)
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29512"
for kc in 256 512 1024 2048; do
  HEDDLE_PLACE_K5_KC=$kc python bench/configs.py --only large --reps 3 2>&1 | grep '^{' | sed "s/^{/{\"kc\": $kc, /" >> gpurun_out/mg2_kc1.jsonl
done
for kc in 512 1024; do for ctas in 2 3 4; do
  HEDDLE_PLACE_K5_KC=$kc HEDDLE_PLACE_K5_CTAS=$ctas $T --nproc-per-node 4 bench.py --gpus 4 --workload large --steps 3 2>&1 | grep '^{' | sed "s/^{/{\"kc\": $kc, \"ctas\": $ctas, /" >> gpurun_out/mg2_kc4.jsonl
done; done
echo done
