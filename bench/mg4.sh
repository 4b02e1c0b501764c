mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29514"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/mg4_pytest.log 2>&1; echo "pytest=$?" >> gpurun_out/mg4_status.txt
timeout 300 $T --nproc-per-node 4 tests/mgpu_split_check.py > gpurun_out/mg4_split4.log 2>&1; echo "split4=$?" >> gpurun_out/mg4_status.txt
for top in 0 256; do
  if [ $top = 0 ]; then unset HEDDLE_PLACE_K5_TOP; else export HEDDLE_PLACE_K5_TOP=$top; fi
  timeout 300 python bench/configs.py --only large --reps 3 2>&1 | grep '^{' | sed "s/^{/{\"top\": $top, /" >> gpurun_out/mg4_large1.jsonl
  for kc in 512 1024 2048; do
    HEDDLE_PLACE_K5_KC=$kc timeout 300 $T --nproc-per-node 4 bench.py --gpus 4 --workload large --steps 3 2>&1 | grep '^{' | sed "s/^{/{\"kc\": $kc, \"top\": $top, /" >> gpurun_out/mg4_large4.jsonl
  done
done
unset HEDDLE_PLACE_K5_TOP
timeout 300 python bench/configs.py --reps 3 > gpurun_out/mg4_configs.jsonl 2>&1
echo done
