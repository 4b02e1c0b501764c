#!/bin/bash
# K5 diagonal-chunk sweep (HEDDLE_PLACE_K5_KD) on the layered configs, 1 GPU.  Usage: bench/k5kd.sh <tag>
TAG=${1:-k5kd}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "layered or split or tp_sweep or large or context or edge or ragged" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for cfg in tp_sweep paper_6.2 large; do
  for kd in 2048 256 128 64; do
    HEDDLE_PLACE_K5_KD=$kd timeout 300 python bench/configs.py --only $cfg --reps 5 --kernel layered 2>&1 | grep '^{' | sed "s/^{/{\"kd\": $kd, /" >> gpurun_out/${TAG}.jsonl
  done
done
for kc in 1024 4096; do
  for kd in 128; do
    HEDDLE_PLACE_K5_KC=$kc HEDDLE_PLACE_K5_KD=$kd timeout 300 python bench/configs.py --only large --reps 3 --kernel layered 2>&1 | grep '^{' | sed "s/^{/{\"kc\": $kc, \"kd\": $kd, /" >> gpurun_out/${TAG}.jsonl
  done
done
echo done
