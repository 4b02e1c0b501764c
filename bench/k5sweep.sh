#!/bin/bash
# K5 chunk-size sweep (HEDDLE_PLACE_K5_KC x HEDDLE_PLACE_K5_KD) on configs[4], plus tp_sweep traces.  Usage: bench/k5sweep.sh <tag>
TAG=${1:-k5sweep}
mkdir -p gpurun_out /tmp/k5tr
for kd in 0 128; do
  rm -f /tmp/k5tr/tp.bin
  [ "$kd" = 0 ] && unset HEDDLE_PLACE_K5_KD || export HEDDLE_PLACE_K5_KD=$kd
  HEDDLE_PLACE_TILE_TRACE=/tmp/k5tr/tp.bin timeout 300 python bench/configs.py --only tp_sweep --reps 1 --kernel layered > /dev/null 2>&1
  python - <<PY
import sys; sys.path.insert(0, "bench")
import tile_trace as tt
r = list(tt.records("/tmp/k5tr/tp.bin"))[-1]
open("gpurun_out/${TAG}_tp_kd${kd}.bin", "wb").write(open("/tmp/k5tr/tp.bin", "rb").read()[-(48 + 16 * len(r["tiles"]) + 32 * r["ntiles"]):])
PY
done
unset HEDDLE_PLACE_K5_KD
for kc in 2048 4096; do
  for kd in 0 512 256; do
    [ "$kd" = 0 ] && unset HEDDLE_PLACE_K5_KD || export HEDDLE_PLACE_K5_KD=$kd
    HEDDLE_PLACE_K5_KC=$kc timeout 300 python bench/configs.py --only large --reps 3 --kernel layered 2>&1 | grep '^{' | sed "s/^{/{\"kc\": $kc, \"kd\": $kd, /" >> gpurun_out/${TAG}.jsonl
  done
done
echo done
