#!/bin/bash
# K5 timeline: one traced solve per config, summarised on the box (bench/tile_trace.py).
# Usage: bench/k5trace.sh <tag> [configs]
TAG=${1:-k5trace}; CFGS=${2:-"tp_sweep large"}
mkdir -p gpurun_out /tmp/k5tr
for cfg in $CFGS; do
  rm -f /tmp/k5tr/$cfg.bin
  HEDDLE_PLACE_TILE_TRACE=/tmp/k5tr/$cfg.bin timeout 300 python bench/configs.py --only $cfg --reps 1 --kernel layered > /dev/null 2>&1
  python bench/tile_trace.py /tmp/k5tr/$cfg.bin > gpurun_out/${TAG}_$cfg.json 2>&1
done
echo done
