#!/bin/bash
# K5 timeline: plain timings, then one traced solve per config, summarised on the box.  Usage: bench/k5trace.sh <tag>
TAG=${1:-k5trace}
mkdir -p gpurun_out /tmp/k5tr
for cfg in tp_sweep large; do
  timeout 300 python bench/configs.py --only $cfg --reps 5 --kernel layered 2>&1 | grep '^{' >> gpurun_out/${TAG}_plain.jsonl
done
for cfg in tp_sweep paper_6.2 large; do
  HEDDLE_PLACE_TILE_TRACE=/tmp/k5tr/$cfg.bin timeout 300 python bench/configs.py --only $cfg --reps 1 --kernel layered > /dev/null 2>&1
  python bench/tile_trace.py /tmp/k5tr/$cfg.bin > gpurun_out/${TAG}_$cfg.json 2>&1
done
cp /tmp/k5tr/tp_sweep.bin gpurun_out/${TAG}_tp_sweep.bin
echo done
