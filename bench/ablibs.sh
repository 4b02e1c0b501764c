#!/bin/bash
# A/B/... of library builds on one box with bench.py's default line (interleaved, 2 rounds).
# Usage: bench/ablibs.sh <tag> <lib1.so> <lib2.so> ...
TAG=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
  for lib in "$@"; do
    HEDDLE_PLACE_LIB=$PWD/$lib timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-valley 2>&1 | grep '^{' | sed "s|^{|{\"lib\": \"$lib\", |" >> gpurun_out/${TAG}.jsonl
  done
done
echo done
