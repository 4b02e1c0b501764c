#!/bin/bash
# per-rank K5 timelines of the split large instance on N GPUs.  Usage: bench/mgtrace.sh <tag> <N>
TAG=${1:-mgtr}; N=${2:-4}
mkdir -p gpurun_out /tmp/k5tr; rm -f /tmp/k5tr/split.bin*
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29523"
HEDDLE_PLACE_TILE_TRACE=/tmp/k5tr/split.bin timeout 300 $T --nproc-per-node $N bench.py --gpus $N --workload large --steps 1 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1
for r in $(seq 0 $((N-1))); do python bench/tile_trace.py /tmp/k5tr/split.bin.r$r > gpurun_out/${TAG}_r$r.json 2>&1; done
python - <<PY
import sys; sys.path.insert(0, "bench")
import numpy as np, tile_trace as tt
for r in range($N):
    rec = list(tt.records("/tmp/k5tr/split.bin.r%d" % r))[-1]
    t = rec["t"]; print("rank", r, "start", t[:,0].min(), "end", t[:,5].max(), "span_us", (t[:,5].max()-t[:,0].min())/1e3)
PY
echo done
