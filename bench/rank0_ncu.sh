#!/bin/bash
# torchrun entry point (--no-python): rank 0 runs under ncu with a small single-pass metric set
# (NVLink bytes sent / received and duration of one K5 launch in split mode), the other ranks run
# plainly.  The peers' spin-waits time out (10 s) rather than hang if ncu ever replays the kernel.
#   torchrun --no-python --nproc-per-node N bench/rank0_ncu.sh <tag> python bench.py --gpus N --workload large ...
tag=$1; shift
if [ "$RANK" = "0" ]; then
  exec ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum --clock-control none \
      -k regex:k5_persistent -s 3 -c 1 --csv --log-file gpurun_out/${tag}_nvlink_r0.csv "$@"
else
  exec "$@"
fi
