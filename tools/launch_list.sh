#!/bin/bash
# ncu launch list (per-kernel device time, cold-cache, serialised) of a short decode.
# usage: tools/launch_list.sh <out-prefix> [bench args...]
out=$1; shift
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${out}.csv \
    -s 2000 -c 400 python bench.py --no-cpu-baseline --steps 1 --warmup 3 --e2e-steps 1 "$@" > gpurun_out/${out}.log 2>&1
