#!/bin/bash
# In-decode K1 evidence (single-batch WMT-shape decode, tools/step_profile.py):
#  0) the kernel list of 60 launches in the profiled decode (sanity);
#  1) a window of 300 K1 launches with time + DRAM + L2 bytes, caches NOT
#     flushed (the decode's own producer->K1 L2 reuse is part of the pipeline);
#  2) one --set full capture of an in-decode K1 launch (source-level stalls).
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --clock-control none --cache-control none -c 60 \
  --metrics gpu__time_duration.sum --csv --log-file gpurun_out/k1_indecode_list.csv \
  python tools/step_profile.py --n-inputs 1000 > gpurun_out/k1_indecode_list.log 2>&1
timeout 900 ncu --profile-from-start off --clock-control none --cache-control none \
  -k regex:row_lse -s 200 -c 300 \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,launch__grid_size \
  --csv --log-file gpurun_out/k1_indecode_window.csv \
  python tools/step_profile.py --n-inputs 1000 > gpurun_out/k1_indecode_window.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --cache-control none --import-source on \
  -k regex:row_lse -s 250 -c 1 -o gpurun_out/k1_indecode_full \
  python tools/step_profile.py --n-inputs 1000 > gpurun_out/k1_indecode_full.log 2>&1
