#!/bin/bash
# per-kernel device time over a window of the WMT-shape decoder decode
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dec_launches.csv \
   -s 20000 -c 3000 python tools/decoder_probe.py 300 4 12 > gpurun_out/dec_launches.log 2>&1
python tools/launch_summary.py gpurun_out/dec_launches.csv | head -40
