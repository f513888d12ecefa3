timeout 600 python -m pytest tests -m gpu -x -q -k "decoder" 2>&1 | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dec_launches.csv -s 20000 -c 3000 python tools/decoder_probe.py 300 4 12 > gpurun_out/dec_launches.log 2>&1
python tools/launch_summary.py gpurun_out/dec_launches.csv 2>/dev/null | head -4
timeout 600 python tools/decoder_probe.py 600 4 12 2>&1 | grep run1
