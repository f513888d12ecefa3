#!/bin/bash
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for v in 1 0 1 0; do
  echo "VS_PDL=$v :: $(VS_PDL=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --decoder-inputs 1000 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',d['value'],'ms/step',d['ms_per_step'],'K1 GB/s',d['roofline']['achieved'],'share',d['roofline']['share_of_step'],'dec',d['decoder_wmt19']['value'],d['decoder_wmt19']['ms_per_timestep'])")"
done
