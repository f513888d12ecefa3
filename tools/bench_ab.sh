#!/bin/bash
# In-decode A/B: TMA K1 (default) vs legacy K1, short bench runs (no CPU baseline).
for v in "" "VS_K1_LEGACY=1"; do
  echo "== ${v:-tma}"
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('value',d['value'],'ms/step',d['ms_per_step'],'K1',d['roofline']['achieved'],'GB/s share',d['roofline']['share_of_step'],'bytes/launch',d['roofline']['bytes_per_launch'],'fw',d['roofline_full_width']['achieved'])"
done
