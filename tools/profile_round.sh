#!/bin/bash
# One GPU measurement round: bench (JSON), launch list, ncu full captures of K1
# (in-decode and full-width).  Outputs under gpurun_out/; summaries are then
# copied into profiles/<round>/ by tools/collect_profiles.py.
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tools/launch_list.sh launches_decode --n-inputs 2000
ncu --set full --clock-control none --import-source on -k regex:row_lse_topm -s 1200 -c 1 \
    -o gpurun_out/k1_decode python bench.py --no-cpu-baseline --steps 1 --warmup 3 --e2e-steps 1 --n-inputs 2000 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:row_lse_topm -s 3 -c 1 \
    -o gpurun_out/k1_fullwidth python tools/prof_k1.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"beam_step|schedule|hash_logits" -s 1200 -c 3 \
    -o gpurun_out/step_kernels python bench.py --no-cpu-baseline --steps 1 --warmup 3 --e2e-steps 1 --n-inputs 2000 > /dev/null 2>&1
ls -la gpurun_out
