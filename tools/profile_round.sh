#!/bin/bash
# One GPU measurement round: tests, smoke, bench (JSON), launch lists, ncu full
# captures of K1 (in-decode and full-width), the K1-split and K5 kernels, the
# step kernels and the decoder attention.  Outputs under gpurun_out/;
# summaries go to profiles/<round>/ via tools/collect_profiles.py.
set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 tools/launch_list.sh launches_decode --n-inputs 2000 --decoder-inputs 0
timeout 600 ncu --set full --clock-control none --import-source on -k regex:row_lse_topm -s 1200 -c 1 \
    -o gpurun_out/k1_decode python bench.py --no-cpu-baseline --steps 1 --warmup 3 --e2e-steps 1 --n-inputs 2000 --decoder-inputs 0 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:row_lse_topm -s 3 -c 1 \
    -o gpurun_out/k1_fullwidth python tools/prof_k1.py > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_kernel -s 3 -c 1 -o gpurun_out/k1t_fw python tools/prof_k1.py 6400 42024 5 bf16 --split > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_kernel -s 3 -c 1 -o gpurun_out/k1t_573 python tools/prof_k1.py 573 42024 5 bf16 --split > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:proj_ -s 6 -c 2 -o gpurun_out/k5_1300 python tools/prof_k5.py 1300 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"beam_step|schedule|hash_logits" -s 1200 -c 3 \
    -o gpurun_out/step_kernels python bench.py --no-cpu-baseline --steps 1 --warmup 3 --e2e-steps 1 --n-inputs 2000 --decoder-inputs 0 > /dev/null 2>&1
timeout 600 bash tools/decoder_launches.sh > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:row_attention -s 600 -c 2 \
    -o gpurun_out/dec_attention python tools/decoder_probe.py 300 4 12 > /dev/null 2>&1
ls -la gpurun_out
