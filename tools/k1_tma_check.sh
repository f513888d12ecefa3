#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "row_topm" > gpurun_out/k1t_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/k1t_tests.log
for ns in 2 3; do
  echo "ns=$ns :: $(VS_K1T_NS=$ns timeout 120 python tools/prof_k1.py 6400 42024 5 2>&1 | tail -1 | sed 's/.*GB/GB/') || $(VS_K1T_NS=$ns timeout 120 python tools/prof_k1.py 573 42024 5 2>&1 | tail -1| sed 's/.*GB/GB/') || nf $(VS_K1T_NS=$ns timeout 120 python tools/prof_k1.py 573 42024 5 bf16 --noflush 2>&1 | tail -1| sed 's/.*GB/GB/')"
done
bash tools/bench_ab.sh
