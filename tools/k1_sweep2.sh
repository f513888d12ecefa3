#!/bin/bash
# K1 knob sweep: full width (R=6400) and a typical in-decode step (R=573), bf16, M=5, L2 flushed.
for v in 3 1 0 4 5; do
  for pf in 0 1 2 4; do
    a=$(VS_K1_VARIANT=$v VS_K1_PF=$pf timeout 120 python tools/prof_k1.py 6400 42024 5 2>&1 | tail -1)
    b=$(VS_K1_VARIANT=$v VS_K1_PF=$pf timeout 120 python tools/prof_k1.py 573 42024 5 --noflush 2>&1 | tail -1)
    echo "variant=$v pf=$pf | R=6400: $a | R=573: $b"
  done
done
