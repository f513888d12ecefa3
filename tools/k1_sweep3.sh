#!/bin/bash
for v in 1 0 3; do for pf in 0 2 4 8; do
  for args in "6400 42024 5" "573 42024 5" "6400 42024 5 f32"; do
    echo "variant=$v pf=$pf args=$args :: $(VS_K1_PF=$pf VS_K1_VARIANT=$v python tools/prof_k1.py $args 2>&1 | tail -1 | sed 's/K1 ms per launch: \[[^]]*\]//')"
  done; done; done
