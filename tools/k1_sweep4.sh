#!/bin/bash
for v in 1 3 0; do
  for args in "6400 42024 5" "573 42024 5" "573 42024 5 bf16 --noflush" "1500 42024 5" "6400 42024 5 f32" "6400 42024 50"; do
    echo "variant=$v args=$args :: $(VS_K1_VARIANT=$v python tools/prof_k1.py $args 2>&1 | tail -1 | sed 's/K1 ms per launch: \[[^]]*\]//')"
  done; done
