#!/bin/bash
# K1 variants x shapes (standalone, L2 flushed)
for v in 0 1; do
  for args in "6400 42024 5" "573 42024 5" "1500 42024 5" "6400 42024 5 f32" "6400 42024 50" "2560 2048 3" "160 1000 3"; do
    echo "variant=$v args=$args :: $(VS_K1_VARIANT=$v python tools/prof_k1.py $args 2>&1 | tail -1)"
  done
done
