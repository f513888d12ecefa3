#!/bin/bash
for v in 1 2 3 4 0; do
  for fl in 16 32; do
    for args in "6400 42024 5" "573 42024 5"; do
      echo "variant=$v flush=$fl args=$args :: $(VS_K1_FLUSH=$fl VS_K1_VARIANT=$v python tools/prof_k1.py $args 2>&1 | tail -1 | sed 's/K1 ms per launch: \[[^]]*\]//')"
    done
  done
done
