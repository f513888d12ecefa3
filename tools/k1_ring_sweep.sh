#!/bin/bash
# K1 warp kernel: register double-buffering (variants 0/1/3) vs shared-memory ring (4/5).
for v in 3 4 5; do
  echo -n "variant=$v bf16 R=6400 :: "; VS_K1_VARIANT=$v timeout 120 python tools/prof_k1.py 6400 42024 5 --legacy | tail -1
  echo -n "variant=$v bf16 R=573 :: "; VS_K1_VARIANT=$v timeout 120 python tools/prof_k1.py 573 42024 5 --legacy | tail -1
  echo -n "variant=$v f32 R=6400 :: "; VS_K1_VARIANT=$v timeout 120 python tools/prof_k1.py 6400 42024 5 f32 --legacy | tail -1
done
