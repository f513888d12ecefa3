#!/bin/bash
# K1 warp kernel: register top-list (VS_K1_TL=1, default) vs buffered candidates, per variant.
for v in 3 1 0; do for t in 1 0; do
  echo -n "variant=$v tl=$t bf16 R=6400 :: "; VS_K1_VARIANT=$v VS_K1_TL=$t timeout 120 python tools/prof_k1.py 6400 42024 5 --legacy | tail -1
done; done
for t in 1 0; do
  echo -n "tl=$t R=573 :: "; VS_K1_TL=$t timeout 120 python tools/prof_k1.py 573 42024 5 --legacy | tail -1
  echo -n "tl=$t f32 :: "; VS_K1_TL=$t timeout 120 python tools/prof_k1.py 6400 42024 5 f32 --legacy | tail -1
  echo -n "tl=$t M=8 :: "; VS_K1_TL=$t timeout 120 python tools/prof_k1.py 6400 42024 8 --legacy | tail -1
done
