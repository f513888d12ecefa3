#!/bin/bash
# K1 warp kernel: FMA-pipe exponential pairs per vector (VS_K1_POLY) x variant sweep.
for v in 3 1 0; do for p in 0 1 2; do
  echo -n "variant=$v poly=$p bf16 :: "; VS_K1_VARIANT=$v VS_K1_POLY=$p timeout 120 python tools/prof_k1.py 6400 42024 5 --legacy | tail -1
done; done
for p in 0 1 2; do
  echo -n "poly=$p R=573 :: "; VS_K1_POLY=$p timeout 120 python tools/prof_k1.py 573 42024 5 --legacy | tail -1
  echo -n "poly=$p f32 :: "; VS_K1_POLY=$p timeout 120 python tools/prof_k1.py 6400 42024 5 f32 --legacy | tail -1
done
