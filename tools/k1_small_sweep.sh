#!/bin/bash
# K1 latency regime (in-decode R): L2 bulk-prefetch distance and the smem ring.
for cfg in "VS_K1_PF=0" "VS_K1_PF=1" "VS_K1_PF=2" "VS_K1_PF=4" "VS_K1_PF=8" "VS_K1_VARIANT=4" "VS_K1_VARIANT=4 VS_K1_C0=0.05" "VS_K1_PF=4 VS_K1_C0=0.05"; do
  echo -n "$cfg :: "
  for R in 64 573 1500 6400; do
    echo -n "R=$R $(env $cfg timeout 60 python tools/prof_k1.py $R 42024 5 --legacy | tail -1 | sed 's/.*GB\/s: \([0-9.]*\).*/\1/') | "
  done; echo
done
