#!/bin/bash
# K1 time vs warps per row (pinned with VS_K1_C0=-W), back-to-back launches (L2-resident rows).
for W in 1 2 4 8; do
  line="W=$W"
  for R in 1 128 573 1000 2000; do
    r=$(VS_K1_C0=-$W timeout 120 python tools/prof_k1.py $R 42024 5 --b2b 2>&1 | tail -1 | sed 's/.*sorted): \[\([0-9.]*\), \([0-9.]*\), \([0-9.]*\), \([0-9.]*\), \([0-9.]*\), \([0-9.]*\).*GB\/s: \([0-9.]*\).*/\6ms/')
    line="$line | R=$R: $r"
  done
  echo "$line"
done
