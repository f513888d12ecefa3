#!/bin/bash
# K1 register-ring depth (variants 3: U3/NB2, 7: U3/NB3, 6: U2/NB4, 8: U2/NB6): back-to-back
# launches at in-decode row counts (default W), and full width (L2 flushed).
for v in 3 7 6 8; do
  line="variant=$v"
  for R in 1 128 573 1000; do
    r=$(VS_K1_VARIANT=$v timeout 120 python tools/prof_k1.py $R 42024 5 --b2b 2>&1 | tail -1 | sed 's/.*sorted): \[\([0-9.]*\), \([0-9.]*\), \([0-9.]*\), \([0-9.]*\), \([0-9.]*\), \([0-9.]*\).*GB\/s: \([0-9.]*\).*/\6ms/')
    line="$line | R=$R: $r"
  done
  r=$(VS_K1_VARIANT=$v timeout 120 python tools/prof_k1.py 6400 42024 5 2>&1 | tail -1 | sed 's/.*GB\/s: \([0-9.]*\).*/\1/')
  echo "$line | R=6400: $r GB/s"
done
