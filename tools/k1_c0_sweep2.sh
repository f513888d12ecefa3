#!/bin/bash
# K1 warps-per-row cost knob (VS_K1_C0) at in-decode-like row counts: back-to-back
# launches (L2-resident rows, no host gaps between launches), and full width (L2 flushed).
for c0 in 0.25 0.5 2 8; do
  line="c0=$c0"
  for R in 1 128 300 573 1000; do
    r=$(VS_K1_C0=$c0 timeout 120 python tools/prof_k1.py $R 42024 5 --b2b 2>&1 | tail -1 | sed 's/.*sorted): \[\([0-9.]*\), \([0-9.]*\), \([0-9.]*\), \([0-9.]*\), \([0-9.]*\), \([0-9.]*\).*GB\/s: \([0-9.]*\).*/\6ms \7GB\/s/')
    line="$line | R=$R: $r"
  done
  echo "$line"
done
