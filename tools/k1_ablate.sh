#!/bin/bash
# K1 ablation (results of the ablated builds are NOT valid; timing only):
#   NOCAND: no candidate path (and no exact fallback), NOEXP: no exponentials, BOTH.
set -e
cd "$(dirname "$0")/../paper_2010_02164_b200/csrc"
for a in NOCAND NOEXP; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared -Xcompiler -fPIC -I ../../include \
    -DK1_ABL_$a -o ../_lib/abl_$a.so *.cu 2>/dev/null &
done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared -Xcompiler -fPIC -I ../../include \
  -DK1_ABL_NOCAND -DK1_ABL_NOEXP -o ../_lib/abl_BOTH.so *.cu 2>/dev/null
wait
cd ../..
R=${1:-6400}
for l in libvarstream abl_NOCAND abl_NOEXP abl_BOTH; do
  echo -n "$l :: "; VARSTREAM_LIB=paper_2010_02164_b200/_lib/$l.so timeout 100 python tools/prof_k1.py $R 42024 5 --legacy | tail -1
done
rm -f paper_2010_02164_b200/_lib/abl_*.so
