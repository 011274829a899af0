#!/bin/bash
# A/B of library variants on the exact passes: bash tools/ab.sh N D v1 v2 ...
# (variants/<v>.so; "main" = the in-tree build), interleaved twice.
N=$1; D=$2; shift 2
for rep in 1 2; do for v in "$@"; do
  if [ $v = main ]; then L=; else L=variants/$v.so; fi
  echo "== $v"; ISOC_LIB_PATH=$L timeout 300 python tools/time_passes.py $N $D 2 | grep -E "sigma_pass|omega_mst"
done; done
