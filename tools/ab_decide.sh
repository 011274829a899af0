#!/bin/bash
# decide-kernel variants on the C5 tree: single full sweep + whole tree phase
for v in "" variants/dk_*.so; do
  echo "== ${v:-main}"
  ISOC_LIB_PATH=$v timeout 300 python tools/decide_one.py 50000000 3 2>&1 | grep thr
  ISOC_LIB_PATH=$v timeout 300 python tools/time_tree_phase.py 50000000 2>&1 | tail -2
done
