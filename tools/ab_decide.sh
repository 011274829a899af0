#!/bin/bash
# decide-kernel variants on the C5 tree: single full sweep + bench decide totals
for v in "" variants/dk_*.so; do
  echo "== ${v:-main}"
  ISOC_LIB_PATH=$v timeout 300 python tools/decide_one.py 50000000 3 2>&1 | grep thr | head -2
  ISOC_LIB_PATH=$v timeout 300 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value']/1e6,1), 'M/s decide', round(d['kernels']['decide']['ms_total'],2), 'ms')"
done
