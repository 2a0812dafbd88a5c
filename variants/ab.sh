#!/bin/bash
# A/B of library variants on C2/C3/C5 (experiment helper): bash variants/ab.sh base v1 v2 ...
for v in "$@"; do
  if [ "$v" = "base" ]; then unset WIPES_LIB; else export WIPES_LIB=$PWD/variants/$v.so; fi
  for c in ${AB_CFGS:-c2 c3 c5}; do
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-fit --no-mlp 2>/dev/null | tail -1 | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
  print('$v $c', round(d['ms_per_step'],4), 'fwd', round(k['render_fwd'],4), 'bwd', round(k['render_bwd'],4))
except Exception as e: print('$v $c FAILED', e)"
  done
done
