#!/bin/bash
# sort-variant comparison (experiment helper; not part of the product)
for v in "$@"; do
  if [ "$v" = "base" ]; then unset WIPES_LIB; else export WIPES_LIB=$PWD/variants/$v.so; fi
  for c in c2 c3; do
    python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-fit > gpurun_out/svar_${v}_${c}.log 2>&1
    tail -1 gpurun_out/svar_${v}_${c}.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
  print('$v $c', round(d['ms_per_step'],4), 'scatter', round(k['radix_scatter'],4), 'hist', round(k.get('radix_hist',0),4), 'dup', round(k['duplicate'],4))
except Exception as e: print('$v $c FAILED', e)"
  done
done
