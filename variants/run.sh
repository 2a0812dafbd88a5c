#!/bin/bash
# kernel-variant comparison (experiment helper; not part of the product)
for v in "$@"; do
  if [ "$v" = "base" ]; then unset WIPES_LIB; else export WIPES_LIB=$PWD/variants/$v.so; fi
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/var_${v}_c2.log 2>&1
  python bench.py --config c3 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/var_${v}_c3.log 2>&1
  for c in c2 c3; do
    tail -1 gpurun_out/var_${v}_${c}.log | python -c "
import json,sys
try:
  d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
  print('$v $c', round(d['value'],2), round(d['ms_per_step'],4), 'fwd', round(k['render_fwd'],4), 'bwd', round(k['render_bwd'],4))
except Exception as e: print('$v $c FAILED', e)"
  done
done
