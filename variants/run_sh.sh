#!/bin/bash
# SH-variant comparison (experiment helper; not part of the product)
for v in "$@"; do
  if [ "$v" = "base" ]; then unset WIPES_LIB; else export WIPES_LIB=$PWD/variants/$v.so; fi
  python bench.py --config c3 --sh 3 --steps 5 --warmup 3 --no-cpu-baseline --no-fit > gpurun_out/shvar_${v}.log 2>&1
  tail -1 gpurun_out/shvar_${v}.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
print('$v', round(d['ms_per_step'],4), 'pre3d', round(k['preprocess3d'],4), 'pre3d_bwd', round(k['preprocess3d_bwd'],4), 'sh_bwd', round(k.get('sh_bwd',0),4))"
done
