#!/bin/bash
# C3-only kernel-variant comparison (experiment helper)
for v in "$@"; do
  if [ "$v" = "base" ]; then unset WIPES_LIB; else export WIPES_LIB=$PWD/variants/$v.so; fi
  python bench.py --config c3 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/var_${v}_c3.log 2>&1
  tail -1 gpurun_out/var_${v}_c3.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
print('$v', round(d['value'],2), round(d['ms_per_step'],3), {x: round(y,3) for x,y in k.items() if y > 0.1})"
done
