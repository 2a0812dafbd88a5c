#!/bin/bash
for v in base BWD_CHUNKS3 BWD_CHUNKS4 BWD_CHUNKS5 base BWD_CHUNKS3 BWD_CHUNKS5; do
  if [ "$v" = "base" ]; then unset WIPES_LIB; else export WIPES_LIB=$PWD/variants/$v.so; fi
  timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-fit --no-mlp --no-c3 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
print('$v', round(d['ms_per_step'],4), 'bwd', round(k['render_bwd'],4))"
done
