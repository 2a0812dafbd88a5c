#!/bin/bash
for v in MINB3 MINB3_BWD_PRIM_ONCE0 MINB4 MINB4_BWD_PRIM_ONCE0 MINB3; do
  export WIPES_LIB=$PWD/variants/$v.so
  for c in c3; do
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-fit --no-mlp 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
print('$v $c', round(d['ms_per_step'],4), ' '.join('%s %.4f'%(x,k.get(x,0)) for x in ('preprocess3d','preprocess3d_bwd')))"
  done
done
