#!/bin/bash
for t in 16 32 16 32; do
  for c in c3 c5 c2; do
    timeout 300 python bench.py --config $c --tile $t --steps 5 --warmup 3 --no-cpu-baseline --no-fit --no-mlp --no-c3 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
print('tile $t $c', round(d['ms_per_step'],4), ' '.join('%s %.3f'%(x,v) for x,v in k.items()))"
  done
done
