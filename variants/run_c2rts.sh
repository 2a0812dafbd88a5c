#!/bin/bash
for v in 1024 1 1024 1; do
  WIPES_SORT_RTS_TILES=$v timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-fit --no-mlp --no-c3 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
print('rts_tiles $v', round(d['ms_per_step'],4), ' '.join('%s %.4f'%(x,k.get(x,0)) for x in ('radix_hist','radix_scatter','duplicate')))"
done
for v in 1024 100000; do
  WIPES_SORT_RTS_TILES=$v timeout 300 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-fit --no-mlp --no-c3 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
print('c5 rts_tiles $v', round(d['ms_per_step'],4), ' '.join('%s %.4f'%(x,k.get(x,0)) for x in ('radix_hist','radix_scatter','duplicate')))"
done
