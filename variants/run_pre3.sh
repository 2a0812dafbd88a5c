#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "p3d or p6d or c3 or exact or sh or det or chunk" -p no:cacheprovider > gpurun_out/gpu_tests_pre3.log 2>&1
tail -2 gpurun_out/gpu_tests_pre3.log
for v in base prev bm3 base; do
  if [ "$v" = "base" ]; then unset WIPES_LIB; else export WIPES_LIB=$PWD/variants/$v.so; fi
  for c in c3; do
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-fit --no-mlp 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
print('$v $c', round(d['ms_per_step'],4), ' '.join('%s %.4f'%(x,k.get(x,0)) for x in ('preprocess3d','preprocess3d_bwd')))"
  done
done
