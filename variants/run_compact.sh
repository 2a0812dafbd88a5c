#!/bin/bash
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests_compact.log 2>&1
tail -1 gpurun_out/gpu_tests_compact.log; grep -E "^FAILED|Error" gpurun_out/gpu_tests_compact.log | head -5
for v in base prev base prev; do
  if [ "$v" = "base" ]; then unset WIPES_LIB; else export WIPES_LIB=$PWD/variants/$v.so; fi
  for c in c3 c4; do
    timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-fit --no-mlp 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
print('$v $c', round(d['ms_per_step'],4), ' '.join('%s %.4f'%(x,k.get(x,0)) for x in ('duplicate','radix_hist','radix_scatter','scan_blocks')))"
  done
done
