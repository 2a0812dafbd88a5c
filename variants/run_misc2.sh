#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c1_2d or mini or c2_kodak or c3 or alpha or p3d or det" > gpurun_out/gpu_tests_misc2.log 2>&1
tail -1 gpurun_out/gpu_tests_misc2.log
for v in base prev stall base prev stall; do
  if [ "$v" = "base" ]; then unset WIPES_LIB; else export WIPES_LIB=$PWD/variants/$v.so; fi
  for c in c2 c3 c5; do
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-fit --no-mlp 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
print('$v $c', round(d['ms_per_step'],4), ' '.join('%s %.4f'%(x,k.get(x,0)) for x in ('duplicate','render_fwd','render_bwd')))"
  done
done
