#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "p3d or c3_full or views" > gpurun_out/gpu_tests_vg.log 2>&1; tail -1 gpurun_out/gpu_tests_vg.log
WIPES_LIB=$PWD/variants/vg2.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "p3d or c3_full" > gpurun_out/gpu_tests_vg2.log 2>&1; tail -1 gpurun_out/gpu_tests_vg2.log
for v in base vg2 vg4 lm3 base vg2; do
  if [ "$v" = "base" ]; then unset WIPES_LIB; else export WIPES_LIB=$PWD/variants/$v.so; fi
  timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-fit --no-mlp 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
print('$v c3', round(d['ms_per_step'],4), 'pre3d %.4f'%k['preprocess3d'])"
done
