#!/bin/bash
for v in 1 0 1 0; do
  E2E_SPLIT=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-fit --no-mlp --no-c3 2>gpurun_out/e2e_$v.err | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('split $v', round(d['value']), 'e2e', round(d['e2e']['value']), d['process_group'])"
  tail -1 gpurun_out/e2e_$v.err
done
