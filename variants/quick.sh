#!/bin/bash
# quick check: build, render parity tests, C2/C3 bench kernel times (experiment helper)
python paper_2508_12615_b200/build.py > /dev/null || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py -x -q 2>&1 | grep -E "^(FAILED|E |>|tests/|[0-9]+ (passed|failed))|Error|assert" | head -40
for c in "$@"; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-fit --no-mlp > gpurun_out/q_$c.json 2>/dev/null
  tail -1 gpurun_out/q_$c.json | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']
print('$c', round(d['ms_per_step'],4), 'fwd', round(k['render_fwd'],4), 'bwd', round(k['render_bwd'],4), 'frac', round(d['roofline']['frac'],3))"
done
