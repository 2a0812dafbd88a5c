#!/bin/bash
B="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-fit --no-mlp --no-c3"
$B > gpurun_out/plain_c3b.log 2>&1 || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_render_fwd -s 5 -c 1 -o gpurun_out/fwd_c3_final $B > gpurun_out/ncu_fwd_c3.log 2>&1; echo "ncu rc=$?"
