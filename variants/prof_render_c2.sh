#!/bin/bash
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-fit --no-mlp --no-c3"
$B > gpurun_out/plain_c2r.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_render_ -s 8 -c 2 -o gpurun_out/rend_c2_final $B > gpurun_out/ncu_rend_c2.log 2>&1; echo "ncu rc=$?"
python profiles/summarize.py kernel gpurun_out/rend_c2_final.ncu-rep > gpurun_out/render_c2.txt 2>&1; head -5 gpurun_out/render_c2.txt
