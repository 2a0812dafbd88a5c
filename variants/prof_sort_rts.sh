#!/bin/bash
B="python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-fit --no-mlp --no-c3"
$B > gpurun_out/plain_c3s.log 2>&1 || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_sort_pass|k_sort_up" -s 30 -c 12 -o gpurun_out/sort_rts_c3 $B > gpurun_out/ncu_sort_rts.log 2>&1; echo "ncu rc=$?"
