#!/bin/bash
# ncu full capture of the C2 render kernels + stall reasons of the backward
python paper_2508_12615_b200/build.py > /dev/null || exit 1
bash variants/prof_render_c2.sh
ncu -i gpurun_out/rend_c2_final.ncu-rep --page details --csv 2>/dev/null | grep -i "k_render_bwd" | grep -iE "stall|warp cycles per issued|Issue Slot|Eligible" | head -60 > gpurun_out/bwd_stalls.csv
ncu -i gpurun_out/rend_c2_final.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/rend_raw.csv
