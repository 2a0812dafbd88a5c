#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c1_2d or mini or c2_kodak or c3 or c5 or det or exact or partial or chunk" > gpurun_out/gpu_tests_red.log 2>&1
tail -2 gpurun_out/gpu_tests_red.log
bash variants/ab.sh base prev base prev > gpurun_out/ab_red.txt 2>&1
cat gpurun_out/ab_red.txt
