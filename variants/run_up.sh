#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c3 or c4 or c5 or c2_kodak or mini" > gpurun_out/gpu_tests_up.log 2>&1
tail -1 gpurun_out/gpu_tests_up.log
bash variants/ab_sort.sh base up1 up2 up8 base > gpurun_out/ab_up.txt 2>&1
cat gpurun_out/ab_up.txt
