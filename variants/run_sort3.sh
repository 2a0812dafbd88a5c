#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c1_2d or mini or c2_kodak or c3 or more_than or c4" > gpurun_out/gpu_tests_sort3.log 2>&1
tail -2 gpurun_out/gpu_tests_sort3.log
bash variants/ab_sort.sh base lbb4 lbb8 lbb32 base > gpurun_out/ab_sort4.txt 2>&1
cat gpurun_out/ab_sort4.txt
