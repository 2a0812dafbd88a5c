#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c1_2d or mini or c2_kodak or c3 or more_than or c4 or c5" > gpurun_out/gpu_tests_rts2.log 2>&1
tail -2 gpurun_out/gpu_tests_rts2.log
bash variants/ab_sort.sh base rts1 nrts prev base > gpurun_out/ab_rts2.txt 2>&1
cat gpurun_out/ab_rts2.txt
