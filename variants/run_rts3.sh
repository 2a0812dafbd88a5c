#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c1_2d or mini or c2_kodak or c3 or more_than or c4 or c5 or alpha" > gpurun_out/gpu_tests_rts3.log 2>&1
tail -1 gpurun_out/gpu_tests_rts3.log
bash variants/ab_sort.sh base prev base prev > gpurun_out/ab_rts3.txt 2>&1
cat gpurun_out/ab_rts3.txt
