#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests_rts.log 2>&1
tail -2 gpurun_out/gpu_tests_rts.log
bash variants/ab_sort.sh base prev base prev > gpurun_out/ab_rts.txt 2>&1
cat gpurun_out/ab_rts.txt
