#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests_sort2.log 2>&1
tail -2 gpurun_out/gpu_tests_sort2.log
bash variants/ab_sort.sh base rank0 lb8 fuse base > gpurun_out/ab_sort3.txt 2>&1
cat gpurun_out/ab_sort3.txt
