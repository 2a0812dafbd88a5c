#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests_kv.log 2>&1
tail -1 gpurun_out/gpu_tests_kv.log
bash variants/ab_sort.sh base prev base prev > gpurun_out/ab_kv.txt 2>&1
cat gpurun_out/ab_kv.txt
