#!/bin/bash
timeout 1800 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/gpu_tests_modes.log 2>&1
tail -1 gpurun_out/gpu_tests_modes.log; grep -E "FAIL|Error" gpurun_out/gpu_tests_modes.log | head -5
bash variants/ab_sort.sh base base 2>&1 | tail -6
