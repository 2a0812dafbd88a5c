#!/bin/bash
# binning launch fusion: A/B against the previous library, then the GPU suite
bash variants/ab.sh base old base old > gpurun_out/ab_fuse.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_fuse.log 2>&1
tail -3 gpurun_out/gpu_tests_fuse.log
cat gpurun_out/ab_fuse.txt
