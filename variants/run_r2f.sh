bash variants/ab.sh base > gpurun_out/ab_pexp.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
