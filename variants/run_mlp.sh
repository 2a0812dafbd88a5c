timeout 1500 python -m pytest tests/test_gpu_mlp.py -q -s -p no:cacheprovider -k "parity" > gpurun_out/gpu_tests_mlp.log 2>&1
