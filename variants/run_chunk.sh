timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_abi.py -q -s -p no:cacheprovider -k "chunked or abi or c1_2d or mini" > gpurun_out/gpu_tests_chunk.log 2>&1
