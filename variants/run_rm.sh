bash variants/ab.sh base rm0 > gpurun_out/ab_rm.txt 2>&1
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py -q -s -p no:cacheprovider -k "sum or c1_2d or c2_kodak or c5 or row_sharding or fit or exact or sh_colour or chunked or partial" > gpurun_out/gpu_tests_rm.log 2>&1
