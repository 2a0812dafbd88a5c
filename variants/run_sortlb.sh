bash variants/run_sort.sh base > gpurun_out/ab_sortlb.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -s -p no:cacheprovider -k "c1_2d or mini or c2_kodak or full_size_sampled_gradient or more_than" > gpurun_out/gpu_tests_sortlb.log 2>&1
