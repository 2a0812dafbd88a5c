bash variants/ab.sh base sr0 > gpurun_out/ab_sr.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -s -p no:cacheprovider -k "c1_2d or tile_size or mini or partial or deterministic or forward_run or counters or c2_kodak or exact or sh_colour" > gpurun_out/gpu_tests_sr.log 2>&1
