bash variants/ab.sh base bwd0 fwd0 fu1 b56 head > gpurun_out/ab_pack2.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -s -p no:cacheprovider -k "c1_2d or tile_size or mini or partial or deterministic or forward_run" > gpurun_out/gpu_tests_pack.log 2>&1
