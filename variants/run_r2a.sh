bash variants/ab.sh base nopack head > gpurun_out/ab_pack.txt 2>&1
timeout 600 python tools/diag_grad3d.py > gpurun_out/diag3d_kappa.log 2>&1
timeout 2700 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
