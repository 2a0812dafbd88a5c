#!/bin/bash
# round-1 close: GPU tests, smoke, C2/C5 bench lines after the adaptive SUM-backward chunk count
python paper_2508_12615_b200/build.py > /dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-mlp --no-fit > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
