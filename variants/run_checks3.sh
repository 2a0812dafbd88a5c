#!/bin/bash
# device-assert build (WIPES_CHECKS): every index checked; the whole path and the parity suite
export WIPES_LIB=$PWD/variants/checks.so
timeout 900 python tools/sanitize_run.py 2d 3d next > gpurun_out/checks_sanitize.log 2>&1; echo "exit $?" >> gpurun_out/checks_sanitize.log
timeout 2700 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > gpurun_out/checks_parity.log 2>&1; echo "exit $?" >> gpurun_out/checks_parity.log
for c in c3 c4; do timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-fit --no-mlp --no-c3 > /dev/null 2> gpurun_out/checks_bench_$c.err; echo "bench $c exit $?" >> gpurun_out/checks_parity.log; done
tail -3 gpurun_out/checks_sanitize.log; tail -4 gpurun_out/checks_parity.log
