#!/bin/bash
# session re-entry check: build, render parity subset, C2/C3/C5 kernel times, default bench line
bash variants/quick.sh c2 c3 c5
timeout 600 python bench.py > gpurun_out/s2_bench_c2.json 2> gpurun_out/s2_bench_c2.err; echo "c2 rc=$?"; tail -c 600 gpurun_out/s2_bench_c2.json
