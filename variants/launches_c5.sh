#!/bin/bash
# C5 launch list (serialised, cold cache; kernel shares, not absolute times)
python paper_2508_12615_b200/build.py > /dev/null || exit 1
timeout 500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-mlp --no-fit > /dev/null 2>&1; echo "ncu c5 rc=$?"
