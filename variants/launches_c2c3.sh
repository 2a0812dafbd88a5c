#!/bin/bash
# launch list (serialised, cold cache; kernel shares, not absolute times): bash variants/launches_c2c3.sh c2
c=${1:-c2}
python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-mlp --no-fit --no-c3 > gpurun_out/plain_$c.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-mlp --no-fit --no-c3 > /dev/null 2>&1; echo "ncu $c rc=$?"
python profiles/summarize.py launches gpurun_out/launches_$c.csv > gpurun_out/launches_$c.txt; head -30 gpurun_out/launches_$c.txt
