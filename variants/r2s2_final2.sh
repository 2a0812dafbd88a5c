#!/bin/bash
# session-2 final: GPU suite, smoke, bench lines C2/C3/C5, C2 launch list + render capture
python paper_2508_12615_b200/build.py > /dev/null || exit 1
timeout 2400 python -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "c2 rc=$?"
timeout 900 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --config c5 --no-cpu-baseline --no-mlp --no-fit > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "c5 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-mlp --no-fit --no-c3 > /dev/null 2>&1; echo "ncu c2 rc=$?"
python profiles/summarize.py launches gpurun_out/launches_c2.csv > gpurun_out/launches_c2.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-mlp --no-fit > /dev/null 2>&1; echo "ncu c5 rc=$?"
python profiles/summarize.py launches gpurun_out/launches_c5.csv > gpurun_out/launches_c5.txt 2>&1
bash variants/prof_render_c2.sh
