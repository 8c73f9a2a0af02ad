#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -4 gpurun_out/pytest_gpu.txt
MIGPLAN_GA_TIMERS=1 timeout 600 python tools/probe_ga.py gen24_8.7 3 2>&1 | tail -30
timeout 600 python tools/probe_ga.py slos_24 10 2>&1 | tail -2
timeout 300 python tools/probe_topk.py slos_24 48 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:topk --csv --log-file gpurun_out/topk_launches.csv python tools/probe_topk.py slos_24 48 > /dev/null 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ga.json 2> gpurun_out/bench_ga.err; cat gpurun_out/bench_ga.json
