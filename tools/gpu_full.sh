#!/bin/bash
# full GPU suite + GA host timeline (MIGPLAN_GA_TIMERS)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
MIGPLAN_GA_TIMERS=1 timeout 60 python tools/probe_ga_timers.py 10 2 > gpurun_out/ga_timeline.txt 2>&1
tail -40 gpurun_out/ga_timeline.txt
