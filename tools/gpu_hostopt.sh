#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
MIGPLAN_HOST_TIMERS=1 timeout 60 python tools/probe_ga_timers.py 10 2 > gpurun_out/ht.txt 2>&1
grep "\[host\]" gpurun_out/ht.txt | tail -6
timeout 60 python tools/probe_ga_timers.py 10 3 | grep rep
