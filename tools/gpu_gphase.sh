#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_search.py tests/test_big_goldens.py tests/test_ga_parallel.py tests/test_greedy.py -m gpu -q -x > gpurun_out/gcheck.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/gcheck.txt; tail -2 gpurun_out/gcheck.txt
timeout 60 python tools/probe_ga_timers.py 10 3
MIGPLAN_PHASE_TIMERS=1 timeout 60 python tools/probe_ga_timers.py 10 2 2>/dev/null
