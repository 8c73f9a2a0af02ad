#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_search.py tests/test_mcts_modes.py tests/test_big_goldens.py tests/test_ga_parallel.py tests/test_cli.py tests/test_bridge.py -m gpu -q -x > gpurun_out/mcheck.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/mcheck.txt
tail -2 gpurun_out/mcheck.txt
MIGPLAN_GA_TIMERS=1 timeout 60 python tools/probe_ga_timers.py 10 3 > gpurun_out/ga_timeline.txt 2>&1
grep "rep" gpurun_out/ga_timeline.txt; grep "mcts group" gpurun_out/ga_timeline.txt | tail -10
