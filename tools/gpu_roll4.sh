#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rollouts.py tests/test_big_goldens.py tests/test_ga_parallel.py tests/test_search.py tests/test_mcts_modes.py -m gpu -q -x > gpurun_out/rcheck.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/rcheck.txt; tail -3 gpurun_out/rcheck.txt
for lib in tools/ab/q4.so tools/ab/cur.so; do
timeout 120 python tools/probe_rollouts.py $lib gen48_7.0 1e6 | tail -1
timeout 120 python tools/probe_rollouts.py $lib gen48_7.0 1e5 | tail -1
timeout 120 python tools/probe_rollouts.py $lib slos_24 1024 | tail -1
done
timeout 120 python tools/probe_ga_timers.py tools/ab/cur.so 10 3
