#!/bin/bash
# greedy change check: greedy parity tests, the per-step diagnostic and plan timings
mkdir -p gpurun_out
out=gpurun_out/greedy_check.txt; : > $out
timeout 900 python -m pytest tests/test_greedy.py tests/test_greedy_modes.py tests/test_big_goldens.py tests/test_shard.py tests/test_search.py -m gpu -q -x >> $out 2>&1
echo "pytest rc=$?" >> $out
MIGPLAN_PHASE_TIMERS=1 timeout 120 python tools/probe_ab_golden.py tools/ab/diag.so slos_24 > gpurun_out/diag_slos24.txt 2>&1
timeout 120 python tools/probe_greedy.py slos_24 gen24_8.7 >> $out 2>&1
timeout 120 python tools/probe_ga_timers.py 10 3 >> $out 2>&1
timeout 300 python tools/probe_stress.py 128 8.0 1 >> $out 2>&1
tail -12 $out
