#!/bin/bash
# K7 change check: MCTS/GA parity tests, then the config-#2 GA timing (plain and with timers).
mkdir -p gpurun_out
out=gpurun_out/mcts_check.txt; : > $out
timeout 900 python -m pytest tests/test_search.py tests/test_mcts_modes.py tests/test_big_goldens.py tests/test_ga_parallel.py tests/test_cli.py -m gpu -q -x >> $out 2>&1
echo "pytest rc=$?" >> $out
timeout 120 python tools/probe_ga_timers.py 10 3 >> $out 2>&1
MIGPLAN_MCTS_TIMERS=1 timeout 120 python tools/probe_ga_timers.py 10 1 > gpurun_out/mcts_check_timers.txt 2>&1
timeout 300 python tools/probe_mcts.py slos_24 48 10 >> $out 2>&1
timeout 300 python tools/probe_mcts.py gen48_7.0 200 3 >> $out 2>&1
tail -12 $out
