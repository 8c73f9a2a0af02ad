#!/bin/bash
# K7 phase split in the headline GA (slos_24 two_phase, 10 rounds, MCTS 48) and from zero.
mkdir -p gpurun_out
bash tools/dev/mcts_timers.sh > /dev/null 2>&1
grep -c "solve" gpurun_out/mcts_timers.txt
timeout 300 python tools/probe_mcts.py slos_24 48 10 > gpurun_out/mcts_probe.txt 2>&1
MIGPLAN_MCTS_TIMERS=1 timeout 300 python tools/probe_mcts.py slos_24 48 3 > gpurun_out/mcts_probe_timers.txt 2>&1
timeout 300 python tools/probe_ga.py slos_24 10 >> gpurun_out/mcts_probe.txt 2>&1
cat gpurun_out/mcts_probe.txt; tail -4 gpurun_out/mcts_probe_timers.txt
