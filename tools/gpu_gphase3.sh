#!/bin/bash
# GA10 greedy phase split (scan / barrier / reduce / decide / extension) for the refill launches
mkdir -p gpurun_out
MIGPLAN_PHASE_TIMERS=1 timeout 120 python tools/probe_ga_timers.py 10 2 > gpurun_out/gphase3.txt 2>&1
timeout 120 python tools/probe_ga_timers.py 10 2 >> gpurun_out/gphase3.txt 2>&1
grep -v "^\[mcts\]" gpurun_out/gphase3.txt | tail -12
