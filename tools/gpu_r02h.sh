#!/bin/bash
# r02h: K7 top-K dense/by-support A/B in the config-#2 GA; greedy phase split on slos_24 / gen24_8.7.
mkdir -p gpurun_out
out=gpurun_out/r02h.txt; : > $out
for d in 60 0 30 80 100; do
  echo "== MIGPLAN_MCTS_DENSE_PCT=$d" >> $out
  MIGPLAN_MCTS_DENSE_PCT=$d timeout 120 python tools/probe_ga_timers.py 10 3 >> $out 2>&1
done
echo "== greedy phase timers" >> $out
MIGPLAN_PHASE_TIMERS=1 timeout 120 python tools/probe_greedy.py slos_24 gen24_8.7 >> $out 2>&1
echo "== greedy print phases" >> $out
timeout 120 python tools/probe_greedy.py slos_24 gen24_8.7 >> $out 2>&1
cat $out | grep -v "^\[mcts\]" | tail -40
