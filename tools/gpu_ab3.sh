#!/bin/bash
# A/B tools/ab/base.so (HEAD) vs tools/ab/cur.so (working tree) on one box.
mkdir -p gpurun_out
out=gpurun_out/ab3.txt; : > $out
for round in 1 2; do
  for lib in ${AB_LIBS:-tools/ab/base.so tools/ab/cur.so}; do
    timeout 120 python tools/probe_ab.py $lib 128 8.0 1 >> $out 2>&1
    timeout 60 python tools/probe_ab_golden.py $lib slos_24 3 >> $out 2>&1
    timeout 60 python tools/probe_ab_golden.py $lib gen24_8.7 2 >> $out 2>&1
    timeout 60 python tools/probe_ga_timers.py $lib 10 3 >> $out 2>&1
  done
done
if [ -n "$AB_TIMERS" ]; then
  MIGPLAN_MCTS_TIMERS=1 timeout 60 python tools/probe_ga_timers.py tools/ab/cur.so 10 1 > gpurun_out/ab3_timers.txt 2>&1
fi
cat $out
if [ -n "$AB_SKEW" ]; then
  for d in 60 0; do
    MIGPLAN_MCTS_DENSE_PCT=$d MIGPLAN_MCTS_TIMERS=1 timeout 60 python tools/probe_ga_timers.py tools/ab/skew.so 10 1 2>&1 | grep "top-K" | tail -1 > gpurun_out/ab3_skew_$d.txt
  done
fi
