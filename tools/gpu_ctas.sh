#!/bin/bash
# seed greedy (cooperative grid) at fewer CTAs: slos_24 / gen24_8.7 kernel time and plan match per grid size
mkdir -p gpurun_out; out=gpurun_out/ctas.txt; : > $out
L=paper_2109_11067_b200/_native/libmigplan_b200.so
for rep in 1 2; do
for c in 148 96 74 48 32 16; do
  echo "CTAS=$c" >> $out
  MIGPLAN_GREEDY_CTAS=$c timeout 60 python tools/probe_ab_golden.py $L slos_24 3 2>&1 | tail -1 >> $out
  MIGPLAN_GREEDY_CTAS=$c timeout 60 python tools/probe_ab_golden.py $L gen24_8.7 3 2>&1 | tail -1 >> $out
done
echo "cluster16" >> $out
MIGPLAN_GREEDY_CLUSTER=16 timeout 60 python tools/probe_ab_golden.py $L slos_24 3 2>&1 | tail -1 >> $out
done
cat $out
