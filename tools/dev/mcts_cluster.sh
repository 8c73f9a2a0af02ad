#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/mcts_cluster.txt; rm -f $out
for c in 1 2 4 8 16; do
  echo "== C=$c" >> $out
  MIGPLAN_MCTS_CLUSTER=$c timeout 300 python tools/probe_ga.py slos_24 10 >> $out 2>&1
  MIGPLAN_MCTS_CLUSTER=$c timeout 300 python tools/probe_mcts.py slos_24 48 10 >> $out 2>&1
done
cat $out
