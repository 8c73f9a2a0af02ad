#!/bin/bash
# top-K phase split in the GA context for several dense-scan thresholds
mkdir -p gpurun_out
for pct in 0 60 100; do
  echo "== dense pct $pct"
  MIGPLAN_MCTS_DENSE_PCT=$pct bash tools/dev/mcts_timers.sh > /dev/null 2>&1
  grep "top-K" gpurun_out/mcts_timers.txt | tail -1
  grep solve gpurun_out/mcts_timers.txt | awk '{for(i=1;i<=NF;i++){if($i=="sel")s+=$(i+1);if($i=="expand-host")e+=$(i+1);if($i=="topk")t+=$(i+1);if($i=="rollout-ctl")r+=$(i+1);if($i=="miss-host")m+=$(i+1)};c++} END {printf "GA ctx per search (cycles): sel %d exp %d miss %d topk %d roll %d (n=%d)\n", s/c, e/c, m/c, t/c, r/c, c}'
done
