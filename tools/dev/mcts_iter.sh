#!/bin/bash
# K7 iteration: MCTS-related GPU parity tests, then the phase split (GA context + from zero).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_search.py tests/test_mcts_modes.py tests/test_big_goldens.py tests/test_ga_parallel.py \
    -m gpu -q -x > gpurun_out/mcts_tests.log 2>&1
echo "mcts tests rc=$?" >> gpurun_out/mcts_tests.log
tail -3 gpurun_out/mcts_tests.log
bash tools/dev/mcts_split.sh
for pct in ${DENSE_PCTS:-}; do
  echo "== dense pct $pct"; MIGPLAN_MCTS_DENSE_PCT=$pct timeout 300 python tools/probe_ga.py slos_24 10 2>&1 | tail -1
done
grep "top-K" gpurun_out/mcts_timers.txt | tail -1
grep solve gpurun_out/mcts_timers.txt | awk '{for(i=1;i<=NF;i++){if($i=="sel")s+=$(i+1);if($i=="expand-host")e+=$(i+1);if($i=="topk")t+=$(i+1);if($i=="rollout-ctl")r+=$(i+1);if($i=="miss-host")m+=$(i+1)};c++} END {printf "GA ctx per search (cycles): sel %d exp %d miss %d topk %d roll %d (n=%d)\n", s/c, e/c, m/c, t/c, r/c, c}'
