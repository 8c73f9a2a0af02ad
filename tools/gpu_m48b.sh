#!/bin/bash
for d in 60 100 30 0; do echo "== dense $d"; MIGPLAN_MCTS_DENSE_PCT=$d timeout 120 python tools/probe_mcts.py gen48_7.0 200 3; done
MIGPLAN_MCTS_TIMERS=1 timeout 120 python tools/probe_mcts.py gen48_7.0 200 1 2>&1 | grep "top-K" | tail -1
