#!/bin/bash
timeout 900 python -m pytest tests/test_big_goldens.py tests/test_search.py tests/test_mcts_modes.py tests/test_ga_parallel.py tests/test_rollouts.py -m gpu -q -x 2>&1 | tail -2
timeout 120 python tools/probe_mcts.py gen48_7.0 200 3
timeout 120 python tools/probe_mcts.py slos_24 48 10
timeout 60 python tools/probe_ga_timers.py 10 3 | grep rep
timeout 60 python tools/probe_rollouts.py gen48_7.0 1e6 | tail -1
