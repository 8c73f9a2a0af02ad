#!/bin/bash
timeout 600 python -m pytest tests/test_rollouts.py tests/test_big_goldens.py tests/test_ga_parallel.py tests/test_search.py -m gpu -q -x 2>&1 | tail -2
MIGPLAN_ROLLOUT_PERSIST=1 timeout 600 python -m pytest tests/test_rollouts.py tests/test_big_goldens.py -k rollout -m gpu -q -x 2>&1 | tail -2
MIGPLAN_ROLLOUT_PERSIST=0 timeout 600 python -m pytest tests/test_rollouts.py tests/test_big_goldens.py -k rollout -m gpu -q -x 2>&1 | tail -2
for lib in tools/ab/cur.so; do
timeout 120 python tools/probe_rollouts.py $lib gen48_7.0 1e6 | tail -1
timeout 120 python tools/probe_rollouts.py $lib gen48_7.0 1e5 | tail -1
timeout 120 python tools/probe_rollouts.py $lib slos_24 1024 | tail -1
MIGPLAN_ROLLOUT_PERSIST=0 timeout 120 python tools/probe_rollouts.py $lib slos_24 1024 | tail -1
timeout 120 python tools/probe_rollouts.py $lib gen48_7.0 16384 | tail -1
MIGPLAN_ROLLOUT_PERSIST=0 timeout 120 python tools/probe_rollouts.py $lib gen48_7.0 16384 | tail -1
done
timeout 300 python tools/probe_c3.py
