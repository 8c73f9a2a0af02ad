#!/bin/bash
for d in 60 0 30 100 60 0; do
  echo "== dense pct $d"
  MIGPLAN_ROLLOUT_DENSE_PCT=$d timeout 60 python tools/probe_rollouts.py tools/ab/cur.so gen48_7.0 1e6 | tail -1
  MIGPLAN_ROLLOUT_DENSE_PCT=$d timeout 60 python tools/probe_rollouts.py tools/ab/cur.so gen48_7.0 1e5 | tail -1
  MIGPLAN_ROLLOUT_DENSE_PCT=$d timeout 60 python tools/probe_rollouts.py tools/ab/cur.so slos_24 1024 | tail -1
done
