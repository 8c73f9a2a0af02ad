#!/bin/bash
for c in 16 8 4 16 8 4; do echo "== small cluster $c"; MIGPLAN_GREEDY_CLUSTER_SMALL=$c timeout 60 python tools/probe_ga_timers.py tools/ab/cur.so 10 3 | tail -1; done
