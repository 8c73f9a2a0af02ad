#!/bin/bash
mkdir -p gpurun_out
MIGPLAN_PHASE_TIMERS=1 timeout 60 python tools/probe_ga_timers.py 10 2 2>/dev/null
MIGPLAN_PHASE_TIMERS=1 timeout 60 python tools/probe_ab_golden.py paper_2109_11067_b200/_native/libmigplan_b200.so slos_24 2 2>/dev/null
