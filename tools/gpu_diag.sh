#!/bin/bash
# greedy per-step scan skew (tools/ab/diag.so = MGB_GREEDY_STEP_DIAG) on slos_24 and gen24_8.7
mkdir -p gpurun_out
MIGPLAN_PHASE_TIMERS=1 timeout 120 python tools/probe_ab_golden.py tools/ab/diag.so slos_24 > gpurun_out/diag_slos24.txt 2>&1
MIGPLAN_PHASE_TIMERS=1 timeout 120 python tools/probe_ab_golden.py tools/ab/diag.so gen24_8.7 > gpurun_out/diag_gen24.txt 2>&1
tail -5 gpurun_out/diag_slos24.txt
