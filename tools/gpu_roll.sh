#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/probe_rollouts.py gen48_7.0 1e6
MIGPLAN_ROLLOUT_TIMERS=1 timeout 120 python tools/probe_rollouts.py gen48_7.0 1e6
