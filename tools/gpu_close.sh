#!/bin/bash
MIGPLAN_HOST_TIMERS=1 timeout 300 python tools/probe_close.py 10 2>&1 | grep -v "greedy batch\|mcts group"
