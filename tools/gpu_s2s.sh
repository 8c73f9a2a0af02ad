#!/bin/bash
MIGPLAN_MCTS_TIMERS=1 timeout 600 python tools/probe_ga.py slos_24 2 2>&1 | tail -30
