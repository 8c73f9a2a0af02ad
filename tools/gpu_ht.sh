#!/bin/bash
MIGPLAN_HOST_TIMERS=1 timeout 60 python tools/probe_ga_timers.py 10 2 > gpurun_out/ht.txt 2>&1
grep "\[host\]" gpurun_out/ht.txt | tail -30
grep "rep" gpurun_out/ht.txt
