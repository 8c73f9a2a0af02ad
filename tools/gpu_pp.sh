#!/bin/bash
timeout 60 python tools/probe_ga_timers.py tools/ab/phases.so 10 1 > gpurun_out/pp.txt 2>&1
grep "greedy cta0" gpurun_out/pp.txt | head -5
grep "greedy cta0" gpurun_out/pp.txt | awk '{pro+=$4; loop+=$10; epi+=$15; n++} END {print n, "instances: prologue", pro/n, "us, loop", loop/n, "us, epilogue", epi/n, "us"}'
