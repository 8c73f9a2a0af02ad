#!/bin/bash
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --show-backtrace device python tools/probe_greedy.py slos_day > gpurun_out/sanitizer.txt 2>&1
head -60 gpurun_out/sanitizer.txt
