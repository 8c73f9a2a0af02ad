#!/bin/bash
# ncu --set full of the greedy kernel on the stress workload (n=128), application replay.
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:greedy_kernel -c 1 \
   -o gpurun_out/greedy_gen128 python tools/probe_stress.py 128 8.0 1 > gpurun_out/ncu_gen128.log 2>&1
tail -5 gpurun_out/ncu_gen128.log
ls -la gpurun_out
