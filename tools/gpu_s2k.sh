#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:topk1 -s 50 -c 1 -o gpurun_out/topk1_s2k \
    python tools/probe_topk.py slos_24 > gpurun_out/ncu_topk.log 2>&1; tail -1 gpurun_out/ncu_topk.log
