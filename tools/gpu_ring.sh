#!/bin/bash
# Streaming-scan variants of the greedy kernel at n = 128 / 48 (MIGPLAN_RING stages per warp).
mkdir -p gpurun_out
for r in 0 2 3 4; do
  echo "== RING=$r" >> gpurun_out/ring.txt
  MIGPLAN_RING=$r timeout 300 python tools/probe_stress.py 128 8.0 2 >> gpurun_out/ring.txt 2>&1
  MIGPLAN_RING=$r timeout 300 python tools/probe_stress.py 48 7.0 3 >> gpurun_out/ring.txt 2>&1
done
cat gpurun_out/ring.txt
