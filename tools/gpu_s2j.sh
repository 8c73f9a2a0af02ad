#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -4 gpurun_out/pytest_gpu.txt
for r in 4 0 2 6; do
  MIGPLAN_RING=$r timeout 300 python tools/probe_stress.py 128 8.0 1 > gpurun_out/s128_ring$r.txt 2>&1
  echo "ring=$r: $(tail -1 gpurun_out/s128_ring$r.txt)"
done
MIGPLAN_RING=4 timeout 300 python tools/probe_stress.py 48 7.0 2 2>&1 | tail -1
MIGPLAN_RING=0 timeout 300 python tools/probe_stress.py 48 7.0 2 2>&1 | tail -1
timeout 300 python tools/probe_greedy.py 2>&1
