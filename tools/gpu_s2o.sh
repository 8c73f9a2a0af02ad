#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -4 gpurun_out/pytest_gpu.txt
for pf in 4 2 8; do
  MIGPLAN_PREFETCH=$pf timeout 300 python tools/probe_stress.py 128 8.0 1 > gpurun_out/s128_pf$pf.txt 2>&1
  echo "prefetch=$pf: $(tail -1 gpurun_out/s128_pf$pf.txt)"
done
timeout 300 python tools/probe_stress.py 48 7.0 2 2>&1 | tail -1
timeout 300 python tools/probe_greedy.py 2>&1 | cut -c1-150
