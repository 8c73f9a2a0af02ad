#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
for v in "0 4" "1 4" "2 4" "1 8" "1 2" "1 0"; do set -- $v
  MIGPLAN_LOAD_MODE=$1 MIGPLAN_PREFETCH=$2 timeout 300 python tools/probe_stress.py 128 8.0 1 > gpurun_out/s128_$1_$2.txt 2>&1
  echo "load_mode=$1 prefetch=$2: $(tail -1 gpurun_out/s128_$1_$2.txt)"
done
timeout 300 python tools/probe_topk.py slos_24 48 > gpurun_out/probe_topk.txt 2>&1; cat gpurun_out/probe_topk.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:topk --csv --log-file gpurun_out/topk_launches.csv python tools/probe_topk.py slos_24 48 > /dev/null 2>&1
timeout 300 python tools/probe_rollouts.py slos_24 100000 > gpurun_out/probe_roll.txt 2>&1; cat gpurun_out/probe_roll.txt
