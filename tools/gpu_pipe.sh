#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/pipe.txt
for t in 512 1024; do
  echo "== THREADS=$t PIPE=1" >> gpurun_out/pipe.txt
  MIGPLAN_GREEDY_THREADS=$t MIGPLAN_PIPE=1 MIGPLAN_PHASE_TIMERS=1 timeout 300 python tools/probe_stress.py 128 8.0 2 >> gpurun_out/pipe.txt 2>&1
  MIGPLAN_GREEDY_THREADS=$t MIGPLAN_PIPE=1 timeout 300 python tools/probe_stress.py 48 7.0 2 >> gpurun_out/pipe.txt 2>&1
done
MIGPLAN_GREEDY_THREADS=1024 MIGPLAN_PIPE=1 timeout 900 python -m pytest tests/test_greedy.py tests/test_shard.py tests/test_greedy_modes.py -m gpu -q -x > gpurun_out/pipe_tests.txt 2>&1
tail -3 gpurun_out/pipe_tests.txt >> gpurun_out/pipe.txt
cat gpurun_out/pipe.txt
