#!/bin/bash
timeout 600 python -m pytest tests/test_rollouts.py tests/test_big_goldens.py tests/test_ga_parallel.py -m gpu -q -x 2>&1 | tail -2
for lib in tools/ab/cur.so; do
timeout 120 python tools/probe_rollouts.py $lib gen48_7.0 1e6 | tail -1
timeout 120 python tools/probe_rollouts.py $lib gen48_7.0 1e5 | tail -1
timeout 120 python tools/probe_rollouts.py $lib slos_24 1024 | tail -1
done
timeout 300 python tools/probe_c3.py
bash tools/gpu_cl.sh
