#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
timeout 60 python tools/probe_rollouts.py gen48_7.0 1e6 | tail -1
timeout 60 python tools/probe_rollouts.py gen48_7.0 1e5 | tail -1
timeout 60 python tools/probe_rollouts.py slos_24 1024 | tail -1
timeout 300 python tools/probe_c3.py
