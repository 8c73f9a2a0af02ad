#!/bin/bash
# Session r02d: brute force over the max_mix = min(n, 7) pool first, then the whole GPU suite.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_brute_force.py -m gpu -q -x > gpurun_out/bf_tests.log 2>&1
echo "bf rc=$?" >> gpurun_out/bf_tests.log
tail -5 gpurun_out/bf_tests.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -5 gpurun_out/gpu_tests.log
