#!/bin/bash
# GPU session: the -m gpu suite (log + junit) and one short default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x ${PYTEST_ARGS} --junitxml=gpurun_out/gpu_junit.xml \
    > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -5 gpurun_out/gpu_tests.log
