#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -12 gpurun_out/pytest_gpu.txt
timeout 600 python tools/probe_ga.py slos_24 10 2>&1
timeout 600 python tools/probe_ga.py gen24_8.7 3 2>&1
