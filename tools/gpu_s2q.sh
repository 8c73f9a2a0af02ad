#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -4 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-extras > gpurun_out/bench_ga.json 2> gpurun_out/bench_ga.err; cat gpurun_out/bench_ga.json
