#!/bin/bash
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -4 gpurun_out/pytest_gpu.txt
MIGPLAN_MCTS_TIMERS=1 timeout 600 python tools/probe_ga.py slos_24 2 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 --no-extras > gpurun_out/bench_ga.json 2> gpurun_out/bench_ga.err; cut -c1-700 gpurun_out/bench_ga.json
