#!/bin/bash
# tests + A/B of the streaming-scan changes + new top-K + rollouts + bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python tools/probe_stress.py 128 8.0 2 > gpurun_out/stress128.txt 2>&1
MIGPLAN_NO_PREFETCH=1 timeout 300 python tools/probe_stress.py 128 8.0 1 > gpurun_out/stress128_nopf.txt 2>&1
timeout 300 python tools/probe_stress.py 48 7.0 2 > gpurun_out/stress48.txt 2>&1
cat gpurun_out/stress128.txt gpurun_out/stress128_nopf.txt gpurun_out/stress48.txt
timeout 300 python tools/probe_topk.py slos_24 48 > gpurun_out/probe_topk.txt 2>&1; cat gpurun_out/probe_topk.txt
timeout 300 python tools/probe_greedy.py > gpurun_out/probe_greedy.txt 2>&1; cat gpurun_out/probe_greedy.txt
timeout 300 python tools/probe_rollouts.py slos_24 100000 > gpurun_out/probe_roll.txt 2>&1
timeout 600 python tools/probe_rollouts.py gen48_7.0 1000000 >> gpurun_out/probe_roll.txt 2>&1
cat gpurun_out/probe_roll.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ga.json 2> gpurun_out/bench_ga.err; cat gpurun_out/bench_ga.json
