#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -8 gpurun_out/pytest_gpu.txt
timeout 300 python tools/probe_stress.py 128 8.0 2 > gpurun_out/stress128.txt 2>&1; cat gpurun_out/stress128.txt
timeout 300 python tools/probe_stress.py 48 7.0 2 > gpurun_out/stress48.txt 2>&1; cat gpurun_out/stress48.txt
timeout 300 python tools/probe_greedy.py > gpurun_out/probe_greedy.txt 2>&1; cat gpurun_out/probe_greedy.txt
timeout 300 python tools/probe_topk.py slos_24 48 > gpurun_out/probe_topk.txt 2>&1; cat gpurun_out/probe_topk.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:topk --csv --log-file gpurun_out/topk_launches.csv python tools/probe_topk.py slos_24 48 > /dev/null 2>&1
timeout 300 python tools/probe_shard.py 128 8.0 4 > gpurun_out/probe_shard.txt 2>&1; cat gpurun_out/probe_shard.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ga.json 2> gpurun_out/bench_ga.err; cat gpurun_out/bench_ga.json
