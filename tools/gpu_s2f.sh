#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -15 gpurun_out/pytest_gpu.txt
timeout 300 python tools/probe_topk.py slos_24 48 > gpurun_out/probe_topk.txt 2>&1; cat gpurun_out/probe_topk.txt
for r in 8192 16384 65536; do MIGPLAN_TOPK_ROWS_PER_CTA=$r timeout 300 python tools/probe_topk.py slos_24 48 2>&1 | sed "s/^/rows_per_cta=$r /"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:topk --csv --log-file gpurun_out/topk_launches.csv python tools/probe_topk.py slos_24 48 > /dev/null 2>&1
MIGPLAN_CTX_TIMERS=1 timeout 300 python tools/probe_shard.py 48 7.0 2 > gpurun_out/probe_shard.txt 2>&1
timeout 300 python tools/probe_shard.py 128 8.0 2 >> gpurun_out/probe_shard.txt 2>&1; cat gpurun_out/probe_shard.txt
timeout 300 python tools/probe_rollouts.py slos_24 100000 > gpurun_out/probe_roll.txt 2>&1
timeout 300 python tools/probe_rollouts.py gen48_7.0 1000000 >> gpurun_out/probe_roll.txt 2>&1; cat gpurun_out/probe_roll.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ga.json 2> gpurun_out/bench_ga.err; cat gpurun_out/bench_ga.json
