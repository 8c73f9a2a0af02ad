#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -15 gpurun_out/pytest_gpu.txt
timeout 300 python tools/probe_shard.py 48 7.0 2 > gpurun_out/probe_shard.txt 2>&1
timeout 300 python tools/probe_shard.py 128 8.0 2 >> gpurun_out/probe_shard.txt 2>&1; cat gpurun_out/probe_shard.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:topk1 -s 30 -c 1 -o gpurun_out/topk1_s2 \
    python tools/probe_topk.py slos_24 > gpurun_out/ncu_topk.log 2>&1; tail -2 gpurun_out/ncu_topk.log
timeout 300 python tools/probe_rollouts.py slos_24 100000 > gpurun_out/probe_roll.txt 2>&1; cat gpurun_out/probe_roll.txt
