#!/bin/bash
# Session 2 first GPU call: re-establish the state (tests, default bench, stress probes).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,l2_cache_size --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/host.txt
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_ga.json 2> gpurun_out/bench_ga.err
timeout 300 python tools/probe_stress.py 48 7.0 2 > gpurun_out/stress48.txt 2>&1
timeout 600 python tools/probe_stress.py 128 8.0 2 > gpurun_out/stress128.txt 2>&1
cat gpurun_out/stress48.txt gpurun_out/stress128.txt
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none \
    -k regex:greedy_kernel -c 1 --csv --log-file gpurun_out/greedy_gen128_dram.csv python tools/probe_stress.py 128 8.0 1 > /dev/null 2>&1
ls gpurun_out
