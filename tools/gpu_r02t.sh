#!/bin/bash
# r02t: the shift-formed Wf offsets — ncu --set full of the config-#5 greedy kernel, bench + reference arm, launch list
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:greedy_kernel -c 1 -o gpurun_out/greedy_gen128_r02t \
    python tools/probe_stress.py 128 8.0 1 > gpurun_out/ncu_greedy.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_gen128.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-secondary --no-extras > /dev/null 2>&1
tail -3 gpurun_out/ncu_greedy.log; head -c 600 gpurun_out/bench.json
