#!/bin/bash
# r02o: bench + reference arm, ncu of the lane-per-rollout advance kernel, GA launch list
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rollout_advance -s 200 -c 1 -o gpurun_out/roll_adv_r02o python tools/probe_rollouts.py gen48_7.0 1e6 > gpurun_out/ncu_roll.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_ga.csv \
    python bench.py --workload slos24_ga10 --steps 1 --warmup 0 --no-cpu-baseline --no-secondary --no-extras > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_roll.csv \
    python tools/probe_rollouts.py gen48_7.0 1e6 > /dev/null 2>&1
head -c 600 gpurun_out/bench.json
