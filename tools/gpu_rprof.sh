#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rollout_advance -s 200 -c 1 -o gpurun_out/roll_adv_r02l python tools/probe_rollouts.py gen48_7.0 1e6 > gpurun_out/ncu_roll.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rollout_build -s 30 -c 1 -o gpurun_out/roll_build_r02l python tools/probe_rollouts.py gen48_7.0 1e6 >> gpurun_out/ncu_roll.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/roll_launches.csv python tools/probe_rollouts.py gen48_7.0 1e6 > /dev/null 2>&1
ls -la gpurun_out
