#!/bin/bash
# r02g: K7 phase split in the config-#2 GA (timers), ncu --set full of one GA mcts_kernel launch,
# of the slos_24 seed greedy, and of the config-#5 greedy kernel (current code).
mkdir -p gpurun_out
timeout 300 python tools/probe_ga_timers.py 10 2 > gpurun_out/probe_ga_timers.txt 2>&1
MIGPLAN_MCTS_TIMERS=1 timeout 300 python tools/probe_ga_timers.py 10 1 > gpurun_out/probe_ga_timers_on.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mcts_kernel -s 3 -c 1 -o gpurun_out/mcts_ga_r02g \
    python tools/probe_ga_timers.py 10 1 > gpurun_out/ncu_mcts.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:greedy_kernel -c 1 -o gpurun_out/greedy_slos24_r02g \
    python tools/probe_ga_timers.py 10 1 > gpurun_out/ncu_greedy_slos.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:greedy_kernel -c 1 -o gpurun_out/greedy_gen128_r02g \
    python tools/probe_stress.py 128 8.0 1 > gpurun_out/ncu_greedy.log 2>&1
ls -la gpurun_out; tail -3 gpurun_out/probe_ga_timers.txt
