#!/bin/bash
mkdir -p gpurun_out
# rollout kernel (config #4 scale-down: gen48, 1e5 rollouts), MCTS kernel, GA kernels, greedy slos_24: ncu sections
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rollout_kernel -c 1 -o gpurun_out/rollout_gen48 \
    python tools/probe_rollouts.py gen48_7.0 100000 > gpurun_out/ncu_roll.log 2>&1; tail -1 gpurun_out/ncu_roll.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mcts_kernel -c 1 -o gpurun_out/mcts_slos24 \
    python tools/probe_ga.py slos_24 1 > gpurun_out/ncu_mcts.log 2>&1; tail -1 gpurun_out/ncu_mcts.log
timeout 600 ncu --set full --clock-control none -k regex:ga_ -c 2 -o gpurun_out/ga_slos24 \
    python tools/probe_ga.py slos_24 2 > gpurun_out/ncu_ga.log 2>&1; tail -1 gpurun_out/ncu_ga.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:greedy_kernel -s 1 -c 1 -o gpurun_out/greedy_slos24 \
    python tools/probe_greedy.py slos_24 > gpurun_out/ncu_greedy24.log 2>&1; tail -1 gpurun_out/ncu_greedy24.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_ga.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json
ls -la gpurun_out
