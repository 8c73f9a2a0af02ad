#!/bin/bash
# round-1c evidence: GPU tests, default bench + reference arm, launch list of one bench step,
# ncu --set full of the MCTS kernel (slos_24 GA) and of the stress greedy kernel (n = 128)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; head -c 400 gpurun_out/bench_default.json; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; head -c 300 gpurun_out/bench_ref.json; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_ga.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extras > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mcts_kernel -c 1 -o gpurun_out/mcts_r01c \
    python tools/probe_ga.py slos_24 1 > gpurun_out/ncu_mcts.log 2>&1; tail -1 gpurun_out/ncu_mcts.log
timeout 600 ncu --set full --clock-control none -k regex:greedy_kernel -c 1 -o gpurun_out/greedy_slos24_r01c \
    python tools/probe_greedy.py slos_24 > gpurun_out/ncu_g24.log 2>&1; tail -1 gpurun_out/ncu_g24.log
ls -la gpurun_out | tail -12
