#!/bin/bash
# One GPU session: tests, bench lines, ncu launch list + full capture of the greedy kernel.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
python bench.py --steps 5 --warmup 2 > gpurun_out/bench_ga.json 2> gpurun_out/bench_ga.err
python bench.py --workload slos24_greedy --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_greedy.json 2> gpurun_out/bench_greedy.err
python bench.py --workload gen24_8.7_greedy --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_gen24.json 2> gpurun_out/bench_gen24.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_ga.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:greedy_kernel -s 1 -c 1 -o gpurun_out/greedy_slos24 \
    python tools/probe_greedy.py slos_24 > gpurun_out/ncu_greedy.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:topk_kernel -s 5 -c 1 -o gpurun_out/topk_slos24 \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_topk.log 2>&1
ls -la gpurun_out
