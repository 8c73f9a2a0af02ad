#!/bin/bash
# Profiling session: bench lines (3 workloads), ncu launch list of the bench step,
# ncu --set full on the greedy kernel (gen24_8.7) and the top-K kernel.
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_ga.json 2> gpurun_out/bench_ga.err
python bench.py --workload slos24_greedy --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_greedy.json 2>&1
python bench.py --workload gen24_8.7_greedy --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gen24.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches_ga.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:greedy_kernel -s 1 -c 1 -o gpurun_out/greedy_gen24 \
    python tools/probe_greedy.py gen24_8.7 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:topk1 -s 30 -c 1 -o gpurun_out/topk1 \
    python tools/probe_topk.py slos_24 > /dev/null 2>&1
python tools/probe_topk.py slos_24 48 > gpurun_out/probe_topk.txt 2>&1
python tools/probe_greedy.py > gpurun_out/probe_greedy.txt 2>&1
ls gpurun_out
