#!/bin/bash
# r02p: final evidence — full GPU suite, bench + reference arm, GA launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_ga.csv \
    python bench.py --workload slos24_ga10 --steps 1 --warmup 0 --no-cpu-baseline --no-secondary --no-extras > /dev/null 2>&1
tail -2 gpurun_out/gpu_tests.log; head -c 400 gpurun_out/bench.json
