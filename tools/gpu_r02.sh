#!/bin/bash
# Round-2 evidence session: GPU tests, the default bench line (config #5 + secondary + extras),
# the reference arm, the ncu launch list of a bench step and a full capture of the greedy kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x --junitxml=gpurun_out/gpu_junit.xml > gpurun_out/gpu_tests.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
fi
timeout 900 python bench.py ${BENCH_ARGS:---steps 5 --warmup 3} > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference ${BENCH_ARGS:---steps 5 --warmup 3} > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
if [ -z "$SKIP_NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-secondary --no-extras > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:greedy_kernel -c 1 -o gpurun_out/greedy_gen128 \
      python tools/probe_stress.py 128 8.0 1 > gpurun_out/ncu_greedy.log 2>&1
fi
tail -3 gpurun_out/gpu_tests.log; head -c 3000 gpurun_out/bench.json; echo; cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench.err
