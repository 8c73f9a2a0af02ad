#!/bin/bash
# r02m: full GPU suite, sanitizer on the new rollout kernels, default bench + reference arm
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_rollouts.py tests/test_big_goldens.py -k "rollout" -m gpu -x -q > gpurun_out/san_memcheck.txt 2>&1
echo "rc=$?" >> gpurun_out/san_memcheck.txt
timeout 600 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_rollouts.py -k "golden" -m gpu -x -q > gpurun_out/san_racecheck.txt 2>&1
echo "rc=$?" >> gpurun_out/san_racecheck.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/gpu_tests.log; tail -3 gpurun_out/san_memcheck.txt; tail -3 gpurun_out/san_racecheck.txt; head -c 600 gpurun_out/bench.json
