#!/bin/bash
mkdir -p gpurun_out
for r in 4 2; do
  MIGPLAN_RING=$r timeout 300 python tools/probe_stress.py 128 8.0 1 > gpurun_out/s128_ring$r.txt 2>&1
  echo "ring=$r: $(tail -1 gpurun_out/s128_ring$r.txt)"
done
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json
