#!/bin/bash
# ab8: Wf byte offsets formed by one shift per row half (shift.so) vs HEAD (base.so); then the GPU suite on the new build
mkdir -p gpurun_out; out=gpurun_out/ab8.txt; : > $out
for round in 1 2; do
  for lib in tools/ab/base.so tools/ab/shift.so; do
    timeout 120 python tools/probe_ab.py $lib 128 8.0 2 >> $out 2>&1
    timeout 60 python tools/probe_ab.py $lib 48 7.0 2 >> $out 2>&1
    timeout 60 python tools/probe_ab_golden.py $lib slos_24 3 >> $out 2>&1
  done
done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
cat $out; tail -2 gpurun_out/gpu_tests.log
