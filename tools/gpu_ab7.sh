#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/ab7.txt; : > $out
for round in 1 2; do
  for lib in tools/ab/base.so tools/ab/noinl.so tools/ab/unroll.so; do
    timeout 120 python tools/probe_ab.py $lib 128 8.0 1 >> $out 2>&1
    timeout 60 python tools/probe_ab.py $lib 48 7.0 2 >> $out 2>&1
    timeout 60 python tools/probe_ab_golden.py $lib slos_24 3 >> $out 2>&1
    timeout 60 python tools/probe_ab_golden.py $lib gen24_8.7 2 >> $out 2>&1
  done
done
cat $out
