#!/bin/bash
# A/B of the streaming scan loop on the HBM-bound config #5 (and n = 48)
mkdir -p gpurun_out; out=gpurun_out/ab5.txt; : > $out
for round in 1 2 3; do
  for lib in ${AB_LIBS:-tools/ab/base.so tools/ab/cur.so}; do
    timeout 120 python tools/probe_ab.py $lib 128 8.0 1 >> $out 2>&1
    timeout 60 python tools/probe_ab.py $lib 48 7.0 2 >> $out 2>&1
  done
done
cat $out
