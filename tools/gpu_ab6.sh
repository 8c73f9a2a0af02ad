#!/bin/bash
mkdir -p gpurun_out; out=gpurun_out/ab6.txt; : > $out
for round in 1 2; do
  for lib in ${AB_LIBS:-tools/ab/cur.so tools/ab/q8.so tools/ab/q8o5.so}; do
    timeout 60 python tools/probe_rollouts.py $lib gen48_7.0 1e6 2>&1 | tail -1 >> $out
    timeout 60 python tools/probe_rollouts.py $lib gen48_7.0 1e5 2>&1 | tail -1 >> $out
    timeout 60 python tools/probe_rollouts.py $lib slos_24 1e5 2>&1 | tail -1 >> $out
  done
done
cat $out
