#!/bin/bash
# ab9: streaming loop with an int trip count + walking pointer + carried thresholds (ptr.so), the same
# with two register sets in turn (ptr2.so), vs HEAD (shift.so)
mkdir -p gpurun_out; out=gpurun_out/ab9.txt; : > $out
for round in 1 2; do
  for lib in tools/ab/shift.so tools/ab/ptr.so tools/ab/ptr2.so; do
    timeout 120 python tools/probe_ab.py $lib 128 8.0 2 >> $out 2>&1
    timeout 60 python tools/probe_ab.py $lib 48 7.0 2 >> $out 2>&1
    timeout 60 python tools/probe_ab_golden.py $lib slos_24 2 >> $out 2>&1
    timeout 60 python tools/probe_ab_golden.py $lib gen24_8.7 2 >> $out 2>&1
  done
done
cat $out
