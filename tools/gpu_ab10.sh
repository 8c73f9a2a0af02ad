#!/bin/bash
# ab10: which half of the ab9 ptr change hurt: carried thresholds only (ff.so), walking pointer only (ptrw.so), vs HEAD (shift.so)
mkdir -p gpurun_out; out=gpurun_out/ab10.txt; : > $out
for round in 1 2; do
  for lib in tools/ab/shift.so tools/ab/ff.so tools/ab/ptrw.so; do
    timeout 120 python tools/probe_ab.py $lib 128 8.0 2 >> $out 2>&1
    timeout 60 python tools/probe_ab.py $lib 48 7.0 2 >> $out 2>&1
    timeout 60 python tools/probe_ab_golden.py $lib slos_24 2 >> $out 2>&1
    timeout 60 python tools/probe_ab_golden.py $lib gen24_8.7 2 >> $out 2>&1
  done
done
cat $out
