#!/bin/bash
# A/B the library variants in tools/ab/*.so on one box (same clocks, same HBM).
mkdir -p gpurun_out
out=gpurun_out/ab.txt; rm -f $out
for round in 1 2; do
  for cfg in ${AB_CFGS:-"512 1" "512 0" "1024 0"}; do
    set -- $cfg
    for lib in ${AB_LIBS:-tools/ab/*.so}; do
      echo "-- threads=$1 pipe=$2 $(basename $lib)" >> $out
      MIGPLAN_GREEDY_THREADS=$1 MIGPLAN_PIPE=$2 timeout 120 python tools/probe_ab.py $lib ${AB_N:-128} ${AB_MU:-8.0} 1 >> $out 2>&1
    done
  done
done
cat $out
