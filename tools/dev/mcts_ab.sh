#!/bin/bash
# A/B of K7 library variants (tools/ab/*.so): GA context (slos_24, 10 rounds) and from zero.
mkdir -p gpurun_out
for rep in 1 2; do
for lib in ${LIBS:-tools/ab/*.so}; do
  timeout 300 python tools/probe_ga.py $lib slos_24 10 2>&1 | grep " two_phase:" | tail -1
  timeout 300 python tools/probe_mcts.py $lib slos_24 48 5 2>&1 | tail -1
done
done
