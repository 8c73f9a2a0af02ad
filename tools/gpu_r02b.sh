#!/bin/bash
# MCTS walk A/B, new GA tests, and an application-replay ncu capture of the config #5 greedy kernel.
mkdir -p gpurun_out
out=gpurun_out/r02b.txt; rm -f $out
timeout 600 python -m pytest tests/test_ga_parallel.py tests/test_search.py tests/test_big_goldens.py tests/test_rollouts.py \
    -m gpu -q -x > gpurun_out/r02b_tests.log 2>&1; echo "tests rc=$?" >> $out; tail -3 gpurun_out/r02b_tests.log >> $out
for round in 1 2; do
  for lib in tools/ab/mcts_old.so tools/ab/mcts_new.so; do
    timeout 120 python tools/probe_mcts.py $lib slos_24 48 20 >> $out 2>&1
    timeout 300 python tools/probe_mcts.py $lib gen48_7.0 200 3 >> $out 2>&1
  done
done
timeout 1800 ncu --set full --replay-mode application --clock-control none --import-source on -k regex:greedy_kernel -c 1 \
    -o gpurun_out/greedy_gen128_r02 python tools/probe_stress.py 128 8.0 1 > gpurun_out/ncu_greedy_r02.log 2>&1
echo "ncu rc=$?" >> $out
cat $out
