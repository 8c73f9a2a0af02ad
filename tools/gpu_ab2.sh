#!/bin/bash
# A/B on one box: extension append layout (greedy, n = 128 / 48) and the MCTS walk (slos_24, gen48).
mkdir -p gpurun_out
out=gpurun_out/ab2.txt; rm -f $out
for round in 1 2; do
  for lib in tools/ab/cur.so tools/ab/ext_pieces.so; do
    timeout 120 python tools/probe_ab.py $lib 128 8.0 1 >> $out 2>&1
    timeout 120 python tools/probe_ab.py $lib 48 7.0 2 >> $out 2>&1
  done
  for lib in tools/ab/mcts_old.so tools/ab/cur.so; do
    timeout 120 python tools/probe_mcts.py $lib slos_24 48 20 >> $out 2>&1
    timeout 300 python tools/probe_mcts.py $lib gen48_7.0 200 3 >> $out 2>&1
  done
done
timeout 600 python -m pytest tests/test_greedy.py tests/test_search.py tests/test_big_goldens.py tests/test_shard.py -m gpu -q -x \
    > gpurun_out/ab2_tests.log 2>&1; echo "tests rc=$?" >> $out; tail -2 gpurun_out/ab2_tests.log >> $out
cat $out
