#!/bin/bash
# ab14: K7 pair top-K: next support row range prefetched in the by-support scan (pf.so, product) vs loaded per support (nopf.so); then the MCTS / GA goldens
# then the MCTS / GA goldens on the product library
mkdir -p gpurun_out; out=gpurun_out/ab14.txt; : > $out
LIBS="tools/ab/nopf.so tools/ab/pf.so" bash tools/dev/mcts_ab2.sh >> $out 2>&1
for lib in tools/ab/nopf.so tools/ab/pf.so; do
  timeout 300 python tools/probe_mcts.py $lib slos_24 48 20 2>&1 | tail -1 >> $out
  timeout 300 python tools/probe_mcts.py $lib gen48_7.0 200 1 2>&1 | tail -1 >> $out
done
timeout 900 python -m pytest tests/test_search.py tests/test_mcts_modes.py tests/test_big_goldens.py tests/test_rollouts.py tests/test_ga_parallel.py -m gpu -q -x >> $out 2>&1
cat $out
