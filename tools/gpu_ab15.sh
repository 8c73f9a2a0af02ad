#!/bin/bash
# ab15: K7 (and the pair top-K) at 256 threads per CTA (t256.so) vs 512 (t512.so, product); plans printed for parity
mkdir -p gpurun_out; out=gpurun_out/ab15.txt; : > $out
LIBS="tools/ab/t512.so tools/ab/t256.so" bash tools/dev/mcts_ab2.sh >> $out 2>&1
for lib in tools/ab/t512.so tools/ab/t256.so; do
  timeout 300 python tools/probe_mcts.py $lib slos_24 48 20 2>&1 | tail -1 >> $out
  timeout 300 python tools/probe_mcts.py $lib gen48_7.0 200 1 2>&1 | tail -1 >> $out
done
cat $out
