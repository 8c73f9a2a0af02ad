#!/bin/bash
# K7 A/B in the GA context: mcts ms per two_phase (slos_24, 10 rounds), 4 alternating reps.
mkdir -p gpurun_out
#timeout 600 python -m pytest tests/test_search.py tests/test_mcts_modes.py tests/test_big_goldens.py -m gpu -q -x 2>&1 | tail -1
for rep in 1 2 3 4; do
for lib in ${LIBS:-tools/ab/*.so}; do
  timeout 300 python tools/probe_ga.py $lib slos_24 10 2>&1 | grep " two_phase:" | tail -1 | grep -o "^[^ ]*\|mcts [0-9.]* ms" | tr "\n" " "; echo
done
done
