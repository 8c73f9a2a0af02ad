#!/bin/bash
# parity tests of the working tree, then the base/cur A/B (tools/gpu_ab3.sh)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_greedy.py tests/test_greedy_modes.py tests/test_big_goldens.py tests/test_shard.py tests/test_search.py tests/test_mcts_modes.py tests/test_ga_parallel.py -m gpu -q -x > gpurun_out/check.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/check.txt
tail -3 gpurun_out/check.txt
bash tools/gpu_ab3.sh > /dev/null 2>&1
grep -v "rep 0\|rep 1" gpurun_out/ab3.txt
