#!/bin/bash
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_big_goldens.py -k "rollouts_gen48" -m gpu -x -q > gpurun_out/san.txt 2>&1
echo "rc=$?" >> gpurun_out/san.txt
grep -A12 "Invalid\|=========" gpurun_out/san.txt | head -60
