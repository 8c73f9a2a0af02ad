#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_rollouts.py tests/test_big_goldens.py tests/test_ga_parallel.py tests/test_search.py tests/test_cli.py -m gpu -q -x > gpurun_out/rcheck.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/rcheck.txt; tail -3 gpurun_out/rcheck.txt
timeout 120 python tools/probe_rollouts.py gen48_7.0 1e6
timeout 120 python tools/probe_rollouts.py gen48_7.0 1e5
timeout 120 python tools/probe_rollouts.py slos_24 1024
