#!/bin/bash
# r02u: the bitonic K-th in K7 — full GPU suite + smoke, bench + reference arm, ncu --set full of one K7 search
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/gpu_tests.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mcts_kernel -c 1 -o gpurun_out/mcts_slos24_r02u \
    python tools/probe_mcts.py slos_24 48 1 > gpurun_out/ncu_mcts.log 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/ncu_mcts.log; head -c 600 gpurun_out/bench.json
