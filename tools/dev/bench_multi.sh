#!/bin/bash
# bench.py's N > 1 path on a 1-GPU box: 2 ranks share cuda:0 over gloo (code-path check only).
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --steps 2 --warmup 1 --workload slos24_greedy --dist-backend gloo \
    > gpurun_out/bench_multi.json 2> gpurun_out/bench_multi.err
echo "rc=$?"; cat gpurun_out/bench_multi.json; tail -5 gpurun_out/bench_multi.err
