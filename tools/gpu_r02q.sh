#!/bin/bash
# r02q: final bench + reference arm; the sharded config-#5 path with 2 ranks sharing the one GPU (gloo: a code-path check)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --steps 2 --warmup 1 --dist-backend gloo --no-extras > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err
head -c 400 gpurun_out/bench.json; echo; head -c 1500 gpurun_out/bench_2rank_gloo.json; tail -3 gpurun_out/bench_2rank_gloo.err
