#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
ncu --set full --clock-control none --import-source on -k regex:greedy_kernel -s 1 -c 1 -o gpurun_out/greedy_slos24_r01b \
    python tools/probe_greedy.py slos_24 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:greedy_kernel -s 0 -c 1 -o gpurun_out/greedy_gen48 \
    python tools/probe_stress.py 48 7.0 1 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none \
    -k regex:greedy_kernel -s 0 -c 1 --csv --log-file gpurun_out/greedy_gen128_dram.csv python tools/probe_stress.py 128 8.0 1 > /dev/null 2>&1
python tools/probe_stress.py 128 8.0 2 > gpurun_out/stress128.txt 2>&1
python bench.py --workload gen128_8.0_greedy --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_gen128.json 2>&1
ls gpurun_out
