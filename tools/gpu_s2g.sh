#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:topk1 -s 50 -c 1 -o gpurun_out/topk1_s2g \
    python tools/probe_topk.py slos_24 > gpurun_out/ncu_topk.log 2>&1; tail -2 gpurun_out/ncu_topk.log
timeout 600 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section SchedulerStats \
    --section LaunchStats --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,sass__inst_executed_shared_loads,dram__bytes_read.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum \
    --clock-control none --replay-mode application -k regex:greedy_kernel -c 1 -o gpurun_out/greedy_gen128_s2g \
    python tools/probe_stress.py 128 8.0 1 > gpurun_out/ncu_g128.log 2>&1; tail -2 gpurun_out/ncu_g128.log
