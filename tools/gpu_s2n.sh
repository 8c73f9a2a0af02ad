#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section SchedulerStats \
    --section ComputeWorkloadAnalysis --section LaunchStats --section Occupancy \
    --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,sass__inst_executed_shared_loads,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum \
    --clock-control none --replay-mode application -k regex:greedy_kernel -c 1 -o gpurun_out/greedy_gen128_s2n \
    python tools/probe_stress.py 128 8.0 1 > gpurun_out/ncu_g128.log 2>&1; tail -2 gpurun_out/ncu_g128.log
