#!/bin/bash
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --no-extras > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_e2e.json').read().strip().splitlines()[-1]); e=d['e2e']
print(e['step_ms_rank0']); print(e['kernel_ms_rank0']); print(e['host_ctx_plan_close_ms_rank0']); print(e['cold_ms'])"
