import sys, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import torch
import support as S
from support import mp
import bench
ps = S.profiles(); sv = S.fixture_services("slos_24", ps); R = mp.PartitionRuleSet.defaults()
flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
ctx = mp.make_plan_context(sv, ps, R)
for _ in range(3): bench.run_step(mp, "slos24_ga", ctx, sv, ps, 0, 8)
for i in range(12):
    flush.zero_(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    c2 = mp.make_plan_context(sv, ps, R)
    t1 = time.perf_counter()
    bench.run_step(mp, "slos24_ga", c2, sv, ps, 0, 8)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    c2.close()
    t3 = time.perf_counter()
    print(f"ctx {1e3*(t1-t0):.2f} plan {1e3*(t2-t1):.2f} close {1e3*(t3-t2):.2f}", flush=True)
