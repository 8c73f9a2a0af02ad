import cProfile, pstats, sys, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import support as S
from support import mp
import bench
ps = S.profiles(); sv = S.fixture_services("slos_24", ps)
ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults())
for _ in range(3): bench.run_step(mp, "slos24_ga", ctx, sv, ps, 0, 8)
pr = cProfile.Profile()
pr.enable()
t = time.perf_counter()
for _ in range(20): bench.run_step(mp, "slos24_ga", ctx, sv, ps, 0, 8)
dt = (time.perf_counter() - t) / 20
pr.disable()
print(f"{dt*1e3:.3f} ms/step (under cProfile)")
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
