"""Where the end-to-end time goes: context build vs the first (cold) and later plans."""
import sys
import time

sys.path.insert(0, "tests")
import support as S  # noqa: E402
from support import mp  # noqa: E402

import bench  # noqa: E402

ps = S.profiles()
sv = S.fixture_services("slos_24", ps)
R = mp.PartitionRuleSet.defaults()
for rep in range(4):
    t0 = time.perf_counter()
    ctx = mp.make_plan_context(sv, ps, R)
    t1 = time.perf_counter()
    mp.two_phase(sv, ps, R, bench.ga_params(0, 8), ctx=ctx)
    t2 = time.perf_counter()
    mp.two_phase(sv, ps, R, bench.ga_params(0, 8), ctx=ctx)
    t3 = time.perf_counter()
    ctx.close()
    t4 = time.perf_counter()
    print(f"ctx {1e3*(t1-t0):.2f} ms, first plan {1e3*(t2-t1):.2f} ms, second {1e3*(t3-t2):.2f} ms, close {1e3*(t4-t3):.2f} ms")
