"""Greedy latency A/B (development aid): python tools/dev/greedy_ab.py LIB.so [...]
slos_24 from zero and 6 residuals (erase 9 GPUs) per library."""
import os, random, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import support as S
from support import mp
ps = S.profiles(); sv = S.fixture_services("slos_24", ps)
for lib in sys.argv[1:]:
    b = mp.Backend.load(lib)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=b)
    plan = mp.fast_algo(mp.zero_completion(len(sv)), ctx)
    random.seed(1)
    res = [mp.completion_of(random.sample(plan, len(plan) - 9), sv, ps) for _ in range(6)]
    for rep in range(3):
        ctx.reset_stats()
        mp.fast_algo(mp.zero_completion(len(sv)), ctx)
        z = ctx.stats()["greedy_ms"]
        ctx.reset_stats()
        for c in res:
            mp.fast_algo(c, ctx)
        r = ctx.stats()["greedy_ms"] / len(res)
        print(f"{os.path.basename(lib)}: from zero {z:.3f} ms, residual {r:.3f} ms/call", flush=True)
