import os, random, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import support as S
from support import mp
ps = S.profiles(); sv = S.fixture_services("slos_24", ps)
b = mp.Backend.load(sys.argv[1]) if len(sys.argv) > 1 else None
ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=b)
plan = mp.fast_algo(mp.zero_completion(len(sv)), ctx)
random.seed(1)
for _ in range(3):
    c = mp.completion_of(random.sample(plan, len(plan) - 9), sv, ps)
    ctx.reset_stats(); mp.fast_algo(c, ctx); print("kernel ms", ctx.stats()["greedy_ms"], flush=True)
