"""Residual greedy latency (the GA's fast_ref / descent calls): slos_24 plan, erase 10%, refill."""
import os, random, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import support as S
from support import mp
ps = S.profiles(); sv = S.fixture_services("slos_24", ps)
ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults())
plan = mp.fast_algo(mp.zero_completion(len(sv)), ctx)
random.seed(1)
for rep in range(6):
    keep = random.sample(plan, len(plan) - 9)
    comp = mp.completion_of(keep, sv, ps)
    ctx.reset_stats()
    t0 = time.perf_counter()
    refill = mp.fast_algo(comp, ctx)
    wall = 1e3 * (time.perf_counter() - t0)
    st = ctx.stats()
    print(f"residual {rep}: {len(refill)} steps, kernel {st['greedy_ms']:.3f} ms ({1e3 * st['greedy_ms'] / max(1, len(refill)):.1f} us/step), "
          f"wall {wall:.3f} ms, rows {st['greedy_rows']}, ext events {st['ext_events']}, phases {[round(x, 3) for x in st['phase_ms']]}", flush=True)
ctx.reset_stats()
t0 = time.perf_counter()
p = mp.fast_algo(mp.zero_completion(len(sv)), ctx)
st = ctx.stats()
print(f"from zero: {len(p)} steps, kernel {st['greedy_ms']:.3f} ms ({1e3 * st['greedy_ms'] / len(p):.1f} us/step), phases {[round(x, 3) for x in st['phase_ms']]}")
