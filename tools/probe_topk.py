"""Latency probe of the device top-K (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import support as S  # noqa: E402
from support import mp  # noqa: E402


def main():
    ps = S.profiles()
    for name in sys.argv[1:] or ["slos_24"]:
        sv = S.fixture_services(name, ps) if name.startswith("slos") else S.gen(int(name), 7.0)[1]
        ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults())
        rng = mp.Rng(1)
        comps = [[mp.uniform01(rng) for _ in sv] for _ in range(200)]
        for c in comps[:20]:
            mp.topk_candidates(ctx, c, 10)
        ctx.reset_stats()
        t = time.perf_counter()
        for c in comps:
            mp.topk_candidates(ctx, c, 10)
        dt = (time.perf_counter() - t) / len(comps)
        st = ctx.stats()
        print(f"{name}: pool {len(ctx.pool)} rows, python-level {dt*1e6:.1f} us/call, device(event) "
              f"{st['topk_ms']*1e3/len(comps):.1f} us/call", flush=True)


if __name__ == "__main__":
    main()
