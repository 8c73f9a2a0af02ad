"""Timing probe of the product greedy on golden workloads (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import support as S  # noqa: E402
from support import mp  # noqa: E402


def main():
    gold = S.load_golden("greedy.json")
    names = sys.argv[1:] or ["slos_day", "slos_24", "gen24_6.35", "gen24_8.0", "gen24_8.7"]
    for name in names:
        if name not in gold:
            continue
        g = gold[name]
        sv = [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in g["services"]]
        ps = S.profiles() if g["store"] == "fixture" else S.two_model_store()
        t0 = time.perf_counter()
        ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults())
        t1 = time.perf_counter()
        for rep in range(3):
            ctx.reset_stats()
            t2 = time.perf_counter()
            plan = mp.fast_algo(mp.zero_completion(len(sv)), ctx)
            t3 = time.perf_counter()
        st = ctx.stats()
        ok = S.plan_key(plan) == g["plan"]
        ph = " ".join(f"{x:.2f}" for x in st["phase_ms"])
        print(f"{name}: ctx {1e3*(t1-t0):.1f} ms, plan {1e3*(t3-t2):.2f} ms, GPUs {len(plan)} match={ok}, "
              f"steps {st['greedy_steps']} events {st['ext_events']} ext_rows {st['ext_rows']}, kernel "
              f"{st['greedy_ms']:.2f} ms [scan {ph.split()[0]} bar {ph.split()[1]} red {ph.split()[2]} "
              f"decide {ph.split()[3]} ext {ph.split()[4]}], {st['greedy_rows']/max(st['greedy_ms'],1e-9)/1e6:.2f} "
              f"Grows/s (ref {g['ref_wall_s']} s)", flush=True)


if __name__ == "__main__":
    main()
