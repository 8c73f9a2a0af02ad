"""Stress probe: gen_workload(n, lognormal mu) greedy on the B200 (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import support as S  # noqa: E402
from support import mp  # noqa: E402


def main():
    n, mu = int(sys.argv[1]), float(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    ps, sv = S.gen(n, mu)
    t0 = time.perf_counter()
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults())
    t1 = time.perf_counter()
    print(f"n={n} mu={mu}: ctx {1e3*(t1-t0):.1f} ms, base pool {len(ctx.pool)} rows, LB {mp.lower_bound(sv, ps)}",
          flush=True)
    for r in range(reps):
        ctx.reset_stats()
        t2 = time.perf_counter()
        plan = mp.fast_algo(mp.zero_completion(n), ctx)
        t3 = time.perf_counter()
        st = ctx.stats()
        ok = mp.is_satisfied(mp.completion_of(plan, sv, ps))
        gbs = 8 * st["greedy_rows"] / (st["greedy_ms"] * 1e-3) / 1e9
        print(f"  plan {1e3*(t3-t2):.1f} ms, GPUs {len(plan)} sha {S.plan_sha(plan)} satisfied={ok}, steps {st['greedy_steps']}, events "
              f"{st['ext_events']}, ext rows {st['ext_rows']}, rows scored {st['greedy_rows']:.3e}, kernel "
              f"{st['greedy_ms']:.1f} ms, {st['greedy_rows']/st['greedy_ms']/1e6:.1f} Grows/s, {gbs:.0f} GB/s",
              flush=True)
        if os.environ.get("MIGPLAN_PHASE_TIMERS"):
            print("  phase ms (scan, barrier, reduce+update, maybe_extend, ext enum):",
                  " ".join(f"{x:.1f}" for x in st["phase_ms"]), flush=True)


if __name__ == "__main__":
    main()
