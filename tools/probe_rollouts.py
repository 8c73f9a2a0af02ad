"""Throughput-mode rollouts probe (development aid): root-parallel rollouts on the B200."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import support as S  # noqa: E402
from support import mp  # noqa: E402


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1].endswith(".so") else None
    args = sys.argv[2:] if lib else sys.argv[1:]
    b = mp.Backend.load(lib) if lib else None
    wl = args[0] if args else "slos_24"
    R = int(float(args[1])) if len(args) > 1 else 100000
    if wl.startswith("gen"):
        n, mu = wl[3:].split("_")
        ps, sv = S.gen(int(n), float(mu))
    else:
        ps = S.profiles()
        sv = S.fixture_services(wl, ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=b)
    z = mp.zero_completion(len(sv))
    greedy = mp.fast_algo(z, ctx)
    for rep in range(2):
        ctx.reset_stats()
        t0 = time.perf_counter()
        r = mp.rollouts(z, ctx, mp.RolloutParams(n_rollouts=R, seed=1, max_depth=2 * len(greedy)))
        t1 = time.perf_counter()
        print(f"{os.path.basename(lib or 'product')} {wl}: R={R} greedy {len(greedy)} GPUs, best rollout {r.best_len} (id {r.best_id}), completed "
              f"{r.completed} capped {r.capped}, steps {r.steps:.3e}, keys {r.keys}, rounds {r.rounds}, device "
              f"{r.device_ms:.1f} ms, wall {1e3*(t1-t0):.1f} ms, {r.steps/(r.device_ms*1e-3):.3e} steps/s, "
              f"{R/(r.device_ms*1e-3):.3e} rollouts/s", flush=True)


if __name__ == "__main__":
    main()
