"""Device MCTS (K7) timing probe (development aid):
    python tools/probe_mcts.py [LIB.so] [workload] [budget] [reps]
mcts_solve from zero completion (fast_ref + device search + descent completion); prints the
search kernel's device time per call and the plan length."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import support as S  # noqa: E402
from support import mp  # noqa: E402


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1].endswith(".so") else None
    rest = sys.argv[2:] if lib else sys.argv[1:]
    wl = rest[0] if rest else "slos_24"
    budget = int(rest[1]) if len(rest) > 1 else 48
    reps = int(rest[2]) if len(rest) > 2 else 10
    b = mp.Backend.load(lib) if lib else None
    if wl.startswith("gen"):
        n, mu = wl[3:].split("_")
        ps, sv = S.gen(int(n), float(mu))
    else:
        ps = S.profiles()
        sv = S.fixture_services(wl, ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=b)
    z = mp.zero_completion(len(sv))
    mp.mcts_solve(z, ctx, mp.MctsParams(budget_iters=budget), 1)
    ctx.reset_stats()
    t0 = time.perf_counter()
    lens = []
    for seed in range(1, reps + 1):
        lens.append(len(mp.mcts_solve(z, ctx, mp.MctsParams(budget_iters=budget), seed)))
    wall = (time.perf_counter() - t0) / reps
    st = ctx.stats()
    print(f"{os.path.basename(lib or 'product')} {wl} budget {budget}: mcts kernel {st['mcts_ms'] / reps:.3f} ms/search, "
          f"greedy {st['greedy_ms'] / reps:.3f} ms, wall {1e3 * wall:.2f} ms/call, plans {lens}", flush=True)


if __name__ == "__main__":
    main()
