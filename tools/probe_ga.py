"""Throughput-mode GA probe (development aid): device two_phase_parallel vs parity two_phase."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import support as S  # noqa: E402
from support import mp  # noqa: E402


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1].endswith(".so") else None
    args = sys.argv[2:] if lib else sys.argv[1:]
    wl = args[0] if args else "slos_24"
    rounds = int(args[1]) if len(args) > 1 else 10
    b = mp.Backend.load(lib) if lib else None
    if wl.startswith("gen"):
        n, mu = wl[3:].split("_")
        ps, sv = S.gen(int(n), float(mu))
    else:
        ps = S.profiles()
        sv = S.fixture_services(wl, ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=b)
    for rep in range(2):
        for fn in (mp.two_phase_parallel, mp.two_phase):
            ctx.reset_stats()
            t0 = time.perf_counter()
            dep = fn(sv, ps, mp.PartitionRuleSet.defaults(), mp.GaParams(seed=24, max_rounds=rounds, time_budget_s=1e9,
                                                                          workers=8), ctx=ctx, backend=b)
            dt = time.perf_counter() - t0
            st = ctx.stats()
            print(f"{os.path.basename(lib or 'product')} {wl} {fn.__name__}: {rounds} rounds {len(dep.gpus)} GPUs in {1e3*dt:.1f} ms, rows {st['rows_scored']:.3e}"
                  f", greedy {st['greedy_ms']:.1f} ms / {st['greedy_calls']} calls, mcts {st['mcts_ms']:.1f} ms, topk {st['topk_ms']:.1f} ms / "
                  f"{st['topk_calls']} calls, launches {st['kernel_launches']}", flush=True)


if __name__ == "__main__":
    main()
