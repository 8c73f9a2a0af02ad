"""Parity two_phase probe (development aid): BASELINE config #2 (slos_24, seed 24, P=16, MCTS 48)
with MIGPLAN_MCTS_TIMERS=1 prints each search's phase split to stderr.
    python tools/probe_ga_timers.py [LIB.so] [rounds] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import support as S  # noqa: E402
from support import mp  # noqa: E402


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 and sys.argv[1].endswith(".so") else None
    args = sys.argv[2:] if lib else sys.argv[1:]
    rounds = int(args[0]) if args else 10
    reps = int(args[1]) if len(args) > 1 else 2
    b = mp.Backend.load(lib) if lib else None
    ps = S.profiles()
    sv = S.fixture_services("slos_24", ps)
    rules = mp.PartitionRuleSet.defaults()
    ctx = mp.make_plan_context(sv, ps, rules, backend=b)
    for rep in range(reps):
        ctx.reset_stats()
        t0 = time.perf_counter()
        dep = mp.two_phase(sv, ps, rules, mp.GaParams(seed=24, max_rounds=rounds, time_budget_s=1e9, workers=8),
                           ctx=ctx, backend=b)
        dt = time.perf_counter() - t0
        st = ctx.stats()
        print(f"{os.path.basename(lib or 'product')} rep {rep}: {rounds} rounds {len(dep.gpus)} GPUs in {1e3 * dt:.2f} ms, "
              f"greedy {st['greedy_ms']:.2f} ms / {st['greedy_calls']} calls, mcts {st['mcts_ms']:.2f} ms / "
              f"{st['mcts_launches']} launches, launches {st['kernel_launches']}, greedy phases [scan bar red decide ext] "
              f"{' '.join(f'{x:.2f}' for x in st['phase_ms'])} ms, steps {st['greedy_steps']}, events {st['ext_events']}, "
              f"ext rows {st['ext_rows']}", flush=True)


if __name__ == "__main__":
    main()
