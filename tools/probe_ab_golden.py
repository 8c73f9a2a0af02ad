"""One fast_algo from zero on a golden workload through a given library build (development aid):
    python tools/probe_ab_golden.py LIB.so WORKLOAD [reps]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import support as S  # noqa: E402
from support import mp  # noqa: E402


def main():
    lib, name = sys.argv[1], sys.argv[2]
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    b = mp.Backend.load(lib)
    g = S.load_golden("greedy.json")[name]
    sv = [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in g["services"]]
    ps = S.profiles() if g["store"] == "fixture" else S.two_model_store()
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=b)
    for _ in range(reps):
        ctx.reset_stats()
        plan = mp.fast_algo(mp.zero_completion(len(sv)), ctx)
        st = ctx.stats()
        print(f"{os.path.basename(lib)} {name}: kernel {st['greedy_ms']:.3f} ms, GPUs {len(plan)} match={S.plan_key(plan) == g['plan']}, "
              f"phase {' '.join(f'{x:.2f}' for x in st['phase_ms'])}", flush=True)


if __name__ == "__main__":
    main()
