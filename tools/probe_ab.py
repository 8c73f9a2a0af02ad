"""A/B probe of library variants on one GPU box (development aid):
    python tools/probe_ab.py LIB.so n mu reps
Loads the given build of include/migplan_b200.h (paper_2109_11067_b200/build.py variant) and
times fast_algo on gen_workload(n, mu) like probe_stress.py."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import support as S  # noqa: E402
from support import mp  # noqa: E402


def main():
    lib, n, mu = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    b = mp.Backend.load(lib)
    ps, sv = S.gen(n, mu)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=b)
    for _ in range(reps):
        ctx.reset_stats()
        plan = mp.fast_algo(mp.zero_completion(n), ctx)
        st = ctx.stats()
        gbs = 8 * st["greedy_rows"] / (st["greedy_ms"] * 1e-3) / 1e9
        print(f"{os.path.basename(lib)} n={n}: kernel {st['greedy_ms']:.1f} ms, {gbs:.0f} GB/s, sha {S.plan_sha(plan)}, "
              f"phase {' '.join(f'{x:.1f}' for x in st['phase_ms'])}", flush=True)


if __name__ == "__main__":
    main()
