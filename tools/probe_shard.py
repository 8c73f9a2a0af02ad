"""Sharded greedy probe (development aid): P virtual ranks on one GPU vs the unsharded plan."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import support as S  # noqa: E402
from support import mp  # noqa: E402
from paper_2109_11067_b200 import dist as D  # noqa: E402


def main():
    n, mu, P = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3])
    ps, sv = S.gen(n, mu)
    base = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults())
    t0 = time.perf_counter()
    ref = S.plan_key(mp.fast_algo(mp.zero_completion(n), base))
    t1 = time.perf_counter()
    rows = base.stats()["greedy_rows"]
    ctxs = [mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults()) for _ in range(P)]
    D.shard_local(ctxs)
    t2 = time.perf_counter()
    out = [S.plan_key(D.fast_algo_local(ctxs, mp.zero_completion(n)))]
    t3 = time.perf_counter()
    srows = sum(c.stats()["greedy_rows"] for c in ctxs)
    print(f"n={n} mu={mu} P={P}: unsharded {len(ref)} GPUs {1e3*(t1-t0):.1f} ms; sharded plans equal: "
          f"{all(o == ref for o in out)}, {1e3*(t3-t2):.1f} ms, rows {srows} vs {rows} "
          f"(per rank {[c.stats()['greedy_rows'] for c in ctxs]})", flush=True)


if __name__ == "__main__":
    main()
