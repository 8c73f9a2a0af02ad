"""Config #3 throughput-mode GA (two_phase_parallel with the rollout refill) timing probe."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import support as S  # noqa: E402
from support import mp  # noqa: E402


def main():
    ps, sv = S.gen(24, 8.7)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults())
    slow = mp.RolloutParams(n_rollouts=1024, topk=10)
    for rounds in (2, 2, 10, 50):
        prm = mp.GaParams(seed=4242, max_rounds=rounds, time_budget_s=1e9, stall_rounds=1 << 30)
        ctx.reset_stats()
        t0 = time.perf_counter()
        dep = mp.two_phase_parallel(sv, ps, mp.PartitionRuleSet.defaults(), prm, ctx=ctx, slow=slow)
        st = ctx.stats()
        print(f"config3 rounds {rounds}: {len(dep.gpus)} GPUs, wall {1e3 * (time.perf_counter() - t0):.1f} ms, greedy "
              f"{st['greedy_ms']:.1f} ms, rollouts {st['rollout_ms']:.1f} ms / {st['rollout_calls']} calls, launches "
              f"{st['kernel_launches']}", flush=True)


if __name__ == "__main__":
    main()
