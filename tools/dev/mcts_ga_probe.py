import sys, os
sys.path.insert(0, 'tests')
import support as S
from support import mp
ps = S.profiles(); sv = S.fixture_services("slos_24", ps)
ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults())
prm = mp.GaParams(seed=24, max_rounds=10, time_budget_s=1e9, population=16, workers=8, slow=mp.MctsParams(budget_iters=48))
for rep in range(3):
    ctx.reset_stats()
    mp.two_phase(sv, ps, mp.PartitionRuleSet.defaults(), prm, ctx=ctx)
    st = ctx.stats()
    print({k: st[k] for k in ('mcts_ms', 'mcts_launches', 'mcts_topk_calls', 'greedy_ms', 'greedy_calls', 'kernel_launches')}, flush=True)
