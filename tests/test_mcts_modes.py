"""The device MCTS search (K7) reproduces the reference's search in every configuration of
its top-K: the on-chip 32-bit pair rows (default for max_mix <= 2), the 64-bit row path
(MIGPLAN_MCTS_PAIR=0) and a search spread over a thread-block cluster with a DSMEM merge
(MIGPLAN_MCTS_CLUSTER=k).  Golden plans and per-iteration traces: tests/golden/mcts.json."""
import pytest

import support as S
from support import mp

MCTS = S.load_golden("mcts.json")
NAMES = sorted(MCTS)[:6]
MODES = [{"MIGPLAN_MCTS_PAIR": "0"}, {"MIGPLAN_MCTS_CLUSTER": "2"}, {"MIGPLAN_MCTS_CLUSTER": "4"},
         {"MIGPLAN_MCTS_CLUSTER": "2", "MIGPLAN_MCTS_PAIR": "0"}]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", MODES, ids=lambda m: ",".join(f"{k[13:]}={v}" for k, v in m.items()))
@pytest.mark.parametrize("name", NAMES)
def test_mcts_modes_match_reference(name, mode, monkeypatch):
    for k, v in mode.items():
        monkeypatch.setenv(k, v)
    g = MCTS[name]
    sv = [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in g["services"]]
    ps = S.profiles() if g["store"] == "fixture" else S.two_model_store()
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=S.product_backend())
    tr = []
    plan = mp.mcts_solve(mp.zero_completion(len(sv)), ctx, mp.MctsParams(budget_iters=g["budget"]), g["seed"],
                         trace=lambda *a: tr.append(list(a)))
    assert S.plan_key(plan) == g["plan"]
    assert tr == g["trace"]
    ctx.close()
