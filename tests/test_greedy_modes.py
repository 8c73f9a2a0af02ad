"""The greedy kernel's launch modes all reproduce the reference's plan bit for bit.

`fast_algo` picks a launch mode per context (engine.cu): a cooperative grid over every SM
with the all-reduce argmax (default), one 16-CTA thread-block cluster with a DSMEM argmax
(small working sets), and optionally interleaved unit dealing.  Each mode is forced through
its environment switch (read per call) and checked against the golden traces
(tests/golden/greedy.json, from the reference)."""
import os

import pytest

import support as S
from support import mp

GOLD = S.load_golden("greedy.json")
NAMES = [n for n in ("slos_day", "slos_night", "slos_24", "gen24_6.35") if n in GOLD]
MODES = [{"MIGPLAN_GREEDY_CLUSTER": "0"}, {"MIGPLAN_GREEDY_CLUSTER": "16"}, {"MIGPLAN_GREEDY_CLUSTER": "8"},
         {"MIGPLAN_GREEDY_CLUSTER": "0", "MIGPLAN_INTERLEAVE": "1"},
         {"MIGPLAN_GREEDY_CLUSTER": "16", "MIGPLAN_INTERLEAVE": "1"}]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", MODES, ids=lambda m: ",".join(f"{k[8:]}={v}" for k, v in m.items()))
@pytest.mark.parametrize("name", NAMES)
def test_greedy_modes_match_reference(name, mode, monkeypatch):
    for k, v in mode.items():
        monkeypatch.setenv(k, v)
    g = GOLD[name]
    sv = [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in g["services"]]
    ps = S.profiles() if g["store"] == "fixture" else S.two_model_store()
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=S.product_backend())
    ctx.reset_stats()
    trace = []
    plan = mp.fast_algo(mp.zero_completion(len(sv)), ctx,
                        trace=lambda i, c, s, comp: trace.append([S.fhex(s), S.comp_digest(comp)]))
    assert S.plan_key(plan) == g["plan"]
    assert trace == g["trace"]
    assert ctx.stats()["rows_scored"] == g["rows_scored"]
    ctx.close()
