"""Greedy fast algorithm on the B200 vs the reference's golden traces (bit-exact).

Golden vectors: tests/golden/greedy.json, produced by the unmodified reference
(oracle/gen_golden.py).  Pins: plan (configs in pick order), best_score bits and the
completion vector after every step (greedy.hpp:139-140), base pool size
(config_enum.hpp:192-202) and the number of rows the working set held at each step
(the extension semantics of greedy.hpp:107-119).
"""
import pytest

import support as S
from support import mp

pytestmark = pytest.mark.gpu

GOLD = S.load_golden("greedy.json")


def services_of(entry):
    return [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in entry["services"]]


def store_of(entry):
    return S.profiles() if entry["store"] == "fixture" else S.two_model_store()


@pytest.mark.parametrize("name", sorted(GOLD))
def test_greedy_matches_reference(name):
    g = GOLD[name]
    sv, ps = services_of(g), store_of(g)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults())
    assert len(ctx.pool) == g["pool_size"]
    ctx.reset_stats()
    trace = []
    plan = mp.fast_algo(mp.zero_completion(len(sv)), ctx,
                        trace=lambda i, c, s, comp: trace.append([S.fhex(s), S.comp_digest(comp)]))
    assert S.plan_key(plan) == g["plan"]
    assert trace == g["trace"]
    assert ctx.stats()["rows_scored"] == g["rows_scored"]
    final = mp.completion_of(plan, sv, ps)
    assert [S.fhex(c) for c in final] == g["final_comp"]
    assert mp.is_satisfied(final)


def test_greedy_already_satisfied_is_empty():
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 350.0, 100.0)], ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults())
    assert mp.fast_algo([1.0], ctx) == []
    assert mp.fast_algo([2.5], ctx) == []
