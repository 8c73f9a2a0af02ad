"""Greedy fast algorithm (greedy.hpp) — golden traces and proj/tests/test_greedy.cpp.

Golden vectors (tests/golden/greedy.json) come from the unmodified reference
(oracle/gen_golden.py).  Pins per workload: the plan in pick order, best_score bits and a
digest of the completion vector after every step (greedy.hpp:139-140), the base pool size
and the total rows the working set held over all steps (the extension semantics of
greedy.hpp:107-119; product only — the CPU libraries do not count rows).
"""
import pytest

import support as S
from support import mp

GOLD = S.load_golden("greedy.json")


def services_of(entry):
    return [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in entry["services"]]


def store_of(entry):
    return S.profiles() if entry["store"] == "fixture" else S.two_model_store()


@pytest.mark.parametrize("name", sorted(GOLD))
def test_greedy_matches_reference_trace(impl, name):
    g = GOLD[name]
    if impl.name != "product" and g["ref_wall_s"] > 0.5:
        pytest.skip("large workload: checked on the GPU only")
    sv, ps = services_of(g), store_of(g)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    assert len(ctx.pool) == g["pool_size"]
    ctx.reset_stats()
    trace = []
    plan = mp.fast_algo(mp.zero_completion(len(sv)), ctx,
                        trace=lambda i, c, s, comp: trace.append([S.fhex(s), S.comp_digest(comp)]))
    assert S.plan_key(plan) == g["plan"]
    assert trace == g["trace"]
    if impl.name == "product":
        assert ctx.stats()["rows_scored"] == g["rows_scored"]
    final = mp.completion_of(plan, sv, ps)
    assert [S.fhex(c) for c in final] == g["final_comp"]
    assert mp.is_satisfied(final)


def test_score_examples():  # test_greedy.cpp:8-13
    assert mp.score([0.2, 0.3], [0.5, 1.0]) == pytest.approx(0.10)
    assert mp.score([0.4, 0.1], [1.2, 1.0]) == 0.0
    assert mp.score([0.2, 0.3], [0.0, 0.0]) == pytest.approx(0.5)
    with pytest.raises(mp.PlanningError):
        mp.score([0.2], [0.5, 1.0])


def test_score_zero_once_satisfied(impl):  # test_greedy.cpp:15-26
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 700.0, 100.0), mp.ServiceSpec("b", "nlp-a", 260.0, 100.0),
                               mp.ServiceSpec("c", "cnn-a", 450.0, 100.0)], ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    rng = mp.Rng(3, backend=impl)
    n = len(ctx.pool)
    for _ in range(200):
        idx = mp.pick_index(rng, n)
        comp = [1.0 + mp.uniform01(rng) for _ in range(3)]
        assert mp.score(idx, comp, ctx) == 0.0
        assert mp.score(ctx.pool[idx], comp) == 0.0


def test_score_device_equals_host(impl):
    ps = S.profiles()
    sv = S.fixture_services("slos_day", ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    rng = mp.Rng(9, backend=impl)
    for _ in range(200):
        idx = mp.pick_index(rng, len(ctx.pool))
        comp = [mp.uniform01(rng) * 1.3 for _ in sv]
        assert mp.score(idx, comp, ctx) == mp.score(ctx.pool[idx], comp)


def test_single_sublinear_service_gets_1x7(impl):  # test_greedy.cpp:28-40
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 350.0, 100.0)], ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    res = mp.fast_algo([0.0], ctx)
    assert len(res) == 1 and len(res[0].instances) == 7
    assert all(i.placement.slices == 1 and i.service_id == "a" for i in res[0].instances)


def test_satisfied_returns_empty(impl):  # test_greedy.cpp:42-48
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 350.0, 100.0)], ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    assert mp.fast_algo([1.0], ctx) == [] and mp.fast_algo([2.5], ctx) == []


def test_two_disjoint_services(impl):  # test_greedy.cpp:50-64
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 350.0, 100.0), mp.ServiceSpec("b", "nlp-a", 130.0, 100.0)], ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    res = mp.fast_algo([0.0, 0.0], ctx)
    assert len(res) == 2
    assert all(len({i.service_id for i in c.instances}) == 1 for c in res)
    assert mp.is_satisfied(mp.completion_of(res, sv, ps))


def test_scale_invariance(impl):  # test_greedy.cpp:76-99
    ps = S.two_model_store()

    def run(scale):
        sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 350.0 * scale, 100.0),
                                   mp.ServiceSpec("b", "nlp-a", 130.0 * scale, 100.0),
                                   mp.ServiceSpec("c", "cnn-a", 160.0 * scale, 100.0)], ps)
        ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
        return {tuple(sorted((i.placement.slices, i.service_id) for i in c.instances))
                for c in mp.fast_algo([0.0] * 3, ctx)}

    assert run(1.0) == run(3.0) == run(10.0)


def test_determinism_and_nonzero_start(impl):  # test_greedy.cpp:101-108 + residual starts (GA crossover)
    ps, sv = S.random_workload(6, 12345)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    a = mp.fast_algo([0.0] * 6, ctx)
    assert a == mp.fast_algo([0.0] * 6, ctx)
    chk = S.checker_backend()
    if chk is not None and chk is not impl:
        cctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=chk)
        rng = mp.Rng(5, backend=chk)
        for _ in range(8):
            comp = [mp.uniform01(rng) * 1.2 for _ in sv]
            assert mp.fast_algo(comp, ctx) == mp.fast_algo(comp, cctx)
