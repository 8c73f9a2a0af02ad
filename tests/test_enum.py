"""Candidate enumeration (config_enum.hpp) — pool parity and proj/tests/test_rules.cpp:175-235."""
import pytest

import support as S
from support import mp


def pool_set(ctx):
    out = set()
    for c in ctx.pool:
        key = tuple((i.placement.slices, i.placement.start_slot, i.service_id, i.batch) for i in c.config.instances)
        out.add((key, tuple((k, v.hex()) for k, v in c.util), c.util_sum.hex()))
    return out


CASES = [("slos_day", None), ("slos_24", None), ("two_n12", 12), ("two_n5", 5)]


@pytest.mark.parametrize("name,n", CASES)
@pytest.mark.parametrize("max_mix", [1, 2, 3])
def test_pool_is_the_reference_pool(impl, name, n, max_mix):
    """Same candidate SET (configs, utility bits, util_sum bits) as the checker."""
    chk = S.checker_backend()
    if chk is None or chk is impl:
        pytest.skip("needs a distinct checker library")
    if n is None:
        ps = S.profiles()
        sv = S.fixture_services(name, ps)
    else:
        ps, sv = S.random_workload(n, 7)
    if max_mix == 3 and len(sv) > 12:
        pytest.skip("checker enumeration too slow at this size")
    a = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), max_mix, backend=impl)
    b = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), max_mix, backend=chk)
    assert len(a.pool) == len(b.pool)
    assert pool_set(a) == pool_set(b)
    assert a.pool.best_single_util == b.pool.best_single_util


def enumerate_configs(impl, services, ps, max_mix):
    return [c.config for c in mp.make_plan_context(services, ps, mp.PartitionRuleSet.defaults(), max_mix,
                                                   backend=impl).pool]


def test_one_service_max_mix_1_gives_11(impl):
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 500.0, 100.0)], ps)
    cfgs = enumerate_configs(impl, sv, ps, 1)
    assert len(cfgs) == 11
    ms = {tuple(sorted(i.placement.slices for i in c.instances)) for c in cfgs}
    assert ms == {(1,) * 7, (1, 1, 1, 1, 1, 2), (1, 1, 1, 2, 2), (1, 2, 2, 2), (1, 1, 1, 1, 3), (1, 1, 2, 3),
                  (2, 2, 3), (3, 3), (1, 1, 1, 4), (1, 2, 4), (7,)}


def test_seven_slice_only_service(impl):
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "nlp-a", 100.0, 30.0)], ps)
    cfgs = enumerate_configs(impl, sv, ps, 1)
    assert len(cfgs) == 1 and len(cfgs[0].instances) == 1 and cfgs[0].instances[0].placement.slices == 7


def test_utilities_distinct_within_group(impl):
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 700.0, 100.0), mp.ServiceSpec("b", "nlp-a", 260.0, 100.0),
                               mp.ServiceSpec("c", "cnn-a", 900.0, 100.0)], ps)
    groups = {}
    for c in enumerate_configs(impl, sv, ps, 2):
        key = (tuple(sorted(i.placement.slices for i in c.instances)), tuple(sorted(i.service_id for i in c.instances)))
        u = tuple(mp.utility_of(c, sv, ps))
        assert u not in groups.setdefault(key, set())
        groups[key].add(u)


def test_331_and_43_unreachable(impl):
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 500.0, 100.0), mp.ServiceSpec("b", "nlp-a", 300.0, 100.0)], ps)
    for c in enumerate_configs(impl, sv, ps, 2):
        m = sorted(i.placement.slices for i in c.instances)
        assert m not in ([1, 3, 3], [3, 4])


def test_pool_utilities_match_utility_of(impl):
    """Cached sparse utility == utility_of(config) bitwise (config_enum.hpp:169-176)."""
    ps = S.profiles()
    sv = S.fixture_services("slos_day", ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    assert len(ctx.pool) == 472
    for c in ctx.pool:
        dense = mp.utility_of(c.config, sv, ps)
        assert [(i, u) for i, u in enumerate(dense) if u > 0.0] == c.util
        s = 0.0
        for _, u in c.util:
            s += u
        assert s == c.util_sum
