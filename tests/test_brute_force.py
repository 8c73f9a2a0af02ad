"""brute_force_optimum (bench.hpp:160-219) — the exhaustive minimum-GPU oracle.

Golden outcomes come from the reference itself (oracle/gen_golden.py brute_force) on the
instances its own tests use (test_bench.cpp:120-160, test_mcts.cpp:108-126,
acceptance.cpp:202-244) plus 4-service workloads.  Every implementation walks the reference's
DFS order (the device search over rows permuted into pool emission order, one thread per
two-pick prefix), so the plan is the reference's first solution and the node-budget guard
trips at exactly the reference's node count.
"""
import pytest

import support as S
from support import mp

BF = S.load_golden("brute_force.json")
RULES = mp.PartitionRuleSet.defaults()


def case(name):
    g = BF[name]
    ps = S.profiles() if g["store"] == "fixture" else S.two_model_store()
    sv = [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in g["services"]]
    return g, ps, sv


@pytest.mark.parametrize("name", sorted(BF))
def test_matches_reference(impl, name):
    g, ps, sv = case(name)
    want = g["outcome"]
    budget = g.get("node_budget", 20_000_000)
    if isinstance(want, str) and want.startswith("error:"):
        with pytest.raises(mp.PlanningError, match=want[len("error:"):][:20]):
            mp.brute_force_optimum(sv, ps, RULES, g["cap"], node_budget=budget, backend=impl)
        return
    dep = mp.brute_force_optimum(sv, ps, RULES, g["cap"], node_budget=budget, backend=impl)
    if want == "none":
        assert dep is None
        return
    assert dep is not None
    got = S.plan_key([x.config for x in dep.gpus])
    assert got == want
    configs = [x.config for x in dep.gpus]
    assert mp.is_satisfied(mp.completion_of(configs, sv, ps))
    mp.validate_deployment(dep, sv, ps, RULES, backend=impl)


def test_empty_workload_is_zero_gpus(impl):  # test_bench.cpp:129-133
    dep = mp.brute_force_optimum([], S.two_model_store(), RULES, 3, backend=impl)
    assert dep is not None and dep.gpus == []


def test_node_budget_guard(impl):  # test_bench.cpp:154-159
    g, ps, sv = case("gen4_7")
    with pytest.raises(mp.PlanningError, match="budget"):
        mp.brute_force_optimum(sv, ps, RULES, g["cap"], node_budget=2000, backend=impl)


def test_never_beaten_by_fast_algo(impl):  # test_bench.cpp:138-152
    for name in sorted(BF):
        g, ps, sv = case(name)
        if not isinstance(g["outcome"], list) or len(sv) > 2:
            continue
        ctx = mp.make_plan_context(sv, ps, RULES, backend=impl)
        fast = mp.fast_algo([0.0] * len(sv), ctx)
        assert len(fast) >= len(g["outcome"])


def test_cap_zero_is_none(impl):
    g, ps, sv = case("bench_single")
    assert mp.brute_force_optimum(sv, ps, RULES, 0, backend=impl) is None


@pytest.mark.gpu
def test_product_rejects_more_than_sixteen_services():
    ps = S.profiles()
    sv = mp.gen_workload(17, True, 2.0, 0.6, 100.0, 7, ps, backend=S.host_backend())
    with pytest.raises(ValueError, match="16"):
        mp.brute_force_optimum(sv, ps, RULES, 3, backend=S.product_backend())


def test_wide_pool_cases_present():
    """n >= 5 instances (5-7-service configs in the max_mix = min(n, 7) pool) are pinned."""
    wide = [k for k, v in BF.items() if len(v["services"]) >= 5]
    assert len(wide) >= 20
    assert any(isinstance(BF[k]["outcome"], list) and "nodes" in BF[k] for k in wide)
    assert any(str(BF[k]["outcome"]).startswith("error:") for k in wide)


@pytest.mark.parametrize("name", sorted(k for k, v in BF.items() if "nodes" in v))
def test_node_budget_is_exact(impl, name):
    """The budget guard trips at exactly the reference's node count (bench.hpp:191-192):
    the golden `nodes` is the smallest budget the reference passes with."""
    g, ps, sv = case(name)
    dep = mp.brute_force_optimum(sv, ps, RULES, g["cap"], node_budget=g["nodes"], backend=impl)
    assert (dep is None) == (g["outcome"] == "none")
    with pytest.raises(mp.PlanningError, match="budget"):
        mp.brute_force_optimum(sv, ps, RULES, g["cap"], node_budget=g["nodes"] - 1, backend=impl)
