"""Static-partition baselines (bench.hpp:42-90) and lower_bound (bench.hpp:93-108).

Golden outcomes come from the reference itself (oracle/gen_golden.py baseline): the three
kinds on fixture workloads (gpt2-medium is infeasible on 1/7 and 2/7, so those raise the
reference's PlanningError), generated workloads and two-model random workloads.
"""
import pytest

import support as S
from support import mp

BL = S.load_golden("baseline.json")


def case(name):
    g = BL[name]
    ps = S.profiles() if g["store"] == "fixture" else S.two_model_store()
    sv = [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in g["services"]]
    return g, ps, sv


@pytest.mark.parametrize("name", sorted(BL))
def test_baseline_matches_reference(impl, name):
    g, ps, sv = case(name)
    want = g["outcome"]
    if isinstance(want, str):
        with pytest.raises(mp.PlanningError, match="infeasible on a"):
            mp.baseline(g["kind"], sv, ps, backend=impl)
        return
    dep = mp.baseline(g["kind"], sv, ps, backend=impl)
    assert S.plan_key([x.config for x in dep.gpus]) == want
    assert [x.id for x in dep.gpus] == [f"gpu-{i}" for i in range(len(want))]


def test_baseline_names_and_empty(impl):
    assert mp.BASELINE_NAMES == {0: "A100-7/7", 1: "A100-7x1/7", 2: "A100-MIX"}  # bench.hpp:15-22
    assert mp.baseline("7of7", [], S.profiles(), backend=impl).gpus == []


def test_baselines_bracket_the_optimizer(impl):
    """7/7 dedicates whole GPUs: never fewer than the lower bound (bench.hpp:93-108)."""
    for name in sorted(BL):
        g, ps, sv = case(name)
        if isinstance(g["outcome"], list) and g["kind"] == 0:
            assert len(g["outcome"]) >= mp.lower_bound(sv, ps)
