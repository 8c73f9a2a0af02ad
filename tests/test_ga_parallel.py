"""Throughput-mode two_phase (mig_two_phase_parallel, ga.cu): device population.

Golden vectors: oracle/gen_golden.py `ga_parallel` — the reference's own GpuConfig /
fast_algo / completion_of / evaluate_chromosome / fitter under the product's Philox draw
rule (include/migplan_b200.h).  Every implementation must reproduce the plan and every
round log (best GPU count, best slack bits, improved flag) exactly.
"""
import pytest

import support as S
from support import mp

GOLD = S.load_golden("ga_parallel.json")


def services_of(entry):
    return [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in entry["services"]]


def store_of(entry):
    return S.profiles() if entry["store"] == "fixture" else S.two_model_store()


@pytest.mark.parametrize("name", sorted(GOLD))
def test_two_phase_parallel_matches_golden(impl, name):
    g = GOLD[name]
    if impl.name != "product" and g["ref_wall_s"] > 5:
        pytest.skip("large workload: checked on the GPU only")
    logs = []
    dep = mp.two_phase_parallel(services_of(g), store_of(g), mp.PartitionRuleSet.defaults(),
                                mp.GaParams(time_budget_s=1e9, **g["params"]),
                                log=lambda l: logs.append([l.round, l.best_gpus, l.best_slack.hex(), l.improved]),
                                backend=impl)
    assert S.plan_key([x.config for x in dep.gpus]) == g["plan"]
    assert logs == g["log"]


def test_two_phase_parallel_zero_budget_is_greedy(impl):
    ps = S.profiles()
    sv = S.fixture_services("slos_night", ps)
    dep = mp.two_phase_parallel(sv, ps, mp.PartitionRuleSet.defaults(), mp.GaParams(seed=1, time_budget_s=0.0),
                                backend=impl)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    greedy = mp.make_deployment(mp.fast_algo(mp.zero_completion(len(sv)), ctx))
    assert S.plan_key([x.config for x in dep.gpus]) == S.plan_key([x.config for x in greedy.gpus])


def test_two_phase_parallel_valid_and_monotone(impl):
    ps, sv = S.random_workload(5, 31)
    logs = []
    dep = mp.two_phase_parallel(sv, ps, mp.PartitionRuleSet.defaults(),
                                mp.GaParams(seed=3, max_rounds=4, time_budget_s=1e9),
                                log=lambda l: logs.append(l), backend=impl)
    plan = [x.config for x in dep.gpus]
    assert mp.is_satisfied(mp.completion_of(plan, sv, ps))
    best = [(l.best_gpus, l.best_slack) for l in logs]
    assert best == sorted(best, reverse=True) or all(a >= b for a, b in zip(best, best[1:]))


# ---- with the throughput mcts_solve refill (mig_two_phase_parallel_mcts, BASELINE config #3)

GOLD_MCTS = S.load_golden("ga_parallel_mcts.json")


@pytest.mark.parametrize("name", sorted(GOLD_MCTS))
def test_two_phase_parallel_mcts_matches_golden(impl, name):
    g = GOLD_MCTS[name]
    if impl.name != "product" and g["ref_wall_s"] > 5:
        pytest.skip("large workload: checked on the GPU only")
    logs = []
    dep = mp.two_phase_parallel(services_of(g), store_of(g), mp.PartitionRuleSet.defaults(),
                                mp.GaParams(time_budget_s=1e9, **g["params"]),
                                log=lambda l: logs.append([l.round, l.best_gpus, l.best_slack.hex(), l.improved]),
                                backend=impl, slow=mp.RolloutParams(**g["slow"]))
    assert S.plan_key([x.config for x in dep.gpus]) == g["plan"]
    assert logs == g["log"]


def test_two_phase_parallel_mcts_never_worse_than_fast_refill(impl):
    """Per child, the rollout refill replaces the greedy refill only when strictly shorter, so
    with the same Philox stream the first round's best can only improve or tie."""
    ps = S.profiles()
    sv = S.fixture_services("slos_day", ps)
    a = mp.two_phase_parallel(sv, ps, mp.PartitionRuleSet.defaults(), mp.GaParams(seed=3, max_rounds=1, time_budget_s=1e9),
                              backend=impl)
    b = mp.two_phase_parallel(sv, ps, mp.PartitionRuleSet.defaults(), mp.GaParams(seed=3, max_rounds=1, time_budget_s=1e9),
                              backend=impl, slow=mp.RolloutParams(n_rollouts=64))
    assert len(b.gpus) <= len(a.gpus)
