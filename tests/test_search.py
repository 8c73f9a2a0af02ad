"""Top-K, MCTS and GA (mcts.hpp, ga.hpp) — golden vectors + proj/tests/test_mcts.cpp, test_ga.cpp.

Parity mode: the product replays the reference's std::mt19937_64 streams exactly, so under a
matched seed the MCTS/GA plans (and their per-iteration traces / round logs) are identical.
"""
import pytest

import support as S
from support import mp


def services_of(entry):
    return [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in entry["services"]]


def store_of(entry):
    return S.profiles() if entry["store"] == "fixture" else S.two_model_store()


TOPK = S.load_golden("topk.json")
MCTS = S.load_golden("mcts.json")
GA = S.load_golden("ga.json")


# ------------------------------------------------------------------ top-K (mcts.hpp:56-76)

@pytest.mark.parametrize("name", sorted(TOPK))
def test_topk_matches_reference(impl, name):
    g = TOPK[name]
    ctx = mp.make_plan_context(services_of(g), store_of(g), mp.PartitionRuleSet.defaults(), backend=impl)
    index = {tuple(map(tuple, S.plan_key([c.config])[0])): i for i, c in enumerate(ctx.pool)}
    for case in g["cases"]:
        comp = [float.fromhex(x) for x in case["comp"]]
        top = mp.topk_candidates(ctx, comp, case["k"])
        assert S.plan_key([ctx.pool[i].config for i in top]) == case["top"]
        sub = sorted(index[tuple(map(tuple, x))] for x in case["subset"])
        top2 = mp.topk_candidates(ctx, comp, case["k"], sub)
        assert S.plan_key([ctx.pool[i].config for i in top2]) == case["top_subset"]


# ------------------------------------------------------------------ MCTS

@pytest.mark.parametrize("name", sorted(MCTS))
def test_mcts_matches_reference(impl, name):
    g = MCTS[name]
    if impl.name != "product" and len(g["services"]) > 12:
        pytest.skip("large workload: checked on the GPU only")
    ctx = mp.make_plan_context(services_of(g), store_of(g), mp.PartitionRuleSet.defaults(), backend=impl)
    tr = []
    plan = mp.mcts_solve(mp.zero_completion(len(g["services"])), ctx, mp.MctsParams(budget_iters=g["budget"]),
                         g["seed"], trace=lambda *a: tr.append(list(a)))
    assert S.plan_key(plan) == g["plan"]
    assert tr == g["trace"]


def twelve(impl):
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec(f"s{i:02d}", "nlp-a" if i % 3 == 2 else "cnn-a", 200.0 + 40.0 * i, 100.0)
                               for i in range(12)], ps)
    return ps, sv


def test_expand_gives_k_children(impl):  # test_mcts.cpp:25-34
    ps, sv = twelve(impl)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    node = mp.SearchNode([0.0] * 12)
    mp.expand(node, ctx, mp.MctsParams(), mp.Rng(5, backend=impl))
    assert len(node.children) == 10 and node.expanded


def test_expand_all_sampled_is_global_topk(impl):  # test_mcts.cpp:36-52
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 700.0, 100.0), mp.ServiceSpec("b", "nlp-a", 260.0, 100.0),
                               mp.ServiceSpec("c", "cnn-a", 450.0, 100.0)], ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    node = mp.SearchNode([0.0] * 3)
    mp.expand(node, ctx, mp.MctsParams(), mp.Rng(5, backend=impl))
    assert 0 < len(node.children) <= 10
    assert [c for c, _ in node.children] == mp.topk_candidates(ctx, node.comp, 10)


def test_expand_cannot_pad(impl):  # test_mcts.cpp:54-64
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "nlp-a", 100.0, 30.0)], ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    node = mp.SearchNode([0.0])
    mp.expand(node, ctx, mp.MctsParams(), mp.Rng(5, backend=impl))
    assert len(node.children) == 1


def test_expand_same_children_as_checker(impl):
    chk = S.checker_backend()
    if chk is None or chk is impl:
        pytest.skip("needs a distinct checker")
    ps, sv = twelve(impl)
    a = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    b = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=chk)
    ra, rb = mp.Rng(77, backend=impl), mp.Rng(77, backend=chk)
    comp = [0.0] * 12
    for step in range(10):
        na, nb = mp.SearchNode(comp), mp.SearchNode(comp)
        mp.expand(na, a, mp.MctsParams(), ra)
        mp.expand(nb, b, mp.MctsParams(), rb)
        assert [a.pool[c].config for c, _ in na.children] == [b.pool[c].config for c, _ in nb.children]
        comp = na.children[0][1].comp


def test_rollout(impl):  # test_mcts.cpp:66-89
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 140.0, 100.0)], ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    p = mp.MctsParams()
    cache, rng = mp.RolloutCache(backend=impl), mp.Rng(17, backend=impl)
    assert mp.rollout([1.0], ctx, p, cache, rng, 10) == 0 and cache.builds == 0
    for _ in range(20):
        assert mp.rollout([0.0], ctx, p, cache, rng, 10) == 1
    for _ in range(50):
        mp.rollout([0.0], ctx, p, cache, rng, 10)
    assert cache.builds == 1


def test_rollout_same_as_checker(impl):
    chk = S.checker_backend()
    if chk is None or chk is impl:
        pytest.skip("needs a distinct checker")
    ps = S.profiles()
    sv = S.fixture_services("slos_day", ps)
    a = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    b = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=chk)
    ca, cb = mp.RolloutCache(backend=impl), mp.RolloutCache(backend=chk)
    ra, rb = mp.Rng(11, backend=impl), mp.Rng(11, backend=chk)
    for _ in range(30):
        pa, pb = [], []
        sa = mp.rollout([0.0] * 5, a, mp.MctsParams(), ca, ra, 36, pa)
        sb = mp.rollout([0.0] * 5, b, mp.MctsParams(), cb, rb, 36, pb)
        assert sa == sb and [a.pool[i].config for i in pa] == [b.pool[i].config for i in pb]
    assert ca.builds == cb.builds


def test_mcts_satisfied_and_zero_budget(impl):  # test_mcts.cpp:91-106
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 350.0, 100.0)], ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    assert mp.mcts_solve([1.3], ctx, mp.MctsParams(), 1) == []
    ps2, sv2 = S.random_workload(4, 77)
    ctx2 = mp.make_plan_context(sv2, ps2, mp.PartitionRuleSet.defaults(), backend=impl)
    assert mp.mcts_solve([0.0] * 4, ctx2, mp.MctsParams(budget_iters=0), 9) == mp.fast_algo([0.0] * 4, ctx2)


def test_mcts_never_worse_than_fast(impl):  # test_mcts.cpp:128-140
    for seed in range(1, 8):
        ps, sv = S.random_workload(3 + seed % 5, seed * 17)
        ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
        fast = mp.fast_algo([0.0] * len(sv), ctx)
        slow = mp.mcts_solve([0.0] * len(sv), ctx, mp.MctsParams(budget_iters=60), seed)
        assert len(slow) <= len(fast)
        assert mp.is_satisfied(mp.completion_of(slow, sv, ps))


# ------------------------------------------------------------------ GA

@pytest.mark.parametrize("name", sorted(GA))
def test_two_phase_matches_reference(impl, name):
    g = GA[name]
    kw = dict(g["params"])
    if "slow" in kw:
        kw["slow"] = mp.MctsParams(budget_iters=kw["slow"])
    logs = []
    dep = mp.two_phase(services_of(g), store_of(g), mp.PartitionRuleSet.defaults(), mp.GaParams(**kw),
                       log=lambda r: logs.append([r.round, r.best_gpus, S.fhex(r.best_slack), r.improved]),
                       backend=impl)
    assert S.plan_key([x.config for x in dep.gpus]) == g["plan"]
    assert logs == g["logs"]


def test_two_phase_workers_deterministic(impl):  # test_ga.cpp:148-168
    ps, sv = S.random_workload(4, 321)
    p = mp.GaParams(seed=77, time_budget_s=60.0, max_rounds=4, slow=mp.MctsParams(budget_iters=16))
    a = mp.two_phase(sv, ps, mp.PartitionRuleSet.defaults(), p, backend=impl)
    p.workers = 4
    c = mp.two_phase(sv, ps, mp.PartitionRuleSet.defaults(), p, backend=impl)
    assert [g.config for g in a.gpus] == [g.config for g in c.gpus]


def test_two_phase_zero_budget_is_fast(impl):  # test_ga.cpp:110-121
    ps, sv = S.random_workload(5, 555)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    expect = mp.make_deployment(mp.fast_algo([0.0] * 5, ctx))
    got = mp.two_phase(sv, ps, mp.PartitionRuleSet.defaults(), mp.GaParams(time_budget_s=0.0), backend=impl)
    assert [g.config for g in got.gpus] == [g.config for g in expect.gpus]


def full_gpu():
    return mp.GpuConfig(tuple(mp.AssignedInstance(mp.Placement(1, s), "a", 8) for s in range(7)))


def test_crossover_cases(impl):  # test_ga.cpp:16-55
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 350.0, 100.0)], ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    parent = mp.evaluate_chromosome([full_gpu()] * 3, ctx)
    child = mp.crossover(parent, mp.MctsProcedure(), ctx, mp.GaParams(erase_fraction=0.3), mp.Rng(2, backend=impl))
    assert len(child.gpus) == 2 and mp.is_satisfied(mp.completion_of(child.gpus, sv, ps))
    for seed in range(1, 8):
        ps2, sv2 = S.random_workload(4, seed * 101)
        ctx2 = mp.make_plan_context(sv2, ps2, mp.PartitionRuleSet.defaults(), backend=impl)
        par = mp.evaluate_chromosome(mp.fast_algo([0.0] * 4, ctx2), ctx2)
        ch = mp.crossover(par, mp.MctsProcedure(mp.MctsParams(budget_iters=24)), ctx2, mp.GaParams(),
                          mp.Rng(seed, backend=impl))
        assert mp.is_satisfied(mp.completion_of(ch.gpus, sv2, ps2))


def test_mutation_cases(impl):  # test_ga.cpp:57-108
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 100.0, 100.0), mp.ServiceSpec("b", "cnn-a", 100.0, 100.0)], ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    A = lambda s, sv_: mp.AssignedInstance(mp.Placement(1, s), sv_, 8)  # noqa: E731
    g1 = mp.GpuConfig((A(0, "a"), A(1, "a"), A(2, "a")))
    g2 = mp.GpuConfig((A(0, "b"), A(1, "b")))
    parent = mp.evaluate_chromosome([g1, g2], ctx)
    child = mp.mutate(parent, mp.GaParams(mutation_pairs=1), mp.Rng(3, backend=impl), ctx)
    cnt = lambda c, i: sum(x.service_id == i for g in c.gpus for x in g.instances)  # noqa: E731
    assert cnt(child, "a") == 3 and cnt(child, "b") == 2 and child.gpus != parent.gpus
    assert mp.completion_of(child.gpus, sv, ps) == mp.completion_of(parent.gpus, sv, ps)
    for seed in range(1, 5):
        ps2, sv2 = S.random_workload(5, seed * 7 + 1)
        ctx2 = mp.make_plan_context(sv2, ps2, mp.PartitionRuleSet.defaults(), backend=impl)
        par = mp.evaluate_chromosome(mp.fast_algo([0.0] * 5, ctx2), ctx2)
        before = mp.completion_of(par.gpus, sv2, ps2)
        rng = mp.Rng(seed, backend=impl)
        for _ in range(50):
            par = mp.mutate(par, mp.GaParams(), rng, ctx2)
            assert mp.completion_of(par.gpus, sv2, ps2) == before  # bitwise


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["mcts", "ga"])
def test_rows_scored_counts_match_checker(kind):
    """The BASELINE metric's work count ("configs scored") is implementation-independent:
    the product and the CPU checker count identical rows for the same MCTS / GA call."""
    chk = S.oracle_backend()
    if chk is None:
        pytest.skip("oracle not built")
    ps = S.profiles()
    sv = S.fixture_services("slos_day", ps)
    counts = []
    for b in (S.product_backend(), chk):
        ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=b)
        ctx.reset_stats()
        if kind == "mcts":
            mp.mcts_solve(mp.zero_completion(len(sv)), ctx, mp.MctsParams(budget_iters=200), 1)
        else:
            mp.two_phase(sv, ps, mp.PartitionRuleSet.defaults(),
                         mp.GaParams(seed=24, max_rounds=2, time_budget_s=1e9), ctx=ctx)
        st = ctx.stats()
        counts.append((st["greedy_rows"], st["topk_rows"], st["topk_calls"], st["greedy_steps"]))
    assert counts[0] == counts[1]


def test_long_plan_is_fetched_not_recomputed(impl):
    """A plan longer than the caller's buffer: MIG_ERR_ARGUMENT with the length, then
    mig_last_plan returns it — the stateful call (here crossover's Rng) is not re-run."""
    import ctypes as C

    from paper_2109_11067_b200 import abi

    ps = S.profiles()
    sv = S.fixture_services("slos_day", ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    parent = mp.evaluate_chromosome(mp.fast_algo(mp.zero_completion(len(sv)), ctx), ctx)
    params = mp.GaParams(erase_fraction=0.5)
    arr = ctx._configs_to_c(parent.gpus)

    def cross(rng, cap):
        out = (abi.ConfigC * max(cap, 1))()
        n = C.c_int32()
        rc = ctx.backend.lib.mig_crossover(ctx._p, arr, len(parent.gpus), 0, C.byref(params.to_c()), rng._p, out, cap,
                                           C.byref(n))
        return rc, n.value, out

    rc, n_big, out_big = cross(mp.Rng(5, ctx.backend), 4096)
    assert rc == 0 and n_big > 4
    r2 = mp.Rng(5, ctx.backend)
    rc, n, _ = cross(r2, 4)
    assert rc == abi.MIG_ERR_ARGUMENT and n == n_big
    after = r2()  # the Rng advanced exactly as in one full call
    r3 = mp.Rng(5, ctx.backend)
    cross(r3, 4096)
    assert after == r3()
    buf = (abi.ConfigC * n)()
    got = C.c_int32()
    assert ctx.backend.lib.mig_last_plan(buf, n, C.byref(got)) == 0 and got.value == n
    assert ctx._configs_from_buf(buf, n) == ctx._configs_from_buf(out_big, n_big)
