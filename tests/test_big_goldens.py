"""Parity on the configurations the headline claims are made on (BASELINE.json configs #2-#5).

Golden vectors (oracle/gen_golden.py, from the UNMODIFIED reference compiled in oracle/_ref):
  ga_big.json        two_phase on slos_24 (seed 24, P=16, MCTS 48; 2 and 10 rounds) and on
                     gen(24, 8.7) (config #3), ga.hpp:126-179 — plan + every round log
  greedy_big.json    fast_algo on gen(48, 7.0) (config #4), greedy.hpp:95-145 — plan, every
                     best_score bit, completion digests, rows scored (~6 min on one core)
  mcts_big.json      mcts_solve on gen(48, 7.0), 200 iterations, seed 1 (mcts.hpp:148-252)
  greedy_prefix.json gen(128, 8.0) (config #5): the reference's fast_algo up to two steps past
                     its first extension event (greedy.hpp:107-119, config_enum.hpp:206-211),
                     every pick and score bit, and each step's working-set size
  pools_big.json     base-pool SET digests at n = 48 and n = 128 (config_enum.hpp:192-202)
  rollouts_big.json  root-parallel rollouts at gen(48, 7.0) (reference primitives, Philox)

The CPU checkers take minutes to hours on these sizes, so only the product runs them
(``-m gpu``); the restatement and the shim are pinned on the small goldens elsewhere.
"""
import ctypes as C
import os

import pytest

import support as S
from support import mp

pytestmark = pytest.mark.gpu


def _gold(name):
    path = os.path.join(S.GOLDEN, name)
    return S.load_golden(name) if os.path.exists(path) else {}


GA_BIG = _gold("ga_big.json")
GREEDY_BIG = _gold("greedy_big.json")
MCTS_BIG = _gold("mcts_big.json")
PREFIX = _gold("greedy_prefix.json")
POOLS = _gold("pools_big.json")
ROLL_BIG = _gold("rollouts_big.json")


def services_of(entry):
    return [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in entry["services"]]


def store_of(entry):
    return S.profiles() if entry["store"] == "fixture" else S.two_model_store()


def product_ctx(g):
    return mp.make_plan_context(services_of(g), store_of(g), mp.PartitionRuleSet.defaults(),
                                backend=S.product_backend())


def step_rows(ctx):
    cap = 1 << 16
    buf = (C.c_int64 * cap)()
    n = C.c_int32()
    ctx.backend.check(ctx.backend.lib.mig_ctx_step_rows(ctx._p, buf, cap, C.byref(n)))
    return list(buf[:min(n.value, cap)])


@pytest.mark.parametrize("name", sorted(GA_BIG))
def test_two_phase_headline_configs(name):
    g = GA_BIG[name]
    kw = {k: v for k, v in g["params"].items() if k not in ("slow",)}
    params = mp.GaParams(time_budget_s=1e9, workers=8, slow=mp.MctsParams(budget_iters=g["params"]["slow"]), **kw)
    logs = []
    dep = mp.two_phase(services_of(g), store_of(g), mp.PartitionRuleSet.defaults(), params,
                       log=lambda r: logs.append([r.round, r.best_gpus, S.fhex(r.best_slack), r.improved]),
                       backend=S.product_backend())
    plan = S.plan_key([x.config for x in dep.gpus])
    assert logs == g["logs"]
    assert S.plan_sha(plan) == g["plan_sha"]
    assert plan == g["plan"]


@pytest.mark.parametrize("name", sorted(GREEDY_BIG))
def test_greedy_gen48(name):
    g = GREEDY_BIG[name]
    ctx = product_ctx(g)
    assert len(ctx.pool) == g["pool_size"]
    trace = []
    ctx.reset_stats()
    plan = mp.fast_algo(mp.zero_completion(ctx.n), ctx,
                        trace=lambda i, c, s, comp: trace.append([S.fhex(s), S.comp_digest(comp)]))
    assert trace == g["trace"]
    assert S.plan_key(plan) == g["plan"]
    assert ctx.stats()["greedy_rows"] == g["rows_scored"]
    sv, ps = services_of(g), store_of(g)
    assert [S.fhex(c) for c in mp.completion_of(plan, sv, ps)] == g["final_comp"]


@pytest.mark.parametrize("name", sorted(MCTS_BIG))
def test_mcts_gen48(name):
    g = MCTS_BIG[name]
    ctx = product_ctx(g)
    tr = []
    plan = mp.mcts_solve(mp.zero_completion(ctx.n), ctx, mp.MctsParams(budget_iters=g["budget"]), g["seed"],
                         trace=lambda *a: tr.append(list(a)))
    assert tr == g["trace"]
    assert S.plan_key(plan) == g["plan"]


@pytest.mark.parametrize("name", sorted(PREFIX))
def test_greedy_gen128_prefix(name):
    """Every pick and best_score bit of the reference's first `steps` steps at n = 128, which
    include two scans over the first extension (tens of millions of rows, HBM-streamed), and
    each step's working-set size (the extension's exact row count)."""
    g = PREFIX[name]
    ctx = product_ctx(g)
    assert len(ctx.pool) == g["pool_size"]
    trace, picks = [], []

    def tr(i, cand, s, comp):
        if i < g["steps"]:
            trace.append([S.fhex(s), S.comp_digest(comp)])
            picks.append(cand.config)

    plan = mp.fast_algo(mp.zero_completion(ctx.n), ctx, trace=tr)
    assert len(plan) > g["steps"]
    assert trace == g["trace"]
    assert S.plan_key(picks) == g["plan"]
    assert step_rows(ctx)[:g["steps"]] == g["step_rows"]
    # the extensions' sizes: one event after each traced step here, so the working set of
    # step j + 1 is step j's plus event j's rows (config_enum.hpp:206-211)
    assert g["first_ext_step"] == 0
    for j in range(g["steps"] - 1):
        assert g["step_rows"][j + 1] - g["step_rows"][j] == g["ext_rows"][j]
    assert mp.is_satisfied(mp.completion_of(plan, services_of(g), store_of(g)))


@pytest.mark.parametrize("name", sorted(POOLS))
def test_base_pool_set_large(name):
    g = POOLS[name]
    ctx = product_ctx(g)
    assert len(ctx.pool) == g["pool_size"]
    assert [S.fhex(x) for x in ctx.pool.best_single_util] == g["best_single_util"]
    assert S.pool_sha(ctx) == g["pool_sha"]


@pytest.mark.parametrize("name", sorted(ROLL_BIG))
def test_rollouts_gen48(name):
    g = ROLL_BIG[name]
    ctx = product_ctx(g)
    r = mp.rollouts(mp.zero_completion(ctx.n), ctx, mp.RolloutParams(**g["params"]), lengths=True)
    assert r.lengths == g["lengths"]
    assert (r.best_len, r.best_id, r.max_depth) == (g["best_len"], g["best_id"], g["max_depth"])
    assert (r.completed, r.capped, r.failed, r.steps, r.keys, r.rounds) == \
        (g["completed"], g["capped"], g["failed"], g["steps"], g["keys"], g["rounds"])
    assert S.plan_key([ctx.pool[i].config for i in r.path]) == g["path"]
