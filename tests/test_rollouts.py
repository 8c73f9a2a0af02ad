"""Throughput-mode root-parallel rollouts (mig_rollouts / mig_mcts_solve_parallel).

Golden vectors: oracle/gen_golden.py `rollouts`, produced by the reference's own primitives
(completion_type_key, detail::topk_candidates, rollout's util add — mcts.hpp:38-143) under
the documented schedule (Philox4x32-10 draws, lock-step rounds, lowest-index key claims).
Every implementation — the B200 kernel (rollout.cu), the CPU restatement and the reference
shim — must reproduce every rollout's length, the best rollout and its path exactly.
"""
import pytest

import support as S
from support import mp

ROLL = S.load_golden("rollouts.json")


def services_of(entry):
    return [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in entry["services"]]


def store_of(entry):
    return S.profiles() if entry["store"] == "fixture" else S.two_model_store()


@pytest.mark.parametrize("name", sorted(ROLL))
def test_rollouts_match_golden(impl, name):
    g = ROLL[name]
    if impl.name != "product" and g["ref_wall_s"] > 5:
        pytest.skip("large workload: checked on the GPU only")
    ctx = mp.make_plan_context(services_of(g), store_of(g), mp.PartitionRuleSet.defaults(), backend=impl)
    prm = mp.RolloutParams(**g["params"])
    r = mp.rollouts(mp.zero_completion(ctx.n), ctx, prm, lengths=True)
    assert r.lengths == g["lengths"]
    assert (r.best_len, r.best_id, r.max_depth) == (g["best_len"], g["best_id"], g["max_depth"])
    assert (r.completed, r.capped, r.failed, r.steps, r.keys, r.rounds) == \
        (g["completed"], g["capped"], g["failed"], g["steps"], g["keys"], g["rounds"])
    assert S.plan_key([ctx.pool[i].config for i in r.path]) == g["path"]
    plan, _ = mp.mcts_solve_parallel(mp.zero_completion(ctx.n), ctx, prm)
    assert S.plan_key(plan) == g["solve_plan"]


def test_rollout_paths_are_valid_plans(impl):
    """The best rollout's configs satisfy every service (is_satisfied, core.hpp:217-221)."""
    ps = S.profiles()
    sv = S.fixture_services("slos_night", ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    r = mp.rollouts(mp.zero_completion(len(sv)), ctx, mp.RolloutParams(n_rollouts=32, seed=1))
    assert r.best_len == len(r.path) > 0
    assert mp.is_satisfied(mp.completion_of([ctx.pool[i].config for i in r.path], sv, ps))


def test_rollouts_batch_and_offset_semantics(impl):
    """Batches share one key cache; id_offset shifts the Philox streams (root-parallel shards)."""
    ps = S.profiles()
    sv = S.fixture_services("slos_day", ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    z = mp.zero_completion(len(sv))
    a = mp.rollouts(z, ctx, mp.RolloutParams(n_rollouts=30, seed=4, id_offset=30), lengths=True)
    b = mp.rollouts(z, ctx, mp.RolloutParams(n_rollouts=60, seed=4), lengths=True)
    # a single batch of ids [30, 60) and the second half of one batch of [0, 60) start from
    # the same root and draw the same streams; only the key claims may differ, so compare
    # with a checker that shares the schedule rather than assuming equality
    assert len(a.lengths) == 30 and len(b.lengths) == 60
    c = mp.rollouts(z, ctx, mp.RolloutParams(n_rollouts=60, seed=4, batch=30), lengths=True)
    d = mp.rollouts(z, ctx, mp.RolloutParams(n_rollouts=60, seed=4, batch=30), lengths=True)
    assert c.lengths == d.lengths  # deterministic
    assert all(0 < x <= c.max_depth for x in c.lengths)


def test_rollouts_zero_and_satisfied(impl):
    ps = S.profiles()
    sv = S.fixture_services("slos_day", ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    r = mp.rollouts([2.0] * len(sv), ctx, mp.RolloutParams(n_rollouts=8, seed=1, max_depth=5), lengths=True)
    assert r.lengths == [0] * 8 and r.best_len == 0 and r.best_id == 0 and r.path == []
    r = mp.rollouts(mp.zero_completion(len(sv)), ctx, mp.RolloutParams(n_rollouts=8, seed=1, max_depth=0),
                    lengths=True)
    assert r.lengths == [0] * 8 and r.best_len == -1 and r.capped == 8
    with pytest.raises(Exception):
        mp.rollouts(mp.zero_completion(len(sv)), ctx, mp.RolloutParams(n_rollouts=8, topk=33))


KAT = [  # Random123 kat_vectors for philox4x32_10 as (seed, stream, step) -> word1:word0
    (0, 0, 0, 0xe169c58d6627e8d5),                                   # ctr = 0, key = 0
    (0xFFFFFFFFFFFFFFFF, 0xFFFFFFFFFFFFFFFF, 0xFFFFFFFFFFFFFFFF,
     0x41c83b0e408f276d),                                            # ctr = ~0, key = ~0
    (0x299f31d0a4093822, 0x0370734413198a2e, 0x85a308d3243f6a88,
     0x94fdccebd16cfe09),                                            # the pi-digits vector
]


def philox_draw(b, seed, stream, step, on_device):
    import ctypes as C

    out = C.c_uint64()
    b.check(b.lib.mig_philox_u64(seed, stream, step, on_device, C.byref(out)))
    return out.value


def test_philox_known_answer_host(impl):
    """Philox4x32-10 known-answer vectors (Random123 kat_vectors: ctr=0/key=0, ctr=~0/key=~0,
    and the pi-digits vector) through each library's own Philox: the product's philox.cuh
    compiled for the host (no GPU needed), the restatement's and the shim's."""
    for seed, stream, step, want in KAT:
        assert philox_draw(impl, seed, stream, step, 0) == want


@pytest.mark.gpu
def test_philox_known_answer_device():
    """The same vectors through philox.cuh's DEVICE code path (one-thread kernel)."""
    b = S.product_backend()
    for seed, stream, step, want in KAT:
        assert philox_draw(b, seed, stream, step, 1) == want


def test_philox_product_host_without_gpu():
    """The product library answers host-path draws even without a CUDA device."""
    b = S.product_backend()
    for seed, stream, step, want in KAT:
        assert philox_draw(b, seed, stream, step, 0) == want


@pytest.mark.gpu
@pytest.mark.parametrize("persist", ["0", "1"])
@pytest.mark.parametrize("name", sorted(ROLL))
def test_rollout_launch_modes_match_golden(name, persist, monkeypatch):
    """Both launch schedules of the device rollouts — one cooperative launch for a batch that fits
    one advance pass, per-round build/advance launches otherwise (rollout.cu) — forced either way
    (MIGPLAN_ROLLOUT_PERSIST), reproduce the goldens."""
    g = ROLL[name]
    monkeypatch.setenv("MIGPLAN_ROLLOUT_PERSIST", persist)
    ctx = mp.make_plan_context(services_of(g), store_of(g), mp.PartitionRuleSet.defaults())
    r = mp.rollouts(mp.zero_completion(ctx.n), ctx, mp.RolloutParams(**g["params"]), lengths=True)
    assert r.lengths == g["lengths"]
    assert (r.best_len, r.best_id, r.keys, r.rounds, r.steps) == (g["best_len"], g["best_id"], g["keys"], g["rounds"], g["steps"])
    assert S.plan_key([ctx.pool[i].config for i in r.path]) == g["path"]


@pytest.mark.gpu
def test_rollouts_wide_services_modes_agree():
    """n > 64 services: the warp-per-rollout stepper (rollout.cu Advancer<8>, the type key over
    several 64-bit words) gives the same rollouts in both launch modes, and the winner's path is
    a plan that satisfies every service.  (The CPU restatement takes minutes at this size; the
    n <= 64 goldens pin the schedule itself.)"""
    import os
    ps, sv = S.gen(72, 5.0, seed=7)
    prm = mp.RolloutParams(n_rollouts=2048, seed=11, topk=6)
    runs = []
    for persist in ("1", "0"):
        os.environ["MIGPLAN_ROLLOUT_PERSIST"] = persist
        try:
            ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults())
            runs.append((ctx, mp.rollouts(mp.zero_completion(len(sv)), ctx, prm, lengths=True)))
        finally:
            del os.environ["MIGPLAN_ROLLOUT_PERSIST"]
    (c0, a), (c1, b) = runs
    assert a.lengths == b.lengths and a.completed == b.completed == 2048
    assert (a.best_len, a.best_id, a.keys, a.rounds, a.steps) == (b.best_len, b.best_id, b.keys, b.rounds, b.steps)
    path = [c0.pool[i].config for i in a.path]
    assert len(path) == a.best_len == min(a.lengths)
    assert mp.is_satisfied(mp.completion_of(path, sv, ps))
