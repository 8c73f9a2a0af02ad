"""Sharded greedy and root-parallel rollouts across ranks.

GPU: P virtual ranks share one B200 — each context scans 1/P of every working set on
SMs/P CTAs and the per-step winners are exchanged through device-memory boards by the
persistent kernel itself (the same code path as NVLink peer boards between GPUs).  The plan,
every best-score bit and the total rows scored must equal the unsharded reference run.
CPU: world size 2 over gloo for the rank-sharded rollouts (id ranges, MIN-reduction,
winner broadcast) with the CPU checker backend.
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as tmp

import support as S
from support import mp

GREEDY = S.load_golden("greedy.json")


def services_of(entry):
    return [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in entry["services"]]


def store_of(entry):
    return S.profiles() if entry["store"] == "fixture" else S.two_model_store()


def run_sharded(ctxs, comp):
    """All ranks in one launch; returns (plan, per-rank rows scored)."""
    from paper_2109_11067_b200 import dist as D

    plan = D.fast_algo_local(ctxs, comp)
    return S.plan_key(plan), [c.stats()["greedy_rows"] for c in ctxs]


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3, 4])
@pytest.mark.parametrize("name", ["slos_24", "gen24_8.7", "rand_n20_s13", "slos_day"])
def test_sharded_greedy_bit_exact(P, name):
    from paper_2109_11067_b200 import dist as D

    g = GREEDY[name]
    sv, ps = services_of(g), store_of(g)
    ctxs = [mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults()) for _ in range(P)]
    D.shard_local(ctxs)
    for rep in range(2):  # the exchange sequence continues across calls
        for c in ctxs:
            c.reset_stats()
        plan, rows = run_sharded(ctxs, mp.zero_completion(len(sv)))
        assert plan == g["plan"]
        assert sum(rows) == g["rows_scored"]
        assert min(rows) > 0 or len(g["plan"]) == 0
    # a partial start (completion from the first half of the plan) shards the same way
    half = [mp.GpuConfig(tuple(mp.AssignedInstance(mp.Placement(a, b), c, d) for a, b, c, d in cfg))
            for cfg in g["plan"][:len(g["plan"]) // 2]]
    comp = mp.completion_of(half, sv, ps)
    single = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults())
    assert run_sharded(ctxs, comp)[0] == S.plan_key(mp.fast_algo(comp, single))


@pytest.mark.gpu
def test_shard_reset_to_single():
    from paper_2109_11067_b200 import dist as D

    g = GREEDY["slos_night"]
    sv, ps = services_of(g), store_of(g)
    ctxs = [mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults()) for _ in range(2)]
    D.shard_local(ctxs)
    assert run_sharded(ctxs, mp.zero_completion(len(sv)))[0] == g["plan"]
    c = ctxs[0]
    c.backend.check(c.backend.lib.mig_ctx_set_shard(c._p, 0, 1, None, 0))
    assert S.plan_key(mp.fast_algo(mp.zero_completion(len(sv)), c)) == g["plan"]


def test_checkers_reject_sharding(impl):
    if impl.name == "product":
        pytest.skip("product shards")
    ps = S.profiles()
    sv = S.fixture_services("slos_day", ps)
    c = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=impl)
    assert c.backend.lib.mig_ctx_set_shard(c._p, 0, 1, None, 0) == 0
    assert c.backend.lib.mig_ctx_set_shard(c._p, 0, 2, None, 0) != 0


# ---------------------------------------------------------------- rank-sharded rollouts (gloo)

def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# ---------------------------------------------------------------- one process per rank (IPC boards)

def ipc_worker(rank, world, port, q, name, mode):
    """One rank of a process-sharded greedy: a gloo group carries the CUDA IPC handles of the
    exchange boards (dist.shard_context); every step's winner then crosses processes through
    the boards inside the persistent kernels.  All ranks share cuda:0 here (1-GPU box), so
    the grids are capped; on an 8-GPU box each rank owns a GPU and its full grid."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if mode == "timeout":
        os.environ["MIGPLAN_EXCH_TIMEOUT_MS"] = "3000"
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import time

        from paper_2109_11067_b200 import dist as D

        g = GREEDY[name]
        ctx = mp.make_plan_context(services_of(g), store_of(g), mp.PartitionRuleSet.defaults(), device=0)
        D.shard_context(ctx, 0, max_ctas=8)
        out = []
        for rep in range(2):
            if mode == "slow" and rank == world - 1:
                time.sleep(1.5)  # a peer that launches late: the others wait inside their kernels
            if mode == "timeout" and rank == world - 1:
                break  # a peer that never launches: the others' watchdog fires
            ctx.reset_stats()
            try:
                plan = S.plan_key(mp.fast_algo(mp.zero_completion(ctx.n), ctx))
                out.append((plan, ctx.stats()["greedy_rows"]))
            except RuntimeError as e:  # noqa: PERF203
                out.append(("error", str(e)))
                break
        q.put((rank, out))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def run_ipc(world, name, mode="normal"):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=ipc_worker, args=(r, world, port, q, name, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.gpu
@pytest.mark.parametrize("world,name,mode", [(2, "slos_day", "normal"), (2, "slos_24", "normal"),
                                             (3, "gen24_8.7", "normal"), (2, "slos_night", "slow")])
def test_process_sharded_greedy_ipc(world, name, mode):
    g = GREEDY[name]
    res = run_ipc(world, name, mode)
    for rep in range(2):
        plans = [res[r][rep][0] for r in range(world)]
        assert all(p == g["plan"] for p in plans)
        assert sum(res[r][rep][1] for r in range(world)) == g["rows_scored"]


@pytest.mark.gpu
def test_process_sharded_greedy_peer_never_launches():
    """A missing peer turns into MIG_ERR_DEVICE after the exchange watchdog, not a hang."""
    res = run_ipc(2, "slos_day", "timeout")
    assert res[1] == []
    assert res[0][0][0] == "error" and "timed out" in res[0][0][1]


def roll_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2109_11067_b200 import dist as D

        ps = S.profiles()
        sv = S.fixture_services("slos_day", ps)
        ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=S.checker_backend())
        prm = mp.RolloutParams(n_rollouts=50, seed=21, max_depth=36)
        win, plan, res = D.root_parallel_rollouts(mp.zero_completion(len(sv)), ctx, prm)
        q.put((rank, win, S.plan_key(plan), res.best_len, res.best_id))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(S.checker_backend() is None, reason="no CPU checker library")
def test_root_parallel_rollouts_world2():
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=roll_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, w0, p0, l0, i0), (_, w1, p1, l1, i1) = res
    assert w0 == w1 and p0 == p1
    # the same shards computed in one process: ids [0,25) and [25,50), each with its own cache
    ps = S.profiles()
    sv = S.fixture_services("slos_day", ps)
    c = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=S.checker_backend())
    shards = [mp.rollouts(mp.zero_completion(len(sv)), c, mp.RolloutParams(n_rollouts=25, seed=21, max_depth=36,
                                                                          id_offset=o)) for o in (0, 25)]
    best = min(range(2), key=lambda r: (shards[r].best_len if shards[r].best_len >= 0 else 1 << 62, r))
    assert w0 == best
    assert p0 == S.plan_key([c.pool[i].config for i in shards[best].path])
    assert (l0, i0) == (shards[0].best_len, shards[0].best_id) and (l1, i1) == (shards[1].best_len, shards[1].best_id)
