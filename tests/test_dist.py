"""Multi-process (world size 2, gloo, CPU) coverage of the multi-GPU drivers in dist.py.

Each rank plans with the CPU checker backend (the product needs a GPU); the exchange logic —
island seeds, fitness-key all-gather, winner broadcast, plan decoding — is exactly what runs
over NCCL between B200s.
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as tmp

import support as S
from support import mp


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2109_11067_b200 import dist as D

        b = S.checker_backend()
        ps, sv = S.random_workload(5, 901)
        ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=b)
        params = mp.GaParams(seed=9, time_budget_s=1e9, max_rounds=3, slow=mp.MctsParams(budget_iters=16))
        win, dep = D.island_two_phase(ctx, params)
        plan = [g.config for g in dep.gpus]
        single = [g.config for g in mp.two_phase(sv, ps, mp.PartitionRuleSet.defaults(), params, backend=b).gpus]
        w2, mplan = D.root_parallel_mcts([0.0] * 5, ctx, mp.MctsParams(budget_iters=40), 3)
        mono = mp.mcts_solve([0.0] * 5, ctx, mp.MctsParams(budget_iters=40), 3)
        q.put((rank, win, S.plan_key(plan), S.plan_key(single), mp.is_satisfied(mp.completion_of(plan, sv, ps)),
               w2, S.plan_key(mplan), len(mono)))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(S.checker_backend() is None, reason="no CPU checker library")
def test_islands_and_root_parallel_world2():
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, w0, plan0, single0, ok0, m0, mp0, mono0), (r1, w1, plan1, single1, ok1, m1, mp1, mono1) = res
    assert w0 == w1 and plan0 == plan1 and ok0 and ok1          # every rank holds the same winner
    assert len(plan0) <= len(single0)                           # never worse than two_phase(seed) on 1 GPU
    assert m0 == m1 and mp0 == mp1 and len(mp0) <= mono0       # root-parallel MCTS: same-or-fewer GPUs


def err_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2109_11067_b200 import dist as D

        ps, sv = S.random_workload(4, 77)
        ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=S.checker_backend())
        comp = [0.0] * 4 if rank == 0 else [0.0] * 3  # rank 1's local solve raises PlanningError
        try:
            D.root_parallel_mcts(comp, ctx, mp.MctsParams(budget_iters=8), 5)
            q.put((rank, "ok"))
        except mp.PlanningError as e:
            q.put((rank, "raised:" + type(e).__name__))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(S.checker_backend() is None, reason="no CPU checker library")
def test_failing_rank_does_not_hang_peers():
    """A rank whose local solve raises still joins the all-gather; every rank then raises."""
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=err_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {0: "raised:PlanningError", 1: "raised:PlanningError"}
