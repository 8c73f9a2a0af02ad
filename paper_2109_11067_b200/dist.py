"""Multi-GPU drivers: one process per GPU, torch.distributed for the (tiny) exchanges.

The optimizer's slow algorithms parallelise without moving candidate data:

* GA islands (ga.hpp:126-179): every rank evolves its own population from the same greedy
  seed with its own stream `mix_seed(seed, rank)`; at the end one all-gather of a 3-word
  fitness key (gpu count, slack bits, rank) picks the fittest island (`fitter`, ga.hpp:19-22)
  and one broadcast ships its plan.  With world size 1 the result is exactly
  `two_phase(seed)`.
* Root-parallel MCTS (mcts.hpp:148-252): every rank runs `mcts_solve` from the same root with
  seed `mix_seed(seed, rank)`; the shortest plan wins (ties: lowest rank).  World size 1 is
  exactly `mcts_solve(seed)`.

Each rank's compute is the B200 product (or any backend passed in); only O(plan) integers
cross the process group, over NCCL (GPUs) or gloo (CPU tests).
"""
from __future__ import annotations

import struct

import torch
import torch.distributed as dist

from . import migplan as mp


def _device(group):
    return torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")


def _encode(plan, ctx) -> list[int]:
    out = [len(plan)]
    for g in plan:
        out.append(len(g.instances))
        for i in g.instances:
            out += [i.placement.slices, i.placement.start_slot, ctx._ids[i.service_id], i.batch]
    return out


def _decode(vals, ctx):
    n, p, plan = vals[0], 1, []
    for _ in range(n):
        k = vals[p]
        p += 1
        inst = []
        for _ in range(k):
            s, t, svc, b = vals[p:p + 4]
            p += 4
            inst.append(mp.AssignedInstance(mp.Placement(s, t), ctx.services[svc].service_id, b))
        plan.append(mp.GpuConfig(tuple(inst)))
    return plan


def _pick_and_broadcast(key: tuple, plan, ctx, group=None):
    """All ranks agree on the rank with the smallest key, then receive its plan."""
    world = dist.get_world_size(group)
    dev = _device(group)
    mine = torch.tensor(list(key), dtype=torch.int64, device=dev)
    keys = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(keys, mine, group=group)
    keys = [tuple(int(x) for x in k.tolist()) for k in keys]
    winner = min(range(world), key=lambda r: keys[r])
    enc = _encode(plan, ctx)
    length = torch.tensor([len(enc)], dtype=torch.int64, device=dev)
    dist.broadcast(length, src=winner, group=group)
    buf = torch.tensor(enc, dtype=torch.int64, device=dev) if dist.get_rank(group) == winner else \
        torch.zeros(int(length.item()), dtype=torch.int64, device=dev)
    dist.broadcast(buf, src=winner, group=group)
    return winner, _decode([int(x) for x in buf.tolist()], ctx)


def _slack_bits(x: float) -> int:
    # non-negative doubles order like their IEEE bit patterns
    return struct.unpack("<q", struct.pack("<d", x))[0]


def island_two_phase(ctx: mp.PlanContext, params: mp.GaParams, group=None, log=None):
    """GA islands: rank r runs two_phase with seed mix_seed(params.seed, r); the fittest wins."""
    rank = dist.get_rank(group)
    p = mp.GaParams(**{**params.__dict__})
    if rank > 0:  # rank 0 keeps the caller's seed: the result is never worse than two_phase(seed)
        p.seed = mp.mix_seed(params.seed, rank)
    dep = mp.two_phase(ctx.services, ctx.profiles, ctx.rules, p, log=log, ctx=ctx)
    plan = [g.config for g in dep.gpus]
    slack = mp.slack_of(mp.completion_of(plan, ctx.services, ctx.profiles))
    winner, best = _pick_and_broadcast((len(plan), _slack_bits(slack), rank), plan, ctx, group)
    return winner, mp.make_deployment(best)


def root_parallel_mcts(comp, ctx: mp.PlanContext, params: mp.MctsParams, seed: int, group=None):
    """Root-parallel MCTS: rank r searches with seed mix_seed(seed, r); the shortest plan wins."""
    rank = dist.get_rank(group)
    s = mp.mix_seed(seed, rank) if rank > 0 else seed  # rank 0 == mcts_solve(seed)
    plan = mp.mcts_solve(comp, ctx, params, s)
    return _pick_and_broadcast((len(plan), rank), plan, ctx, group)
