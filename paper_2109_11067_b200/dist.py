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


_FAILED = (1 << 63) - 1


def _pick_and_broadcast(key: tuple, plan, ctx, group=None, error: BaseException | None = None):
    """All ranks agree on the rank with the smallest key, then receive its plan.  A rank whose
    local solve raised still joins the collectives (key[0] = _FAILED), so no peer blocks in
    the all-gather; then every rank raises the failing rank's error type together."""
    world = dist.get_world_size(group)
    dev = _device(group)
    if error is not None:
        key = (_FAILED,) * (len(key) - 1) + (key[-1],)
    mine = torch.tensor(list(key) + [1 if error is not None else 0], dtype=torch.int64, device=dev)
    keys = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(keys, mine, group=group)
    keys = [tuple(int(x) for x in k.tolist()) for k in keys]
    failed = [r for r in range(world) if keys[r][-1]]
    if failed:
        if error is not None:
            raise error
        raise mp.PlanningError(f"rank {failed[0]} failed its local solve")
    keys = [k[:-1] for k in keys]
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
    try:
        dep = mp.two_phase(ctx.services, ctx.profiles, ctx.rules, p, log=log, ctx=ctx)
    except RuntimeError as e:
        _pick_and_broadcast((0, 0, rank), [], ctx, group, error=e)
    plan = [g.config for g in dep.gpus]
    slack = mp.slack_of(mp.completion_of(plan, ctx.services, ctx.profiles))
    winner, best = _pick_and_broadcast((len(plan), _slack_bits(slack), rank), plan, ctx, group)
    return winner, mp.make_deployment(best)


def root_parallel_mcts(comp, ctx: mp.PlanContext, params: mp.MctsParams, seed: int, group=None):
    """Root-parallel MCTS: rank r searches with seed mix_seed(seed, r); the shortest plan wins."""
    rank = dist.get_rank(group)
    s = mp.mix_seed(seed, rank) if rank > 0 else seed  # rank 0 == mcts_solve(seed)
    try:
        plan = mp.mcts_solve(comp, ctx, params, s)
    except RuntimeError as e:
        _pick_and_broadcast((0, rank), [], ctx, group, error=e)
    return _pick_and_broadcast((len(plan), rank), plan, ctx, group)


# ---------------------------------------------------------------- sharded greedy

def _board_alloc(ctx: mp.PlanContext, n_ranks: int, device: int, ipc: bool):
    import ctypes as C

    lib = ctx.backend.lib
    ptr = C.c_void_p()
    handle = (C.c_uint8 * 64)()
    ctx.backend.check(lib.mig_board_alloc(device, n_ranks, C.byref(ptr), handle if ipc else None))
    return ptr, bytes(handle)


def shard_local(ctxs: list):
    """Ranks sharing ONE GPU (tests, development): context r scans shard r of every working
    set; the exchange boards are plain device buffers.  Plan with fast_algo_local(ctxs, comp):
    the instances run as CTA ranges of one cooperative launch."""
    import ctypes as C

    P = len(ctxs)
    boards = [_board_alloc(c, P, c.device, False)[0] for c in ctxs]
    arr = (C.c_void_p * P)(*[b.value for b in boards])
    for r, c in enumerate(ctxs):
        c.backend.check(c.backend.lib.mig_ctx_set_shard(c._p, r, P, arr, 0))
    return boards


def fast_algo_local(ctxs: list, comp):
    """fast_algo on all ranks of a shard_local group (one launch); returns the common plan."""
    import ctypes as C

    c0 = ctxs[0]
    buf, n = c0._comp(comp)
    arr = (C.c_void_p * len(ctxs))(*[c._p.value for c in ctxs])
    return mp._run_plan(c0, lambda out, cap, nout: c0.backend.lib.mig_fast_algo_group(arr, len(ctxs), buf, n, out, cap,
                                                                                      C.byref(nout)))


def shard_context(ctx: mp.PlanContext, device: int, group=None, max_ctas: int = 0):
    """One rank per GPU (torch.distributed): allocate this rank's exchange board, all-gather
    the CUDA IPC handles, open the peers' boards (NVLink peer memory) and shard the context.
    Afterwards every rank calls mp.fast_algo SPMD and receives the identical plan.
    max_ctas > 0 caps the greedy grid (ranks sharing one GPU in tests)."""
    import ctypes as C

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    own, handle = _board_alloc(ctx, world, device, True)
    handles = [None] * world
    dist.all_gather_object(handles, handle, group=group)
    ptrs = []
    for q in range(world):
        if q == rank:
            ptrs.append(own.value)
            continue
        p = C.c_void_p()
        h = (C.c_uint8 * 64).from_buffer_copy(handles[q])
        ctx.backend.check(ctx.backend.lib.mig_board_open(device, h, C.byref(p)))
        ptrs.append(p.value)
    arr = (C.c_void_p * world)(*ptrs)
    ctx.backend.check(ctx.backend.lib.mig_ctx_set_shard(ctx._p, rank, world, arr, max_ctas))
    ctx._shard_rank = rank
    dist.barrier(group=group)  # every board is zeroed before any rank posts into it
    return ptrs


def unshard_context(ctx: mp.PlanContext, boards, group=None) -> None:
    """Undo shard_context (collective): the context scans its whole working set again; every
    rank closes its IPC mappings of the peers' boards, then (after a barrier) frees its own."""
    import ctypes as C

    rank = ctx._shard_rank
    ctx.backend.check(ctx.backend.lib.mig_ctx_set_shard(ctx._p, 0, 1, None, 0))
    for q, p in enumerate(boards):
        if q != rank:
            ctx.backend.check(ctx.backend.lib.mig_board_free(C.c_void_p(p), 1))
    dist.barrier(group=group)
    ctx.backend.check(ctx.backend.lib.mig_board_free(C.c_void_p(boards[rank]), 0))


def sharded_rows(ctx: mp.PlanContext, group=None) -> int:
    """Greedy rows scored by all ranks together (each rank counts its shard)."""
    dev = _device(group)
    t = torch.tensor([ctx.stats()["greedy_rows"]], dtype=torch.int64, device=dev)
    dist.all_reduce(t, group=group)
    return int(t.item())


# ---------------------------------------------------------------- root-parallel rollouts (throughput mode)

def root_parallel_rollouts(comp, ctx: mp.PlanContext, params: mp.RolloutParams, group=None):
    """params.n_rollouts rollouts sharded over the ranks by global id (rank r runs ids
    [r*R/P, (r+1)*R/P) with its own key cache); MIN-reduction of (best_len, best_id) and a
    broadcast of the winner's path.  Deterministic for a given rank count."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    R = params.n_rollouts
    lo, hi = R * rank // world, R * (rank + 1) // world
    p = mp.RolloutParams(**{**params.__dict__, "n_rollouts": hi - lo, "id_offset": params.id_offset + lo})
    try:
        res = mp.rollouts(comp, ctx, p)
    except RuntimeError as e:
        _pick_and_broadcast((0, 0, rank), [], ctx, group, error=e)
    plan = [ctx.pool[i].config for i in res.path]
    big = 1 << 62
    key = (res.best_len if res.best_len >= 0 else big, res.best_id if res.best_id >= 0 else big, rank)
    winner, best = _pick_and_broadcast(key, plan, ctx, group)
    return winner, best, res
