"""Generate tests/golden/*.json from the compiled reference (oracle/_ref/libmigref.so).

TEST INFRASTRUCTURE ONLY.  Every vector here is produced by the UNMODIFIED reference
headers (behind oracle/ref_shim.cpp) on inputs that are either the reference's own
fixtures (proj/fixtures/*.json, copied to tests/golden/fixtures) or workloads produced
by the reference's own gen_workload (bench.hpp:125-156).  Floats are stored as
float.hex() so comparisons are bit-exact.

    python oracle/gen_golden.py [section ...]     # sections: greedy mcts ga topk partitions
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests"))

import support as S  # noqa: E402
from support import mp  # noqa: E402


def svc_json(services):
    return [[s.service_id, s.model_name, s.required_rps.hex(), s.max_p90_ms.hex()] for s in services]


def store_name(ps):
    return "two_model" if "cnn-a" in ps else "fixture"


def workloads_greedy():
    ps = S.profiles()
    out = []
    for name in ("slos_day", "slos_night", "slos_24"):
        out.append((name, ps, S.fixture_services(name, ps)))
    for n, mu in ((24, 6.35), (24, 8.0), (24, 8.7)):
        p2, sv = S.gen(n, mu)
        out.append((f"gen{n}_{mu}", p2, sv))
    for seed in range(1, 51):  # test_greedy.cpp:66-74
        p2, sv = S.random_workload(2 + seed % 7, seed * 31)
        out.append((f"rand{seed}", p2, sv))
    for n, seed in ((12, 7), (16, 11), (20, 13)):  # larger two-model workloads (many extensions)
        p2, sv = S.random_workload(n, seed)
        out.append((f"rand_n{n}_s{seed}", p2, sv))
    return out


def greedy_entry(ps, sv, ref):
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=ref)
    trace = []
    t = time.time()
    plan = mp.fast_algo(mp.zero_completion(len(sv)), ctx,
                        trace=lambda i, c, s, comp: trace.append([S.fhex(s), S.comp_digest(comp)]))
    wall = time.time() - t
    import ctypes as C
    rows = C.c_int64()
    buf, n = ctx._comp(mp.zero_completion(len(sv)))
    ref.check(ref.lib.mig_ref_count_rows(ctx._p, buf, n, C.byref(rows)))
    return {"store": store_name(ps), "services": svc_json(sv), "pool_size": len(ctx.pool), "plan": S.plan_key(plan),
            "trace": trace, "rows_scored": rows.value, "ref_wall_s": round(wall, 4),
            "final_comp": [S.fhex(c) for c in mp.completion_of(plan, sv, ps)]}


def gen_greedy(ref):
    res = {}
    for name, ps, sv in workloads_greedy():
        res[name] = greedy_entry(ps, sv, ref)
        print(f"greedy {name}: {len(res[name]['plan'])} GPUs, {res[name]['rows_scored']} rows", flush=True)
    return res


def gen_mcts(ref):
    res = {}
    ps = S.profiles()
    cases = [("slos_day", ps, S.fixture_services("slos_day", ps), 200, 1),
             ("slos_night", ps, S.fixture_services("slos_night", ps), 200, 1)]
    for seed in range(1, 16):  # test_mcts.cpp:128-140
        p2, sv = S.random_workload(3 + seed % 5, seed * 17)
        cases.append((f"rand{seed}", p2, sv, 60, seed))
    p2, sv = S.random_workload(5, 4242)  # test_mcts.cpp:142-153
    cases += [("det31", p2, sv, 80, 31), ("det32", p2, sv, 80, 32)]
    p2, sv = S.gen(24, 6.35)
    cases.append(("gen24_6.35", p2, sv, 200, 1))
    for name, p, sv, budget, seed in cases:
        ctx = mp.make_plan_context(sv, p, mp.PartitionRuleSet.defaults(), backend=ref)
        tr = []
        plan = mp.mcts_solve(mp.zero_completion(len(sv)), ctx, mp.MctsParams(budget_iters=budget), seed,
                             trace=lambda *a: tr.append(list(a)))
        res[name] = {"store": store_name(p), "services": svc_json(sv), "budget": budget, "seed": seed,
                     "plan": S.plan_key(plan), "trace": tr}
        print(f"mcts {name}: {len(plan)} GPUs", flush=True)
    return res


def gen_ga(ref):
    res = {}
    ps = S.profiles()
    cases = [("slos_day", ps, S.fixture_services("slos_day", ps), dict(seed=24, max_rounds=3, time_budget_s=1e9)),
             ("slos_night", ps, S.fixture_services("slos_night", ps), dict(seed=24, max_rounds=3, time_budget_s=1e9))]
    p2, sv = S.random_workload(4, 321)  # test_ga.cpp:148-168
    cases.append(("det77", p2, sv, dict(seed=77, max_rounds=4, time_budget_s=60.0, slow=mp.MctsParams(budget_iters=16))))
    p2, sv = S.random_workload(5, 901)  # test_ga.cpp:123-146
    cases.append(("stall9", p2, sv, dict(seed=9, max_rounds=40, time_budget_s=300.0, stall_rounds=10,
                                         slow=mp.MctsParams(budget_iters=24))))
    for name, p, sv, kw in cases:
        params = mp.GaParams(**kw)
        logs = []
        dep = mp.two_phase(sv, p, mp.PartitionRuleSet.defaults(), params,
                           log=lambda r: logs.append([r.round, r.best_gpus, S.fhex(r.best_slack), r.improved]),
                           backend=ref)
        kw2 = {k: (v.budget_iters if isinstance(v, mp.MctsParams) else v) for k, v in kw.items()}
        res[name] = {"store": store_name(p), "services": svc_json(sv), "params": kw2,
                     "plan": S.plan_key([g.config for g in dep.gpus]), "logs": logs}
        print(f"ga {name}: {len(dep.gpus)} GPUs, {len(logs)} rounds", flush=True)
    return res


def gen_topk(ref):
    res = {}
    import random
    rnd = random.Random(5)
    ps = S.profiles()
    for name, p, sv in (("slos_day", ps, S.fixture_services("slos_day", ps)),
                        ("slos_24", ps, S.fixture_services("slos_24", ps)),
                        ("rand_n12", *S.random_workload(12, 7))):
        ctx = mp.make_plan_context(sv, p, mp.PartitionRuleSet.defaults(), backend=ref)
        cases = []
        for trial in range(12):
            comp = [rnd.choice([0.0, rnd.random(), 1.0 + rnd.random(), 0.999999999]) for _ in sv]
            k = rnd.choice([1, 3, 10, 25])
            top = mp.topk_candidates(ctx, comp, k)
            sub = sorted(rnd.sample(range(len(ctx.pool)), min(len(ctx.pool), 40)))
            top_sub = mp.topk_candidates(ctx, comp, k, sub)
            cases.append({"comp": [S.fhex(c) for c in comp], "k": k,
                          "top": S.plan_key([ctx.pool[i].config for i in top]),
                          "subset": S.plan_key([ctx.pool[i].config for i in sub]),
                          "top_subset": S.plan_key([ctx.pool[i].config for i in top_sub])})
        res[name] = {"store": store_name(p), "services": svc_json(sv), "cases": cases}
        print(f"topk {name}", flush=True)
    return res


def gen_partitions(ref):
    out = {}
    r = mp.PartitionRuleSet.defaults()
    out["defaults"] = [[[p.slices, p.start_slot] for p in lp.placements] for lp in mp.enumerate_maximal_partitions(r, ref)]
    r2 = mp.PartitionRuleSet.defaults()
    r2.hard_exclusions = set()
    out["no_exclusion"] = [[[p.slices, p.start_slot] for p in lp.placements]
                           for lp in mp.enumerate_maximal_partitions(r2, ref)]
    return out


def gen_rollouts(ref):
    """Throughput-mode root-parallel rollouts (mig_rollouts) on the reference's own primitives
    (completion_type_key, detail::topk_candidates, rollout's util add) under the product's
    documented schedule: Philox draws, lock-step rounds, lowest-index key claims."""
    res = {}
    ps = S.profiles()
    tw, sv12 = S.random_workload(12, 7)
    cases = [("slos_day", ps, S.fixture_services("slos_day", ps), dict(n_rollouts=64, seed=7)),
             ("slos_night", ps, S.fixture_services("slos_night", ps), dict(n_rollouts=48, seed=3, topk=4)),
             ("slos_day_capped", ps, S.fixture_services("slos_day", ps), dict(n_rollouts=40, seed=9, max_depth=12)),
             ("rand12", tw, sv12, dict(n_rollouts=200, seed=12, topk=16)),
             ("slos_24", ps, S.fixture_services("slos_24", ps), dict(n_rollouts=256, seed=11)),
             ("slos_24_batched", ps, S.fixture_services("slos_24", ps), dict(n_rollouts=256, seed=11, batch=100,
                                                                              id_offset=1000))]
    p2, sv = S.gen(24, 6.35)
    cases.append(("gen24_6.35", p2, sv, dict(n_rollouts=512, seed=5)))
    for name, p, sv, kw in cases:
        ctx = mp.make_plan_context(sv, p, mp.PartitionRuleSet.defaults(), backend=ref)
        prm = mp.RolloutParams(**kw)
        t = time.time()
        r = mp.rollouts(mp.zero_completion(len(sv)), ctx, prm, lengths=True)
        plan, r2 = mp.mcts_solve_parallel(mp.zero_completion(len(sv)), ctx, prm)
        res[name] = {"store": store_name(p), "services": svc_json(sv), "params": kw, "best_len": r.best_len,
                     "best_id": r.best_id, "max_depth": r.max_depth, "keys": r.keys, "steps": r.steps,
                     "rounds": r.rounds, "completed": r.completed, "capped": r.capped, "failed": r.failed,
                     "lengths": r.lengths, "path": S.plan_key([ctx.pool[i].config for i in r.path]),
                     "solve_plan": S.plan_key(plan), "ref_wall_s": round(time.time() - t, 3)}
        print(f"rollouts {name}: best {r.best_len} (id {r.best_id}), keys {r.keys}, solve {len(plan)} GPUs "
              f"({time.time() - t:.1f}s)", flush=True)
    return res


def gen_ga_parallel(ref):
    """Throughput-mode two_phase (mig_two_phase_parallel): the reference's operators and
    fast_algo refill under the product's Philox draw rule."""
    res = {}
    ps = S.profiles()
    tw, sv6 = S.random_workload(6, 77)
    cases = [("slos_day", ps, S.fixture_services("slos_day", ps), dict(seed=24, max_rounds=4)),
             ("slos_night", ps, S.fixture_services("slos_night", ps), dict(seed=5, max_rounds=4, population=8)),
             ("rand6", tw, sv6, dict(seed=9, max_rounds=5, mutation_pairs=3, erase_fraction=0.25)),
             ("slos_24", ps, S.fixture_services("slos_24", ps), dict(seed=24, max_rounds=3)),
             # population 20: from round 5 on, 10 children per generation (two refill batches of 8)
             ("slos_day_p20", ps, S.fixture_services("slos_day", ps), dict(seed=7, max_rounds=7, population=20)),
             ("slos_24_p20", ps, S.fixture_services("slos_24", ps), dict(seed=24, max_rounds=6, population=20))]
    only = os.environ.get("GOLDEN_ONLY")
    for name, p, sv, kw in cases:
        if only and name not in only.split(","):
            continue
        t = time.time()
        logs = []
        dep = mp.two_phase_parallel(sv, p, mp.PartitionRuleSet.defaults(), mp.GaParams(time_budget_s=1e9, **kw),
                                    log=lambda l: logs.append([l.round, l.best_gpus, l.best_slack.hex(), l.improved]),
                                    backend=ref)
        res[name] = {"store": store_name(p), "services": svc_json(sv), "params": kw,
                     "plan": S.plan_key([g.config for g in dep.gpus]), "log": logs,
                     "ref_wall_s": round(time.time() - t, 3)}
        print(f"ga_parallel {name}: {len(dep.gpus)} GPUs ({time.time() - t:.1f}s)", flush=True)
    return res


def gen_greedy_big(ref):
    """gen(48, 7.0): ~6 minutes on one core; pins the n=48 plan bit-exactly."""
    p2, sv = S.gen(48, 7.0)
    e = greedy_entry(p2, sv, ref)
    print(f"greedy gen48_7.0: {len(e['plan'])} GPUs, {e['rows_scored']} rows", flush=True)
    return {"gen48_7.0": e}


def gen_brute_force(ref):
    """brute_force_optimum (bench.hpp:160-219) on the instances the reference's own tests give it:
    test_bench.cpp:120-160, test_mcts.cpp:108-126, acceptance.cpp:202-244 (criterion 6), plus
    4-service random workloads (fixtures.hpp:51-58).  outcome: plan | "none" | "error:<msg>"."""
    rules = mp.PartitionRuleSet.defaults()
    tm, fx = S.two_model_store(), S.profiles()
    cases = [("bench_single", tm, [mp.ServiceSpec("a", "cnn-a", 350.0, 100.0)], 3),
             ("bench_overcap", tm, [mp.ServiceSpec("a", "cnn-a", 3500.0, 100.0)], 3)]
    for seed in range(1, 11):
        cases.append((f"bench_vs_fast_{seed}", tm, [mp.ServiceSpec("a", "cnn-a", 80.0 + 60.0 * (seed % 4), 100.0),
                                                  mp.ServiceSpec("b", "nlp-a", 40.0 + 30.0 * (seed % 3), 100.0)], 4))
    for seed in range(1, 9):
        cases.append((f"mcts_tiny_{seed}", tm, [mp.ServiceSpec("a", "cnn-a", 120.0 + 40.0 * (seed % 5), 100.0),
                                              mp.ServiceSpec("b", "nlp-a", 60.0 + 20.0 * (seed % 3), 100.0)], 3))
    for s in range(1, 41):
        n = 1 + s % 3
        sv = mp.gen_workload(n, True, 4.6, 0.6, 100.0, 31000 + s, fx, backend=S.host_backend())
        cases.append((f"accept_c6_{s}", fx, list(sv), 3))
    for s in range(1, 9):  # 4 services, lighter demand: depth-4 searches over the n=4 pool
        sv = mp.gen_workload(4, True, 4.0 + 0.1 * s, 0.6, 100.0, 500 + s, fx, backend=S.host_backend())
        cases.append((f"gen4_{s}", fx, list(sv), 4))
    # n >= 5: the max_mix = min(n, 7) pool holds 5..7-service configs (the reference's own
    # budget-guard case has 6 services, test_bench.cpp:154-159)
    guard = [mp.ServiceSpec(f"s{i}", "cnn-a", 900.0, 100.0) for i in range(6)]
    cases.append(("budget_guard_6", tm, guard, 4, 2000))
    for n, mu in ((5, 2.5), (6, 2.5), (7, 2.0), (8, 2.0)):
        for s in range(1, 4):
            sv = mp.gen_workload(n, True, mu, 0.6, 100.0, 900 + 10 * n + s, fx, backend=S.host_backend())
            cases.append((f"wide{n}_{s}", fx, list(sv), 3))
    for n in (5, 6, 7):
        for s in range(1, 5):
            sv = mp.gen_workload(n, True, 3.0 + 0.3 * s, 0.6, 100.0, 700 + 10 * n + s, fx, backend=S.host_backend())
            cases.append((f"widegen{n}_{s}", fx, list(sv), 3))
    for n, mu, s in ((10, 1.5, 1), (16, 2.0, 2)):
        sv = mp.gen_workload(n, True, mu, 0.6, 100.0, 900 + 10 * n + s, fx, backend=S.host_backend())
        cases.append((f"wide{n}_{s}", fx, list(sv), 3))
    res = {}
    for case in cases:
        name, ps, sv, cap = case[:4]
        budget = case[4] if len(case) > 4 else 20_000_000
        t = time.time()
        try:
            dep = mp.brute_force_optimum(sv, ps, rules, cap, node_budget=budget, backend=ref)
            out = "none" if dep is None else S.plan_key([g.config for g in dep.gpus])
        except mp.PlanningError as e:
            out = "error:" + str(e)
        res[name] = {"store": store_name(ps), "services": svc_json(sv), "cap": cap, "outcome": out,
                     "ref_wall_s": round(time.time() - t, 3)}
        if budget != 20_000_000:
            res[name]["node_budget"] = budget
        if not (isinstance(out, str) and out.startswith("error")) and res[name]["ref_wall_s"] < 0.3:
            lo, hi = 0, 20_000_000  # the reference's exact node count: the smallest budget that passes
            while lo < hi:
                mid = (lo + hi) // 2
                try:
                    mp.brute_force_optimum(sv, ps, rules, cap, node_budget=mid, backend=ref)
                    hi = mid
                except mp.PlanningError:
                    lo = mid + 1
            res[name]["nodes"] = lo
        print(f"brute_force {name}: {out if isinstance(out, str) else len(out)} ({time.time() - t:.2f}s)", flush=True)
    return res


def gen_baseline(ref):
    """baseline(kind, services, profiles) (bench.hpp:42-90) for the three static partitions on
    fixture workloads (with and without the 1/7- and 2/7-infeasible gpt2-medium services),
    generated workloads and two-model random workloads.  outcome: plan | "error:<msg>"."""
    fx, tm = S.profiles(), S.two_model_store()
    cases = []
    for name in ("slos_day", "slos_night", "slos_24"):
        sv = S.fixture_services(name, fx)
        cases.append((name, fx, sv))
        cases.append((name + "_no_gpt2", fx, [x for x in sv if x.model_name != "gpt2-medium"]))
    for s in (1, 2, 3):
        sv = mp.gen_workload(12, True, 6.0 + s, 0.6, 100.0, 900 + s, fx, backend=S.host_backend())
        cases.append((f"gen12_{s}_no_gpt2", fx, [x for x in sv if x.model_name != "gpt2-medium"]))
    for seed in (3, 4, 7, 8):
        ps, sv = S.random_workload(6, seed)
        cases.append((f"rand6_{seed}", ps, list(sv)))
    res = {}
    for name, ps, sv in cases:
        for kind in (0, 1, 2):
            try:
                dep = mp.baseline(kind, sv, ps, backend=ref)
                out = S.plan_key([g.config for g in dep.gpus])
            except mp.PlanningError as e:
                out = "error:" + str(e)
            res[f"{name}/{kind}"] = {"store": store_name(ps), "services": svc_json(sv), "kind": kind, "outcome": out}
            print(f"baseline {name}/{kind}: {out if isinstance(out, str) else len(out)}", flush=True)
    return res


def gen_ga_big(ref):
    """two_phase on the configs the headline claims are made on:
    config #2 slos_24 (seed 24, P=16, MCTS budget 48, the c7 parameters with max_rounds
    binding, acceptance.cpp:255-259) at 2 and 10 rounds, and config #3 gen(24, 8.7)."""
    res = {}
    ps = S.profiles()
    slos = S.fixture_services("slos_24", ps)
    p3, g3 = S.gen(24, 8.7)
    cases = [("slos_24_r2", ps, slos, dict(seed=24, max_rounds=2)),
             ("slos_24_r10", ps, slos, dict(seed=24, max_rounds=10)),
             ("gen24_8.7_r2", p3, g3, dict(seed=4242, max_rounds=2)),
             ("gen24_8.7_r10", p3, g3, dict(seed=4242, max_rounds=10))]
    only = os.environ.get("GOLDEN_ONLY")
    for name, p, sv, kw in cases:
        if only and name not in only.split(","):
            continue
        params = mp.GaParams(time_budget_s=1e9, population=16, workers=min(os.cpu_count() or 1, 8),
                             slow=mp.MctsParams(budget_iters=48), **kw)
        logs = []
        t = time.time()
        dep = mp.two_phase(sv, p, mp.PartitionRuleSet.defaults(), params,
                           log=lambda r: logs.append([r.round, r.best_gpus, S.fhex(r.best_slack), r.improved]),
                           backend=ref)
        plan = S.plan_key([g.config for g in dep.gpus])
        res[name] = {"store": store_name(p), "services": svc_json(sv), "params": {**kw, "slow": 48, "population": 16},
                     "plan": plan, "plan_sha": S.plan_sha(plan), "logs": logs,
                     "ref_wall_s": round(time.time() - t, 2)}
        print(f"ga_big {name}: {len(dep.gpus)} GPUs, {len(logs)} rounds ({time.time() - t:.1f}s)", flush=True)
    return res


def gen_mcts_big(ref):
    """mcts_solve on config #4's gen(48, 7.0) with a bounded budget."""
    p, sv = S.gen(48, 7.0)
    budget, seed = int(os.environ.get("MCTS_BIG_BUDGET", "200")), 1
    ctx = mp.make_plan_context(sv, p, mp.PartitionRuleSet.defaults(), backend=ref)
    tr = []
    t = time.time()
    plan = mp.mcts_solve(mp.zero_completion(len(sv)), ctx, mp.MctsParams(budget_iters=budget), seed,
                         trace=lambda *a: tr.append(list(a)))
    print(f"mcts_big gen48_7.0: {len(plan)} GPUs ({time.time() - t:.1f}s)", flush=True)
    return {"gen48_7.0": {"store": "fixture", "services": svc_json(sv), "budget": budget, "seed": seed,
                          "plan": S.plan_key(plan), "trace": tr, "ref_wall_s": round(time.time() - t, 2)}}


def gen_greedy_prefix(ref):
    """gen(128, 8.0) (config #5): the reference's own fast_algo up to and including the
    first two steps that scan the first extension (greedy.hpp:107-136; config_enum.hpp:206-211),
    every pick and score bit, plus the instrumented replica's per-step working-set sizes
    (VERDICT r1 item 1d).  The full plan is not completable on a CPU."""
    import ctypes as C

    p, sv = S.gen(128, 8.0)
    ctx = mp.make_plan_context(sv, p, mp.PartitionRuleSet.defaults(), backend=ref)
    trace = []
    plan = []

    def _tr(_u, it, cand, s, cp, nn):
        c = ctx._cand_from_c(cand.contents)
        plan.append(c.config)
        trace.append([S.fhex(s), S.comp_digest(list(cp[:nn]))])

    cb = abi_trace(_tr)
    buf, n = ctx._comp(mp.zero_completion(len(sv)))
    steps, ext_at = C.c_int32(), C.c_int32()
    t = time.time()
    ref.check(ref.lib.mig_ref_fast_algo_prefix(ctx._p, buf, n, -1, 2, cb, None, C.byref(steps), C.byref(ext_at)))
    wall = time.time() - t
    cap = steps.value + 1
    sr = (C.c_int64 * cap)()
    er = (C.c_int64 * 64)()
    ns, ne = C.c_int32(), C.c_int32()
    t2 = time.time()
    ref.check(ref.lib.mig_ref_step_rows(ctx._p, buf, n, steps.value, sr, cap, C.byref(ns), er, 64, C.byref(ne)))
    print(f"greedy_prefix gen128_8.0: {steps.value} steps, first extension after step {ext_at.value}, "
          f"ext rows {list(er[:ne.value])} ({wall:.1f}s + {time.time() - t2:.1f}s)", flush=True)
    return {"gen128_8.0": {"store": "fixture", "services": svc_json(sv), "pool_size": len(ctx.pool),
                           "steps": steps.value, "first_ext_step": ext_at.value, "plan": S.plan_key(plan),
                           "trace": trace, "step_rows": list(sr[:ns.value]), "ext_rows": list(er[:ne.value]),
                           "ref_wall_s": round(wall, 2)}}


def abi_trace(fn):
    from paper_2109_11067_b200 import abi

    return abi.GREEDY_TRACE(fn)


def gen_pools_big(ref):
    """Base-pool SET parity at n = 48 and n = 128 (config_enum.hpp:192-202): count, a digest of
    the sorted canonical rows (configs, utility bits, util_sum bits), best_single_util bits."""
    res = {}
    for n, mu in ((48, 7.0), (128, 8.0)):
        p, sv = S.gen(n, mu)
        t = time.time()
        ctx = mp.make_plan_context(sv, p, mp.PartitionRuleSet.defaults(), backend=ref)
        res[f"gen{n}_{mu}"] = {"store": "fixture", "services": svc_json(sv), "pool_size": len(ctx.pool),
                               "pool_sha": S.pool_sha(ctx),
                               "best_single_util": [S.fhex(x) for x in ctx.pool.best_single_util]}
        print(f"pools_big gen{n}_{mu}: {len(ctx.pool)} rows ({time.time() - t:.1f}s)", flush=True)
    return res


def gen_rollouts_big(ref):
    """Root-parallel rollouts at config #4's gen(48, 7.0); max_depth
    = 2 x the reference greedy's 372 GPUs (mcts.hpp:127)."""
    p, sv = S.gen(48, 7.0)
    res = {}
    for name, kw in (("gen48_7.0", dict(n_rollouts=1024, seed=1, max_depth=744)),
                     ("gen48_7.0_k4", dict(n_rollouts=512, seed=3, max_depth=744, topk=4))):
        ctx = mp.make_plan_context(sv, p, mp.PartitionRuleSet.defaults(), backend=ref)
        prm = mp.RolloutParams(**kw)
        t = time.time()
        r = mp.rollouts(mp.zero_completion(len(sv)), ctx, prm, lengths=True)
        res[name] = {"store": "fixture", "services": svc_json(sv), "params": kw, "best_len": r.best_len,
                     "best_id": r.best_id, "max_depth": r.max_depth, "keys": r.keys, "steps": r.steps,
                     "rounds": r.rounds, "completed": r.completed, "capped": r.capped, "failed": r.failed,
                     "lengths": r.lengths, "path": S.plan_key([ctx.pool[i].config for i in r.path]),
                     "ref_wall_s": round(time.time() - t, 2)}
        print(f"rollouts_big {name}: best {r.best_len}, keys {r.keys} ({time.time() - t:.1f}s)", flush=True)
    return res


def gen_ga_parallel_mcts(ref):
    """Throughput-mode two_phase with the throughput mcts_solve refill
    (mig_two_phase_parallel_mcts; BASELINE config #3's greedy -> GA -> MCTS pipeline with a
    fixed Philox seed): the reference's operators, fast_algo and rollout primitives under the
    product's Philox draw rule."""
    res = {}
    ps = S.profiles()
    tw, sv6 = S.random_workload(6, 77)
    p3, g3 = S.gen(24, 8.7)
    cases = [("slos_day", ps, S.fixture_services("slos_day", ps), dict(seed=24, max_rounds=4),
              dict(n_rollouts=64, topk=10)),
             ("rand6", tw, sv6, dict(seed=9, max_rounds=5, erase_fraction=0.25), dict(n_rollouts=128, topk=4)),
             ("slos_24", ps, S.fixture_services("slos_24", ps), dict(seed=24, max_rounds=3),
              dict(n_rollouts=256, topk=10, batch=128)),
             ("gen24_8.7", p3, g3, dict(seed=4242, max_rounds=2), dict(n_rollouts=256, topk=10))]
    only = os.environ.get("GOLDEN_ONLY")
    for name, p, sv, kw, slow in cases:
        if only and name not in only.split(","):
            continue
        t = time.time()
        logs = []
        dep = mp.two_phase_parallel(sv, p, mp.PartitionRuleSet.defaults(), mp.GaParams(time_budget_s=1e9, **kw),
                                    log=lambda l: logs.append([l.round, l.best_gpus, l.best_slack.hex(), l.improved]),
                                    backend=ref, slow=mp.RolloutParams(**slow))
        res[name] = {"store": store_name(p), "services": svc_json(sv), "params": kw, "slow": slow,
                     "plan": S.plan_key([g.config for g in dep.gpus]), "log": logs,
                     "ref_wall_s": round(time.time() - t, 3)}
        print(f"ga_parallel_mcts {name}: {len(dep.gpus)} GPUs ({time.time() - t:.1f}s)", flush=True)
    return res


SECTIONS = {"ga_parallel_mcts": gen_ga_parallel_mcts, "ga_big": gen_ga_big, "mcts_big": gen_mcts_big, "greedy_prefix": gen_greedy_prefix,
            "pools_big": gen_pools_big, "rollouts_big": gen_rollouts_big,
"baseline": gen_baseline, "brute_force": gen_brute_force, "greedy": gen_greedy, "mcts": gen_mcts, "ga": gen_ga, "topk": gen_topk, "partitions": gen_partitions,
            "greedy_big": gen_greedy_big, "rollouts": gen_rollouts, "ga_parallel": gen_ga_parallel}


def main(argv):
    ref = S.ref_backend()
    if ref is None:
        sys.exit("oracle/_ref/libmigref.so not built (make -C oracle ref)")
    for sec in argv or list(SECTIONS):
        t = time.time()
        data = SECTIONS[sec](ref)
        path = os.path.join(S.GOLDEN, f"{sec}.json")
        if os.environ.get("GOLDEN_MERGE") and os.path.exists(path):  # regenerate some entries only
            with open(path) as f:
                data = {**json.load(f), **data}
        with open(path, "w") as f:
            json.dump(data, f, separators=(",", ":"))
        print(f"wrote {sec}.json in {time.time() - t:.1f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
