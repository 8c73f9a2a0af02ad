"""`migplan` command-line re-host on the B200 planner.

    python -m paper_2109_11067_b200.cli optimize --mode fast --slos S.json --profiles P.json -o dep.json
    python -m paper_2109_11067_b200.cli lowerbound --slos S.json --profiles P.json
    python -m paper_2109_11067_b200.cli oracle --slos S.json --profiles P.json --cap 3 -o dep.json
    python -m paper_2109_11067_b200.cli baseline --kind 7of7|7x1|mix --slos S.json --profiles P.json -o dep.json
    python -m paper_2109_11067_b200.cli gen-workload --n 24 --seed 7 --profiles P.json -o slos.json
    python -m paper_2109_11067_b200.cli enumerate-partitions [--rules R.json] [-o parts.json]

Restates the reference CLI's `optimize` / `lowerbound` / `oracle` / `baseline` /
`gen-workload` / `enumerate-partitions` (proj/tools/migplan.cpp:88-147, 159-215, 244-251,
262-345, 382-397) over the C-ABI:
  - output files are `json.dump(indent=2)` with sorted keys + "\\n" — the byte layout of
    nlohmann's `dump(2)` (write_json_file, io.hpp:44-48; std::map keys are sorted);
  - trace lines go to stdout as compact sorted-key JSON (migplan.cpp:99-137), numbers through
    %.9g (out_num, io.hpp:22-26);
  - every output gets `<out>.manifest.json` with command, flags, fnv1a64 input digests,
    tool_version and wall_ms (write_manifest, migplan.cpp:32-51);
  - exit codes: 2 for SchemaError / usage, 1 for PlanningError (migplan.cpp:414-426).
Modes: fast | mcts | full as the reference (parity mode: identical plans), plus the
throughput modes mcts-parallel (root-parallel rollouts, --rollouts) and full-parallel
(device GA).
"""
from __future__ import annotations

import argparse
import json
import sys
import time

from . import migplan as mp

TOOL_VERSION = "0.1.0"  # migplan.cpp:20
_BACKEND = None  # the product (B200); tests may point --backend at a CPU checker library


def out_num(v: float) -> float:  # io.hpp:22-26
    return float("%.9g" % v)


def fnv1a64(data: bytes) -> int:  # util.hpp:66-73
    h = 1469598103934665603
    for c in data:
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def dump_file(path: str, obj) -> None:  # write_json_file, io.hpp:44-48
    with open(path, "w", newline="\n") as f:
        f.write(json.dumps(obj, indent=2, sort_keys=True, ensure_ascii=False) + "\n")


def dump_line(obj) -> None:
    sys.stdout.write(json.dumps(obj, separators=(",", ":"), sort_keys=True, ensure_ascii=False) + "\n")


def load_rules(path: str) -> mp.PartitionRuleSet:  # io.hpp:212-241
    j = mp._load_json(path)
    if not isinstance(j, dict):
        raise mp.SchemaError(f"{path}: expected an object")
    for k in j:
        if k not in ("slot_positions", "memory_weight", "hard_exclusions", "memory_budget"):
            raise mp.SchemaError(f"{path}: unknown field '{k}'")
    r = mp.PartitionRuleSet.defaults()
    if "slot_positions" in j:
        r.slot_positions = {}
        for size_str, slots in j["slot_positions"].items():
            size = int(size_str)
            if not mp.valid_slices(size):
                raise mp.SchemaError(f"{path}: invalid size '{size_str}'")
            if not isinstance(slots, list):
                raise mp.SchemaError(f"{path}: slot_positions values must be arrays")
            r.slot_positions[size] = sorted(int(s) for s in slots)
    if "memory_weight" in j:
        r.memory_weight = {int(k): int(v) for k, v in j["memory_weight"].items()}
    if "hard_exclusions" in j:
        r.hard_exclusions = set()
        for pair in j["hard_exclusions"]:
            if not isinstance(pair, list) or len(pair) != 2:
                raise mp.SchemaError(f"{path}: hard_exclusions entries must be [size, size]")
            a, b = int(pair[0]), int(pair[1])
            r.hard_exclusions.add((min(a, b), max(a, b)))
    if "memory_budget" in j:
        r.memory_budget = int(j["memory_budget"])
    return r


class Manifest:  # ManifestInfo + write_manifest, migplan.cpp:23-51
    def __init__(self, command: str, flags: dict, inputs: list):
        self.command, self.flags, self.inputs = command, flags, inputs
        self.t0 = time.perf_counter()

    def write(self, out_path: str) -> None:
        inputs = {}
        for p in self.inputs:
            with open(p, "rb") as f:
                inputs[p] = "fnv1a64:%016x" % fnv1a64(f.read())
        dump_file(out_path + ".manifest.json", {"command": self.command, "flags": self.flags, "inputs": inputs,
                                                "tool_version": TOOL_VERSION,
                                                "wall_ms": out_num(1e3 * (time.perf_counter() - self.t0))})


def _instances_json(cfg: mp.GpuConfig):
    return mp.deployment_to_json(mp.Deployment([mp.DeployedGpu("pick", cfg)]))["gpus"][0]["instances"]


def cmd_optimize(a, manifest: Manifest) -> int:  # migplan.cpp:88-147
    profiles = mp.load_profiles(a.profiles)
    services = mp.load_services(a.slos, profiles)
    rules = load_rules(a.rules) if a.rules else mp.PartitionRuleSet.defaults()
    stochastic = ("mcts", "full", "mcts-parallel", "full-parallel")
    if a.mode in stochastic and a.seed is None:
        raise mp.SchemaError("--seed is required for stochastic modes (mcts, full)")
    z = mp.zero_completion(len(services))
    if a.mode == "fast":
        ctx = mp.make_plan_context(services, profiles, rules, backend=_BACKEND, device=a.device)

        def trace(it, cand, s, comp):
            if not a.quiet:
                dump_line({"iter": it, "score": out_num(s), "config": _instances_json(cand.config),
                           "completion": [out_num(c) for c in comp]})

        dep = mp.make_deployment(mp.fast_algo(z, ctx, trace=trace))
    elif a.mode == "mcts":
        ctx = mp.make_plan_context(services, profiles, rules, backend=_BACKEND, device=a.device)

        def mtrace(it, depth, est, best):
            if not a.quiet:
                dump_line({"iter": it, "depth": depth, "rollout_estimate": est, "best_len": best})

        dep = mp.make_deployment(mp.mcts_solve(z, ctx, mp.MctsParams(budget_iters=a.budget_iters, topk=a.topk),
                                               a.seed, trace=mtrace))
    elif a.mode in ("full", "full-parallel"):
        params = mp.GaParams(seed=a.seed, time_budget_s=a.time_budget, max_rounds=a.ga_rounds,
                             population=a.population, erase_fraction=a.erase_fraction, workers=a.workers,
                             slow=mp.MctsParams(budget_iters=a.budget_iters, topk=a.topk))

        def log(r):
            if not a.quiet:
                dump_line({"round": r.round, "best_gpus": r.best_gpus, "best_slack": out_num(r.best_slack),
                           "improved": r.improved})

        ctx = mp.make_plan_context(services, profiles, rules, backend=_BACKEND, device=a.device)
        fn = mp.two_phase if a.mode == "full" else mp.two_phase_parallel
        dep = fn(services, profiles, rules, params, log=log, ctx=ctx)
    elif a.mode == "mcts-parallel":
        ctx = mp.make_plan_context(services, profiles, rules, backend=_BACKEND, device=a.device)
        plan, res = mp.mcts_solve_parallel(z, ctx, mp.RolloutParams(n_rollouts=a.rollouts, topk=a.topk, seed=a.seed))
        if not a.quiet:
            dump_line({"rollouts": a.rollouts, "best_rollout": res.best_len, "completed": res.completed,
                       "keys": res.keys, "device_ms": out_num(res.device_ms)})
        dep = mp.make_deployment(plan)
    else:
        raise mp.SchemaError(f"unknown mode '{a.mode}' (expected fast, mcts, or full)")
    mp.validate_deployment(dep, services, profiles, rules, backend=_BACKEND)
    dump_file(a.output, mp.deployment_to_json(dep))
    manifest.write(a.output)
    return 0


def cmd_lowerbound(a, manifest: Manifest) -> int:  # lower_bound, bench.hpp:93-108
    profiles = mp.load_profiles(a.profiles)
    services = mp.load_services(a.slos, profiles)
    out = {"lower_bound": mp.lower_bound(services, profiles)}
    if a.output:
        dump_file(a.output, out)
        manifest.write(a.output)
    else:
        sys.stdout.write(json.dumps(out, indent=2, sort_keys=True) + "\n")
    return 0


def cmd_oracle(a, manifest: Manifest) -> int:  # migplan.cpp:382-397 (brute_force_optimum on the device)
    profiles = mp.load_profiles(a.profiles)
    services = mp.load_services(a.slos, profiles)
    rules = load_rules(a.rules) if a.rules else mp.PartitionRuleSet.defaults()
    dep = mp.brute_force_optimum(services, profiles, rules, a.cap, backend=_BACKEND, device=a.device)
    if dep is None:
        sys.stderr.write(f"no deployment within {a.cap} GPUs\n")
        return 1
    dump_file(a.output, mp.deployment_to_json(dep))
    manifest.write(a.output)
    return 0


def cmd_baseline(a, manifest: Manifest) -> int:  # migplan.cpp:294-309
    profiles = mp.load_profiles(a.profiles)
    services = mp.load_services(a.slos, profiles)
    if a.kind not in mp.BASELINE_KINDS:
        raise mp.SchemaError(f"unknown baseline kind '{a.kind}' (expected 7of7, 7x1, or mix)")
    dep = mp.baseline(a.kind, services, profiles, backend=_BACKEND)
    dump_file(a.output, mp.deployment_to_json(dep))
    manifest.write(a.output)
    return 0


def cmd_gen_workload(a, manifest: Manifest) -> int:  # migplan.cpp:324-345 (services_to_json, io.hpp:153-161)
    if a.seed is None:
        raise mp.SchemaError("--seed is required for gen-workload")
    if a.dist not in ("normal", "lognormal"):
        raise mp.SchemaError(f"unknown distribution '{a.dist}'")
    normal = a.dist == "normal"
    mu = a.mu if a.mu >= 0.0 else (5000.0 if normal else 8.0)
    sigma = a.sigma if a.sigma >= 0.0 else (2000.0 if normal else 0.6)
    profiles = mp.load_profiles(a.profiles)
    sv = mp.gen_workload(a.n, not normal, mu, sigma, a.latency_ms, a.seed, profiles, backend=_BACKEND)
    dump_file(a.output, {"services": [{"id": s.service_id, "model": s.model_name,
                                       "required_rps": out_num(s.required_rps),
                                       "max_p90_ms": out_num(s.max_p90_ms)} for s in sv]})
    manifest.write(a.output)
    return 0


def cmd_enumerate(a, manifest: Manifest) -> int:  # migplan.cpp:56-64
    rules = load_rules(a.rules) if a.rules else mp.PartitionRuleSet.defaults()
    parts = mp.enumerate_maximal_partitions(rules, backend=_BACKEND)
    j = {"count": len(parts),  # partitions_to_json, io.hpp:371-383
         "partitions": [{"sizes": [p.slices for p in lp.placements],
                         "placements": [{"size": p.slices, "slot": p.start_slot} for p in lp.placements],
                         "maximal": lp.maximal} for lp in parts]}
    if a.output:
        dump_file(a.output, j)
        manifest.write(a.output)
    else:
        sys.stdout.write(json.dumps(j, indent=2, sort_keys=True) + "\n")
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="migplan", description="MIG-SERVING deployment planner (B200)")
    sub = ap.add_subparsers(dest="command", required=True)
    o = sub.add_parser("optimize", help="Compute a GPU-minimizing deployment")
    o.add_argument("--mode", required=True,
                   help="fast | mcts | full (reference semantics) | mcts-parallel | full-parallel")
    o.add_argument("--slos", required=True)
    o.add_argument("--profiles", required=True)
    o.add_argument("--rules", default="")
    o.add_argument("-o", "--output", required=True)
    o.add_argument("--seed", type=int, default=None)
    o.add_argument("--budget-iters", type=int, default=200)
    o.add_argument("--topk", type=int, default=10)
    o.add_argument("--time-budget", type=float, default=60.0)
    o.add_argument("--ga-rounds", type=int, default=1 << 30)
    o.add_argument("--population", type=int, default=16)
    o.add_argument("--erase-fraction", type=float, default=0.10)
    o.add_argument("--workers", type=int, default=1)
    o.add_argument("--rollouts", type=int, default=1 << 16, help="mcts-parallel: root-parallel rollouts")
    o.add_argument("--device", type=int, default=0)
    o.add_argument("--quiet", action="store_true")
    o.add_argument("--backend", default="", help=argparse.SUPPRESS)  # tests: a CPU checker library
    lb = sub.add_parser("lowerbound", help="GPU lower bound ignoring partition rules")
    lb.add_argument("--slos", required=True)
    lb.add_argument("--profiles", required=True)
    lb.add_argument("-o", "--output", default="")
    bl = sub.add_parser("baseline", help="Static-partition baseline deployments")
    bl.add_argument("--kind", required=True, help="7of7 | 7x1 | mix")
    bl.add_argument("--slos", required=True)
    bl.add_argument("--profiles", required=True)
    bl.add_argument("-o", "--output", required=True)
    bl.add_argument("--backend", default="", help=argparse.SUPPRESS)
    gw = sub.add_parser("gen-workload", help="Generate a random workload SLO file")
    gw.add_argument("--dist", default="lognormal", help="normal | lognormal")
    gw.add_argument("--n", type=int, default=24)
    gw.add_argument("--mu", type=float, default=-1.0)
    gw.add_argument("--sigma", type=float, default=-1.0)
    gw.add_argument("--latency-ms", type=float, default=100.0)
    gw.add_argument("--seed", type=int, default=None)
    gw.add_argument("--profiles", required=True)
    gw.add_argument("-o", "--output", required=True)
    gw.add_argument("--backend", default="", help=argparse.SUPPRESS)
    orc = sub.add_parser("oracle", help="Brute-force minimum-GPU deployment (small instances)")
    orc.add_argument("--slos", required=True)
    orc.add_argument("--profiles", required=True)
    orc.add_argument("--rules", default="")
    orc.add_argument("--cap", type=int, default=3, help="Maximum GPUs to search")
    orc.add_argument("-o", "--output", required=True)
    orc.add_argument("--device", type=int, default=0)
    orc.add_argument("--backend", default="", help=argparse.SUPPRESS)
    en = sub.add_parser("enumerate-partitions", help="Print the derived legal partition table")
    en.add_argument("--rules", default="")
    en.add_argument("-o", "--output", default="")
    return ap


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    try:
        a = build_parser().parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    # flags as given on the command line (record_flag, migplan.cpp:268-275)
    flags, i = {}, 1
    while i < len(argv):
        tok = argv[i]
        if tok.startswith("-"):
            name = "--output" if tok == "-o" else tok
            if i + 1 < len(argv) and not argv[i + 1].startswith("--") and name != "--quiet":
                flags[name] = argv[i + 1]
                i += 2
                continue
            flags[name] = "true"
        i += 1
    global _BACKEND
    if getattr(a, "backend", ""):
        _BACKEND = mp.Backend.load(a.backend)
    flags.pop("--backend", None)
    inputs = [x for x in (getattr(a, "slos", None), getattr(a, "profiles", None), getattr(a, "rules", None)) if x]
    manifest = Manifest(a.command, flags, inputs)
    try:
        if a.command == "optimize":
            return cmd_optimize(a, manifest)
        if a.command == "lowerbound":
            return cmd_lowerbound(a, manifest)
        if a.command == "oracle":
            return cmd_oracle(a, manifest)
        if a.command == "baseline":
            return cmd_baseline(a, manifest)
        if a.command == "gen-workload":
            return cmd_gen_workload(a, manifest)
        return cmd_enumerate(a, manifest)
    except mp.SchemaError as e:
        sys.stderr.write(f"error: {e}\n")
        return 2
    except (mp.PlanningError, mp.ExecutionError) as e:
        sys.stderr.write(f"error: {e}\n")
        return 1
    except Exception as e:  # noqa: BLE001 - migplan.cpp:423-425
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
