"""bench.py — MIG-SERVING optimizer hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl product|reference] [--workload NAME]

Metric: candidate configs scored per second (BASELINE.json "candidate configs scored/sec
and end-to-end plan time ... GPUs used"): every greedy step counts its whole working set
(greedy.hpp:123-134), every top-K call its candidate set (mcts.hpp:59-67) — the same count
for every implementation (the CPU restatement counts identical numbers).

Headline workload (N = 1): BASELINE config #5, the largest single-GPU configuration —
gen_workload(128, lognormal mu=8.0, sigma=0.6, seed 4242) on fixtures/profiles.json, one
`fast_algo` plan from zero completion per STEP (base pool 388,288 rows; 128 extension
events grow the working set past 1.3e9 rows; ~1.7e12 rows scored per plan; ~3,000 GPUs).

value  : rows scored / device time, context (device tables + base pool) resident, CUDA events
         bracketing each step after torch.cuda.synchronize(); the working set (>10 GB) is far
         larger than L2 and L2 is also flushed (512 MiB write) between steps; max over ranks.
e2e    : the same metric through the C-ABI from HOST inputs: each step builds the context from
         host profiles/services (table upload, base-pool enumeration), plans, and returns the
         plan to host memory.  Per-call device resources are pooled per process;
         `e2e.cold_ms` is one step after mig_device_cache_release (every arena, stream and
         pinned buffer allocated inside the timed step).
N > 1  : torchrun, one process per GPU.  The config space is sharded: rank r
         keeps 1/N of every working set (base supports dealt by row count, extension supports
         by (colex rank + size + event) mod N) and the persistent greedy kernels exchange each
         step's winner through peer-memory boards (CUDA IPC handles all-gathered once over
         NCCL, dist.shard_context).  Total work is fixed (scaling "strong"); value = all ranks'
         rows / max-over-ranks time; the plan must be identical at every N.
--impl reference : the reference's own CPU implementation (oracle/_ref: the unmodified
         reference headers compiled from /root/reference) on this host, rank 0 only, each step
         a bounded sample of the same workload (config #5: the reference's fast_algo run for
         its first S steps on a resident context — the full plan is not completable on a CPU,
         SURVEY §8d).
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "candidate configs scored/sec"
WORKLOADS = {
    "gen128_8.0_greedy": "BASELINE config #5: gen_workload(128, lognormal mu=8.0, sigma=0.6, seed 4242), "
                         "fast_algo from zero completion (stress greedy sweep)",
    "slos24_ga10": "BASELINE config #2: fixtures/slos_24.json (24 svc), fast_algo seed + two_phase GA "
                   "(seed 24, 10 rounds, P=16, MCTS budget 48, time budget off)",
    "gen24_8.7_ga2": "BASELINE config #3: gen_workload(24, mu=8.7, seed 4242), fast_algo seed + two_phase GA "
                     "(seed 4242, 2 rounds, P=16, MCTS budget 48)",
    "gen48_7.0_greedy": "BASELINE config #4's workload: gen_workload(48, mu=7.0, seed 4242), fast_algo",
    "gen24_8.7_greedy": "gen_workload(24, mu=8.7, seed 4242): fast_algo (~974 GPUs)",
    "slos24_greedy": "fixtures/slos_24.json (24 svc): fast_algo from zero completion",
}
# golden plan digests (tests/golden, generated from the reference): bench lines say whether
# the plan they timed is the reference's
GA_GOLDEN = {"slos24_ga10": "slos_24_r10", "gen24_8.7_ga2": "gen24_8.7_r2"}
L2_NOTE = "working set > L2 (126 MB) and L2 flushed (512 MiB write) between steps"


def load_workload(name):
    import support as S

    ps = S.profiles()
    if name.startswith("slos24"):
        return ps, S.fixture_services("slos_24", ps)
    for tag, (n, mu) in {"gen24_8.7": (24, 8.7), "gen48_7.0": (48, 7.0), "gen128_8.0": (128, 8.0)}.items():
        if name.startswith(tag):
            return S.gen(n, mu)
    raise SystemExit(f"unknown workload {name}")


def ga_params(name, workers, seed_offset=0):
    from paper_2109_11067_b200 import migplan as mp

    rounds, seed = (10, 24) if name == "slos24_ga10" else (2, 4242)
    return mp.GaParams(seed=seed + seed_offset, max_rounds=rounds, time_budget_s=1e9, population=16,
                       workers=workers, slow=mp.MctsParams(budget_iters=48))


def is_ga(name):
    return "_ga" in name


def run_step(mp, name, ctx, sv, ps, workers):
    """One optimizer pass on a resident context; returns the plan (list of GpuConfig)."""
    if is_ga(name):
        dep = mp.two_phase(sv, ps, mp.PartitionRuleSet.defaults(), ga_params(name, workers), ctx=ctx)
        return [g.config for g in dep.gpus]
    return mp.fast_algo(mp.zero_completion(len(sv)), ctx)


def golden_check(name, plan):
    """Is the timed plan the reference's?  Full plans: the golden digest; config #5: the
    reference's first steps (greedy_prefix.json) — the full n=128 plan is not CPU-completable."""
    import support as S

    try:
        if name in GA_GOLDEN:
            g = S.load_golden("ga_big.json")[GA_GOLDEN[name]]
            return {"golden": f"ga_big.json:{GA_GOLDEN[name]}", "match": S.plan_sha(plan) == g["plan_sha"]}
        if name == "gen128_8.0_greedy":
            g = S.load_golden("greedy_prefix.json")["gen128_8.0"]
            return {"golden": f"greedy_prefix.json (reference's first {g['steps']} steps)",
                    "match": S.plan_key(plan[:g["steps"]]) == g["plan"]}
        key = {"gen48_7.0_greedy": ("greedy_big.json", "gen48_7.0"), "gen24_8.7_greedy": ("greedy.json", "gen24_8.7"),
               "slos24_greedy": ("greedy.json", "slos_24")}.get(name)
        if key:
            g = S.load_golden(key[0])[key[1]]
            return {"golden": f"{key[0]}:{key[1]}", "match": S.plan_key(plan) == g["plan"]}
    except (OSError, KeyError):
        pass
    return {"golden": None, "match": None}


class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region (NVML, ~20 ms)."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def _run(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
            while not self._stop.is_set():
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM), mx, [bool(r & b) for b in bits]))
                self._stop.wait(0.02)
            return
        except Exception:
            pass
        fields = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={fields}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                v = [x.strip() for x in out.stdout.strip().split(",")]
                self.samples.append((float(v[0]), float(v[1]), [x == "Active" for x in v[2:6]]))
            except Exception:
                pass
            self._stop.wait(0.2)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2][i]})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons, "samples": len(self.samples)}


READ_STREAM_GBS = 7383.0  # profiles/r02a_readbw.txt: read-only 16-B loads, 512 x 592 CTAs, B200


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# committed `ncu --set full` captures (tools/ncu_summary.py) per kernel and workload
TRAFFIC_PROFILES = {
    ("greedy_kernel", "gen128_8.0_greedy"): "r02t_greedy_gen128_ncu.json",
    ("mcts_kernel", "slos24_ga10"): "r02g_mcts_ga_ncu.json",
    ("greedy_kernel", "slos24_ga10"): "r02g_greedy_slos24_ncu.json",
}


def profile_traffic(kernel, workload):
    """dram__bytes_read + dram__bytes_write per launch of `kernel` from the committed ncu
    capture of the same workload (cold-cache, serialised: a cross-check, not timing)."""
    name = TRAFFIC_PROFILES.get((kernel, workload))
    if not name or not os.path.exists(os.path.join(ROOT, "profiles", name)):
        return None, None
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            d = json.load(f)
        k = next(x for x in d["kernels"] if kernel in x["kernel"])
        return k.get("dram_bytes_per_launch"), name
    except Exception:
        return None, None


def host_info():
    model = platform.processor()
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


# ------------------------------------------------------------------ reference (CPU) samples

def ref_backend():
    import support as S

    ref = S.ref_backend()
    if ref is not None:
        return ref, "reference"
    return S.oracle_backend(), "port"


def cpu_prefix_steps():
    """Config #5 CPU sample: the reference's first S greedy steps, all over the base pool
    (S <= its first extension step, greedy_prefix.json), ~2-3 s of one core."""
    import support as S

    try:
        e = S.load_golden("greedy_prefix.json")["gen128_8.0"]["first_ext_step"]
        return max(1, min(e + 1, 120))
    except (OSError, KeyError):
        return 32


class RefSampler:
    """One bounded step of the reference's CPU implementation of `name` on a resident context."""

    def __init__(self, name, workers):
        import support as S
        from support import mp

        self.mp, self.S, self.name, self.workers = mp, S, name, workers
        self.ps, self.sv = load_workload(name)
        self.ref, self.kind = ref_backend()
        t = time.perf_counter()
        self.ctx = mp.make_plan_context(self.sv, self.ps, mp.PartitionRuleSet.defaults(), backend=self.ref)
        self.build_s = time.perf_counter() - t
        self.cores = workers if is_ga(name) else 1
        self.rows = None
        self.plan = None
        if name == "gen128_8.0_greedy":
            self.steps = cpu_prefix_steps()
            self.rows = self.steps * len(self.ctx.pool)  # steps before the first extension scan the base pool
            self.sample = (f"the reference's fast_algo for its first {self.steps} step(s) — every step before its "
                           f"first extension event (greedy_prefix.json), {len(self.ctx.pool)} base rows each, "
                           f"including the call's WorkingSet set-up — on a resident context (base pool build "
                           f"{self.build_s:.2f} s, untimed); 1 core (fast_algo is single-threaded).  Its most "
                           f"favourable regime: the reference's first 3 steps, which include its first extensions "
                           f"(~24.9 M rows each), took 825 s on one core of the build container "
                           f"(tests/golden/greedy_prefix.json ref_wall_s)")
        else:
            # rows per step: counted by the CPU restatement on the same call sequence (untimed)
            orc = S.oracle_backend()
            octx = mp.make_plan_context(self.sv, self.ps, mp.PartitionRuleSet.defaults(), backend=orc)
            run_step(mp, name, octx, self.sv, self.ps, workers)
            self.rows = octx.stats()["rows_scored"]
            self.sample = (f"1 full step of {name} on a resident context, {self.cores} thread(s)"
                           + (" (GA workers)" if is_ga(name) else ""))

    def step(self):
        import ctypes as C

        mp = self.mp
        t = time.perf_counter()
        if self.name == "gen128_8.0_greedy":
            buf, n = self.ctx._comp(mp.zero_completion(len(self.sv)))
            steps, ext = C.c_int32(), C.c_int32()
            trace = []

            def _tr(_u, it, cand, s, cp, nn):
                trace.append(self.ctx._cand_from_c(cand.contents).config)

            from paper_2109_11067_b200 import abi

            cb = abi.GREEDY_TRACE(_tr)
            self.ref.check(self.ref.lib.mig_ref_fast_algo_prefix(self.ctx._p, buf, n, self.steps, -1, cb, None,
                                                                  C.byref(steps), C.byref(ext)))
            self.plan = trace
        else:
            self.plan = run_step(mp, self.name, self.ctx, self.sv, self.ps, self.workers)
        return time.perf_counter() - t


def reference_arm(args):
    """--impl reference: the reference's CPU implementation, bounded per-step sample."""
    import support as S

    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    workers = min(os.cpu_count() or 1, 8)
    rs = RefSampler(args.workload, workers)
    heavy = is_ga(args.workload)
    warm = min(args.warmup, 1) if heavy else min(args.warmup, 5)
    steps = max(1, min(args.steps, 3)) if heavy else max(1, min(args.steps, 30))
    for _ in range(warm):
        rs.step()
    times = [rs.step() for _ in range(steps)]
    total = sum(times)
    value = rs.rows * steps / total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "configs/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": warm, "ms_per_step": 1e3 * total / steps, "higher_is_better": True,
            "scaling": "strong" if not heavy else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "description": WORKLOADS[args.workload], "l2": L2_NOTE},
            "result": {"rows_per_step": rs.rows, "plan_sha": S.plan_sha(rs.plan), "gpus_in_plan": len(rs.plan),
                       "complete_plan": args.workload != "gen128_8.0_greedy", "context_build_s": rs.build_s},
            "cpu_baseline": {"value": value, "unit": "configs/s", "cores": rs.cores, "kind": rs.kind,
                             "sample": rs.sample, **host_info()},
            "e2e": {"value": value, "unit": "configs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ product

def timed(fn, flush, torch):
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    torch.cuda.synchronize()  # the product launches on its own streams: wait for all of them
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def secondary_ga(mp, local, flush, torch, steps, workers):
    """Config #2 (slos_24 two_phase, 10 rounds) on the product beside the reference's own run:
    the plan is compared with the reference's golden (ga_big.json slos_24_r10)."""
    import support as S

    name = "slos24_ga10"
    ps, sv = load_workload(name)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), device=local)
    for _ in range(2):
        plan = run_step(mp, name, ctx, sv, ps, workers)
    ctx.reset_stats()
    ms = []
    for _ in range(steps):
        plan, t = timed(lambda: run_step(mp, name, ctx, sv, ps, workers), flush, torch)
        ms.append(t)
    st = ctx.stats()
    e2e = []
    for _ in range(steps):
        def e2e_step():
            c2 = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), device=local)
            p = run_step(mp, name, c2, sv, ps, workers)
            c2.close()
            return p
        _, t = timed(e2e_step, flush, torch)
        e2e.append(t)
    rows = st["rows_scored"] / steps
    out = {"workload": name, "description": WORKLOADS[name], "steps": steps, "ms_per_step": statistics.mean(ms),
           "value": rows / (statistics.mean(ms) / 1e3), "unit": "configs/s", "rows_per_step": rows,
           "e2e": {"value": rows / (statistics.mean(e2e) / 1e3), "ms_per_step": statistics.mean(e2e)},
           "gpus_in_plan": len(plan), "plan_sha": S.plan_sha(plan), "parity": golden_check(name, plan),
           "breakdown": {"greedy_ms": st["greedy_ms"] / steps, "mcts_ms": st["mcts_ms"] / steps,
                         "topk_ms": st["topk_ms"] / steps, "launches_per_step": st["kernel_launches"] / steps}}
    ctx.close()
    try:  # the reference's own two_phase on this host, same seed and parameters (one run)
        rs = RefSampler(name, min(os.cpu_count() or 1, 8))
        dt = rs.step()
        out["reference"] = {"value": rs.rows / dt, "ms_per_step": 1e3 * dt, "cores": rs.cores, "kind": rs.kind,
                            "plan_sha": S.plan_sha(rs.plan), "gpus_in_plan": len(rs.plan)}
        out["e2e_ratio_vs_reference"] = dt * 1e3 / out["e2e"]["ms_per_step"]
    except Exception as e:  # pragma: no cover - reported, not fatal
        out["reference"] = {"error": repr(e)}
    return out


def extra_measurements(mp, local):
    """Device-timed evidence for the other BASELINE configs: config #4 (1e6 root-parallel
    rollouts; parity-mode MCTS with 2,000 iterations, ms/iteration) and the device GA."""
    import torch

    import support as S

    out = {}
    try:
        ps, sv = S.gen(48, 7.0)
        ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), device=local)
        z = mp.zero_completion(len(sv))
        greedy = mp.fast_algo(z, ctx)
        prm = mp.RolloutParams(n_rollouts=1_000_000, seed=1, max_depth=2 * len(greedy))
        mp.rollouts(z, ctx, prm)
        r = mp.rollouts(z, ctx, prm)
        out["rollouts"] = {
            "workload": "gen48_7.0, 1e6 root-parallel rollouts (BASELINE config #4), Philox seed 1",
            "device_ms": r.device_ms, "rollouts_per_s": 1e6 / (r.device_ms / 1e3),
            "rollout_steps_per_s": r.steps / (r.device_ms / 1e3), "steps": r.steps, "keys": r.keys,
            "best_rollout_gpus": r.best_len, "greedy_gpus": len(greedy)}
        ctx.reset_stats()
        t0 = time.perf_counter()
        plan = mp.mcts_solve(z, ctx, mp.MctsParams(budget_iters=2000), 1)
        wall = time.perf_counter() - t0
        st = ctx.stats()
        out["mcts_parity"] = {
            "workload": "gen48_7.0 mcts_solve (parity mode: the reference's mt19937_64 stream), 2000 iterations, seed 1",
            "wall_ms": 1e3 * wall, "ms_per_iteration": 1e3 * wall / 2000, "gpus_in_plan": len(plan),
            "greedy_gpus": len(greedy), "mcts_kernel_ms": st["mcts_ms"], "greedy_ms": st["greedy_ms"],
            "reference_ms_per_iteration": "~95 (SURVEY §6, one core, measured at 2,000 iterations)"}
        ctx.close()
    except Exception as e:  # pragma: no cover
        out["config4"] = {"error": repr(e)}
    try:  # config #3: greedy -> GA -> MCTS, throughput mode (Philox), against the reference's GA
        import support as S2

        ps, sv = S.gen(24, 8.7)
        ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), device=local)
        slow = mp.RolloutParams(n_rollouts=1024, topk=10)
        res3 = {"workload": "gen24_8.7 (BASELINE config #3): two_phase_parallel_mcts — device population, Philox "
                            "seed 4242, refill = shorter of greedy and best of 1024 root-parallel rollouts",
                "greedy_gpus": len(mp.fast_algo(mp.zero_completion(len(sv)), ctx))}
        warm = mp.GaParams(seed=4242, max_rounds=2, time_budget_s=1e9, stall_rounds=1 << 30)
        mp.two_phase_parallel(sv, ps, mp.PartitionRuleSet.defaults(), warm, ctx=ctx, slow=slow)  # first-use set-up
        for rounds in (2, 10, 50):
            prm = mp.GaParams(seed=4242, max_rounds=rounds, time_budget_s=1e9, stall_rounds=1 << 30)
            ctx.reset_stats()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dep = mp.two_phase_parallel(sv, ps, mp.PartitionRuleSet.defaults(), prm, ctx=ctx, slow=slow)
            st3 = ctx.stats()
            res3[f"rounds_{rounds}"] = {"gpus_in_plan": len(dep.gpus), "wall_ms": 1e3 * (time.perf_counter() - t0),
                                        "device_ms": {"greedy": st3["greedy_ms"], "rollouts": st3["rollout_ms"]},
                                        "rollout_calls": st3["rollout_calls"], "rollout_steps": st3["rollout_steps"],
                                        "launches": st3["kernel_launches"]}
        t0 = time.perf_counter()  # the parity-mode two_phase (reference RNG) of the same config, 2 rounds
        dep = mp.two_phase(sv, ps, mp.PartitionRuleSet.defaults(), ga_params("gen24_8.7_ga2", 8), ctx=ctx)
        res3["parity_two_phase_2_rounds"] = {"gpus_in_plan": len(dep.gpus), "wall_ms": 1e3 * (time.perf_counter() - t0),
                                             "parity": golden_check("gen24_8.7_ga2", [g.config for g in dep.gpus])}
        try:
            ga = S2.load_golden("ga_big.json")
            res3["reference_two_phase"] = {
                k: {"gpus_in_plan": len(ga[k]["plan"]), "wall_s_build_container": ga[k]["ref_wall_s"],
                    "workers": 8} for k in ("gen24_8.7_r2", "gen24_8.7_r10") if k in ga}
        except (OSError, KeyError):
            pass
        out["config3"] = res3
        ctx.close()
    except Exception as e:  # pragma: no cover
        out["config3"] = {"error": repr(e)}
    try:  # throughput-mode GA on config #2
        ps = S.profiles()
        sv = S.fixture_services("slos_24", ps)
        ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), device=local)
        prm = mp.GaParams(seed=24, max_rounds=10, time_budget_s=1e9)
        mp.two_phase_parallel(sv, ps, mp.PartitionRuleSet.defaults(), prm, ctx=ctx)
        t0 = time.perf_counter()
        dep = mp.two_phase_parallel(sv, ps, mp.PartitionRuleSet.defaults(), prm, ctx=ctx)
        out["ga_parallel"] = {"workload": "slos24 two_phase_parallel: 10 rounds, P=16, Philox seed 24",
                              "wall_ms": 1e3 * (time.perf_counter() - t0), "gpus_in_plan": len(dep.gpus)}
        ctx.close()
    except Exception as e:  # pragma: no cover
        out["ga_parallel"] = {"error": repr(e)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--workload", default="gen128_8.0_greedy", choices=sorted(WORKLOADS))
    ap.add_argument("--workers", type=int, default=8, help="GA worker threads per rank (product)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the config #2 GA object")
    ap.add_argument("--no-extras", action="store_true", help="skip the config #4 / device-GA objects")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process group for N > 1 (gloo: ranks may share a GPU — a code-path check, not a bench)")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist

    import support as S
    from paper_2109_11067_b200 import dist as D
    from paper_2109_11067_b200 import migplan as mp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    n_dev = torch.cuda.device_count()
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(n_dev, 1)
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    name = args.workload
    sharded = world > 1 and not is_ga(name)
    # ranks sharing one GPU (gloo code-path check): split its SMs between their greedy grids
    share = max(1, -(-world // max(n_dev, 1))) if world > 1 else 1
    red_dev = "cuda" if args.dist_backend == "nccl" else "cpu"

    ps, sv = load_workload(name)
    workers = args.workers
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def make_ctx():
        c = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), device=local)
        boards = D.shard_context(c, local, max_ctas=(148 // share if share > 1 else 0)) if sharded else None
        return c, boards

    def close_ctx(c, boards):
        if boards:
            D.unshard_context(c, boards)
        c.close()

    def step(c):
        if is_ga(name) and world > 1:
            p = ga_params(name, workers)
            _, dep = D.island_two_phase(c, p)
            return [g.config for g in dep.gpus]
        return run_step(mp, name, c, sv, ps, workers)

    ctx, boards = make_ctx()
    for _ in range(max(args.warmup, 0)):
        plan = step(ctx)
    # the harness's own long-lived objects (fixtures, goldens) move to the permanent GC
    # generation, so a collection inside a timed step does not traverse them (r02f/r02j: single
    # e2e steps +0.8-1.1 s on the host with identical kernel time)
    gc.collect()
    gc.freeze()

    # ---- resident (value)
    clocks = ClockSampler(local)
    clocks.start()
    ctx.reset_stats()
    dev_ms = 0.0
    barrier()
    for _ in range(args.steps):
        plan, t = timed(lambda: step(ctx), flush, torch)
        dev_ms += t
    barrier()
    st = ctx.stats()
    clock = clocks.stop()
    plan_sha = S.plan_sha(plan)

    # ---- end to end through the C-ABI from host buffers (e2e); the cold step first
    e2e_steps = max(1, min(args.steps, 5))
    close_ctx(ctx, boards)
    barrier()
    mp.release_device_cache(local)
    cold = {}

    e2e_host = []  # per e2e step: host wall of context build, plan call, close (ms)

    def e2e_step():
        t0 = time.perf_counter()
        c2, b2 = make_ctx()
        t1 = time.perf_counter()
        p = step(c2)
        t2 = time.perf_counter()
        s2 = c2.stats()
        close_ctx(c2, b2)
        t3 = time.perf_counter()
        e2e_host.append([round(1e3 * (t1 - t0), 2), round(1e3 * (t2 - t1), 2), round(1e3 * (t3 - t2), 2)])
        return p, s2

    (_, s_cold), cold_ms = timed(e2e_step, flush, torch)
    cold = {"cold_ms": cold_ms, "cold_note": "first step after mig_device_cache_release: arenas, streams and "
                                              "pinned step buffers allocated inside the timed step"}
    e2e_ms = 0.0
    e2e_rows = h2d = d2h = 0
    e2e_list, e2e_kern = [], []
    e2e_clocks = ClockSampler(local)
    e2e_clocks.start()
    barrier()
    for _ in range(e2e_steps):
        (p2, s2), t = timed(e2e_step, flush, torch)
        e2e_list.append(round(t, 3))
        e2e_kern.append(round(s2["greedy_ms"] + s2["mcts_ms"] + s2["topk_ms"], 3))
        e2e_ms += t
        e2e_rows += s2["rows_scored"]
        h2d += s2["h2d_bytes"]
        d2h += s2["d2h_bytes"]
    barrier()
    e2e_clock = e2e_clocks.stop()

    rows = st["rows_scored"]
    t = torch.tensor([dev_ms, e2e_ms, cold_ms, float(rows), float(e2e_rows), st["greedy_ms"]], dtype=torch.float64,
                     device=red_dev if world > 1 else "cuda")
    per_rank_rows = [rows]
    shas = [plan_sha]
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        per_rank_rows = [None] * world
        dist.all_gather_object(per_rank_rows, rows)
        shas = [None] * world
        dist.all_gather_object(shas, plan_sha)
        dev_ms_max, e2e_ms_max, cold_max = tmax[0].item(), tmax[1].item(), tmax[2].item()
        # sharded: each rank scanned its shard; islands: each rank planned the whole workload —
        # either way the job's rows are the sum over ranks
        rows_all, e2e_rows_all = tsum[3].item(), tsum[4].item()
        cold["cold_ms"] = cold_max
    else:
        dev_ms_max, e2e_ms_max, rows_all, e2e_rows_all = dev_ms, e2e_ms, float(rows), float(e2e_rows)

    if rank == 0:
        peak, peak_kind = measured_peak()
        kern = {"greedy_kernel": (st["greedy_ms"], st["greedy_rows"], st["greedy_calls"]),
                "topk1_kernel": (st["topk_ms"], st["topk_rows"] - st["mcts_rows"], st["topk_calls"] - st["mcts_topk_calls"]),
                "mcts_kernel": (st["mcts_ms"], st["mcts_rows"], st["mcts_launches"])}
        dom = max(kern, key=lambda k: kern[k][0])
        k_ms, k_rows, k_calls = kern[dom]
        launch_s = k_ms / 1e3 / max(k_calls, 1)
        k_bytes = 8.0 * k_rows / max(k_calls, 1)  # algorithmic bytes per launch: 8 B per packed row scored
        achieved = k_bytes / launch_s / 1e9 if launch_s > 0 else 0.0
        traffic, traffic_src = profile_traffic(dom, name)
        par = ("dp1" if world == 1 else
               f"config-space shards over {world} GPUs (IPC peer-memory boards, per-step in-kernel exchange)"
               if sharded else f"{world} GA islands")
        line = {
            "metric": METRIC, "value": rows_all / (dev_ms_max / 1e3), "unit": "configs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if (sharded or world == 1) and not is_ga(name) else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "description": WORKLOADS[name], "l2": L2_NOTE},
            "result": {"plan_ms": dev_ms_max / args.steps, "gpus_in_plan": len(plan), "plan_sha": plan_sha,
                       "plan_sha_all_ranks_equal": len(set(shas)) == 1, "rows_per_step": rows_all / args.steps,
                       "rows_per_rank": per_rank_rows, "parity": golden_check(name, plan), "parallelism": par,
                       "greedy_steps": st["greedy_steps"] // max(st["greedy_calls"], 1),
                       "ext_events_per_plan": st["ext_events"] / max(st["greedy_calls"], 1),
                       "ext_rows_per_plan": st["ext_rows"] / max(st["greedy_calls"], 1)},
            "e2e": {"value": e2e_rows_all / (e2e_ms_max / 1e3), "unit": "configs/s",
                    "h2d_bytes_per_step": h2d // e2e_steps, "d2h_bytes_per_step": d2h // e2e_steps,
                    "ms_per_step": e2e_ms_max / e2e_steps, "steps": e2e_steps, "step_ms_rank0": e2e_list,
                    "kernel_ms_rank0": e2e_kern, "host_ctx_plan_close_ms_rank0": e2e_host, "clocks": e2e_clock, **cold},
            "gpu_launches": st["kernel_launches"],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "traffic_source": traffic_src, "kernel": dom,
                         "launch_ms": 1e3 * launch_s, "bytes_per_launch": k_bytes, "bytes_per_unit": 8,
                         "unit_of_work": "packed candidate row scored (8 B: four u16 (service, pattern) codes)",
                         "peak_kind": peak_kind,
                         # `peak` is the driver's copy (read+write) figure; the scan only READS, and a
                         # read-only stream on this pool's B200s measured 7,383 GB/s
                         # (profiles/r02a_readbw.txt, best shape) -- the tighter denominator
                         "read_stream_peak": READ_STREAM_GBS, "frac_of_read_stream": achieved / READ_STREAM_GBS},
            "clocks": clock,
            "breakdown": {"greedy_ms": st["greedy_ms"], "topk_ms": st["topk_ms"], "mcts_ms": st["mcts_ms"],
                          "phase_ms": list(st["phase_ms"]),
                          "greedy_calls": st["greedy_calls"], "greedy_rows": st["greedy_rows"]},
        }
        if world == 1 and not args.no_cpu_baseline:
            try:
                rs = RefSampler(name, min(os.cpu_count() or 1, 8))
                dt = rs.step()
                line["cpu_baseline"] = {"value": rs.rows / dt, "unit": "configs/s", "cores": rs.cores,
                                        "kind": rs.kind, "sample": rs.sample, "step_s": dt,
                                        "plan_prefix_matches": S.plan_key(plan[:len(rs.plan)]) == S.plan_key(rs.plan),
                                        **host_info()}
            except Exception as e:  # pragma: no cover
                line["cpu_baseline"] = {"error": repr(e)}
        if world == 1 and not args.no_secondary and name != "slos24_ga10":
            line["secondary"] = secondary_ga(mp, local, flush, torch, max(1, min(args.steps, 5)), workers)
        if world == 1 and not args.no_extras:
            line["extras"] = extra_measurements(mp, local)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
