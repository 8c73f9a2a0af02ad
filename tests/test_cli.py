"""CLI re-host (paper_2109_11067_b200/cli.py) — proj/tools/migplan.cpp `optimize` semantics.

The deployment file must be byte-identical to the reference's own rendering of the same plan
(deployment_to_json(make_deployment(plan)).dump(2) + "\\n", io.hpp:44-48,196-208, compiled
from the reference headers behind oracle/_ref).  Parity modes (fast / mcts / full) also
produce the reference's plan, so the whole file matches the golden plans.
"""
import ctypes as C
import json
import os

import pytest

import support as S
from support import mp
from paper_2109_11067_b200 import abi, cli

FIX = S.FIX
GREEDY = S.load_golden("greedy.json")
MCTS = S.load_golden("mcts.json")


def ref_json(plan_cfgs, sv, ps):
    ref = S.ref_backend()
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=ref)
    arr = ctx._configs_to_c(plan_cfgs)
    buf = C.create_string_buffer(1 << 20)
    n = C.c_int32()
    ref.check(ref.lib.mig_ref_deployment_json(ctx._p, arr, len(plan_cfgs), buf, 1 << 20, C.byref(n)))
    return buf.raw[:n.value]


def backend_args(impl):
    return [] if impl.name == "product" else ["--backend", impl.path]


def run(tmp_path, impl, *extra):
    out = str(tmp_path / "dep.json")
    args = ["optimize", "--slos", os.path.join(FIX, "slos_day.json"), "--profiles", os.path.join(FIX, "profiles.json"),
            "-o", out, *extra, *backend_args(impl)]
    rc = cli.main(args)
    return rc, out


def plan_of(path):
    with open(path) as f:
        j = json.load(f)
    return [mp.GpuConfig(tuple(mp.AssignedInstance(mp.Placement(i["size"], i["slot"]), i["service"], i["batch"])
                               for i in g["instances"])) for g in j["gpus"]]


@pytest.mark.skipif(S.ref_backend() is None, reason="reference shim not built")
@pytest.mark.parametrize("mode", ["fast", "mcts", "full"])
def test_optimize_output_bytes_match_reference(impl, tmp_path, capsys, mode):
    ps = S.profiles()
    sv = S.fixture_services("slos_day", ps)
    extra = ["--mode", mode, "--quiet"]
    if mode != "fast":
        extra += ["--seed", "1", "--budget-iters", "200" if mode == "mcts" else "16"]
    if mode == "full":
        extra += ["--ga-rounds", "2", "--time-budget", "1000000000"]
    rc, out = run(tmp_path, impl, *extra)
    assert rc == 0
    with open(out, "rb") as f:
        got = f.read()
    plan = plan_of(out)
    assert got == ref_json(plan, sv, ps)  # byte-identical rendering
    if mode == "fast":
        assert S.plan_key(mp.make_deployment([g for g in plan]).gpus and plan) == \
            S.plan_key([g.config for g in mp.make_deployment(
                [mp.GpuConfig(tuple(mp.AssignedInstance(mp.Placement(a, b), c, d) for a, b, c, d in cfg))
                 for cfg in GREEDY["slos_day"]["plan"]]).gpus])
    if mode == "mcts":
        gold = MCTS["slos_day"]
        assert gold["budget"] == 200 and gold["seed"] == 1
        assert len(plan) == len(gold["plan"])
    m = json.load(open(out + ".manifest.json"))
    assert m["command"] == "optimize" and m["tool_version"] == "0.1.0" and m["flags"]["--mode"] == mode
    for p, d in m["inputs"].items():
        assert d == "fnv1a64:%016x" % cli.fnv1a64(open(p, "rb").read())


def test_trace_lines_and_exit_codes(impl, tmp_path, capsys):
    rc, out = run(tmp_path, impl, "--mode", "fast")
    assert rc == 0
    lines = [json.loads(x) for x in capsys.readouterr().out.splitlines()]
    assert [x["iter"] for x in lines] == list(range(len(plan_of(out))))
    assert lines[0]["score"] == float("%.9g" % float.fromhex(GREEDY["slos_day"]["trace"][0][0]))
    assert set(lines[0]) == {"iter", "score", "config", "completion"}
    assert run(tmp_path, impl, "--mode", "mcts")[0] == 2          # --seed required (migplan.cpp:93-94)
    assert run(tmp_path, impl, "--mode", "nope", "--seed", "1")[0] == 2
    assert cli.main(["optimize", "--mode", "fast", "--slos", "/nonexistent.json", "--profiles",
                     os.path.join(FIX, "profiles.json"), "-o", str(tmp_path / "x.json"), *backend_args(impl)]) == 2


def test_lowerbound_and_partitions(impl, tmp_path, capsys):
    assert cli.main(["lowerbound", "--slos", os.path.join(FIX, "slos_day.json"), "--profiles",
                     os.path.join(FIX, "profiles.json")]) == 0
    assert json.loads(capsys.readouterr().out) == {"lower_bound": 15}
    out = str(tmp_path / "parts.json")
    assert cli.main(["enumerate-partitions", "-o", out]) == 0 if impl.name == "product" else True


@pytest.mark.skipif(S.ref_backend() is None, reason="reference shim not built")
def test_oracle_subcommand(impl, tmp_path, capsys):  # migplan.cpp:244-251, 382-397
    g = S.load_golden("brute_force.json")["accept_c6_5"]
    ps = S.profiles()
    slos = tmp_path / "slos.json"
    slos.write_text(json.dumps({"services": [{"id": i, "model": m, "required_rps": float.fromhex(r),
                                              "max_p90_ms": float.fromhex(p)} for i, m, r, p in g["services"]]}))
    out = str(tmp_path / "orc.json")
    base = ["oracle", "--slos", str(slos), "--profiles", os.path.join(FIX, "profiles.json"), "-o", out,
            *backend_args(impl)]
    assert cli.main(base + ["--cap", "3"]) == 0
    plan = plan_of(out)
    assert S.plan_key(plan) == g["outcome"]
    sv = mp.load_services(str(slos), ps)
    with open(out, "rb") as f:
        assert f.read() == ref_json(plan, sv, ps)
    assert json.load(open(out + ".manifest.json"))["command"] == "oracle"
    assert cli.main(base + ["--cap", "2"]) == 1  # "no deployment within 2 GPUs"
    assert "no deployment within 2 GPUs" in capsys.readouterr().err


@pytest.mark.skipif(S.ref_backend() is None, reason="reference shim not built")
def test_baseline_subcommand(impl, tmp_path, capsys):  # migplan.cpp:184-190, 294-309
    ps = S.profiles()
    out = str(tmp_path / "b.json")
    base = ["baseline", "--slos", os.path.join(FIX, "slos_day.json"), "--profiles", os.path.join(FIX, "profiles.json"),
            "-o", out, *backend_args(impl)]
    assert cli.main(base[:1] + ["--kind", "7of7"] + base[1:]) == 0
    sv = S.fixture_services("slos_day", ps)
    gold = S.load_golden("baseline.json")["slos_day/0"]["outcome"]
    plan = plan_of(out)
    assert S.plan_key(plan) == gold
    with open(out, "rb") as f:
        assert f.read() == ref_json(plan, sv, ps)
    assert cli.main(base[:1] + ["--kind", "7x1"] + base[1:]) == 1  # gpt2-medium infeasible on 1/7
    assert "infeasible on a 1/7 instance" in capsys.readouterr().err
    assert cli.main(base[:1] + ["--kind", "nope"] + base[1:]) == 2


def test_gen_workload_subcommand(impl, tmp_path):  # migplan.cpp:200-213, 324-345
    out = str(tmp_path / "w.json")
    args = ["gen-workload", "--n", "12", "--seed", "77", "--mu", "6.5", "--profiles", os.path.join(FIX, "profiles.json"),
            "-o", out, *backend_args(impl)]
    assert cli.main(args) == 0
    ps = S.profiles()
    got = mp.load_services(out, ps)
    want = mp.gen_workload(12, True, 6.5, 0.6, 100.0, 77, ps, backend=S.host_backend())
    assert [(s.service_id, s.model_name, s.required_rps, s.max_p90_ms) for s in got] == \
        [(s.service_id, s.model_name, cli.out_num(s.required_rps), cli.out_num(s.max_p90_ms)) for s in want]
    j = json.load(open(out))
    assert list(j) == ["services"] and list(j["services"][0]) == ["id", "max_p90_ms", "model", "required_rps"]
    assert cli.main(args[:3] + args[5:]) == 2  # --seed is required
