"""the reference's transition planner (transition_planner.hpp:658-697, on CPU)
consumes the B200 planner's plan output unchanged.

The day and night fixtures (proj/fixtures/slos_day.json, slos_night.json) are planned by the
CLI re-host (`optimize --mode fast`); the deployment files go, as written, through the
reference's own loaders (io.hpp) into plan_transition, and the transition plan must be
byte-identical to the one planned from the reference's own deployments of the same SLOs.
"""
import ctypes as C
import json
import os

import pytest

import support as S
from paper_2109_11067_b200 import cli

FIX = S.FIX
pytestmark = pytest.mark.skipif(S.ref_backend() is None, reason="reference shim not built")


def plan_files(tmp_path, impl, tag):
    out = {}
    for day in ("slos_day", "slos_night"):
        path = str(tmp_path / f"{tag}_{day}.json")
        args = ["optimize", "--mode", "fast", "--quiet", "--slos", os.path.join(FIX, f"{day}.json"), "--profiles",
                os.path.join(FIX, "profiles.json"), "-o", path]
        if impl.name != "product":
            args += ["--backend", impl.path]
        assert cli.main(args) == 0
        out[day] = path
    return out


def transition(files, old, new, budget=2):
    ref = S.ref_backend()
    buf = C.create_string_buffer(1 << 22)
    n = C.c_int32()
    ref.check(ref.lib.mig_ref_plan_transition(
        files[old].encode(), files[new].encode(), os.path.join(FIX, f"{old}.json").encode(),
        os.path.join(FIX, f"{new}.json").encode(), os.path.join(FIX, "profiles.json").encode(), budget, buf, 1 << 22,
        C.byref(n)))
    return buf.raw[:n.value]


def test_reference_transition_planner_consumes_the_plans(impl, tmp_path):
    mine = plan_files(tmp_path, impl, "impl")
    theirs = plan_files(tmp_path, S.ref_backend(), "ref")
    for old, new in (("slos_day", "slos_night"), ("slos_night", "slos_day")):
        got = transition(mine, old, new)
        assert got == transition(theirs, old, new)
        plan = json.loads(got)
        assert plan  # a non-empty transition plan document
