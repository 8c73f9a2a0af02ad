"""Shared test helpers: backends, fixtures, workload generators, plan canonicalisation.

Only tests/, bench.py and __graft_entry__.smoke() import the oracle libraries, and only
as checkers.  `/root/reference` is never read here: the fixture JSONs the tests need
were copied into tests/golden/fixtures (input data of the reference's own tests).
"""
from __future__ import annotations

import hashlib
import json
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2109_11067_b200 import abi  # noqa: E402
from paper_2109_11067_b200 import migplan as mp  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
FIX = os.path.join(GOLDEN, "fixtures")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libmigref.so")
ORACLE_LIB = os.path.join(ROOT, "oracle", "liboracle.so")

_cache: dict = {}


def ref_backend():
    if "ref" not in _cache:
        _cache["ref"] = mp.Backend.load(REF_LIB, abi.REF_EXTRAS) if os.path.exists(REF_LIB) else None
    return _cache["ref"]


def oracle_backend():
    if "oracle" not in _cache:
        _cache["oracle"] = mp.Backend.load(ORACLE_LIB) if os.path.exists(ORACLE_LIB) else None
    return _cache["oracle"]


def checker_backend():
    """The CPU checker: the compiled reference if present, else the restatement oracle."""
    return ref_backend() or oracle_backend()


def product_backend():
    return mp.Backend.product()


def host_backend():
    """Any loaded library, for host-only helpers (RNG streams for gen_workload)."""
    return checker_backend() or product_backend()


def profiles():
    return mp.load_profiles(os.path.join(FIX, "profiles.json"))


def fixture_services(name: str, ps=None):
    return mp.load_services(os.path.join(FIX, f"{name}.json"), ps or profiles())


# ---- proj/tests/fixtures.hpp restated (sub-/super-linear synthetic models)

def two_model_store() -> dict:
    def prof(name, table):
        p = mp.ModelProfile(name)
        for size, rows in table.items():
            p.entries[size] = [mp.ProfileEntry(b, float(t), float(l)) for b, t, l in rows]
        return p

    cnn = {1: [(1, 30, 25), (4, 45, 45), (8, 50, 70), (16, 52, 130)],
           2: [(1, 34, 22), (4, 60, 38), (8, 80, 60), (16, 85, 120)],
           3: [(1, 36, 20), (4, 70, 33), (8, 105, 52), (16, 112, 105)],
           4: [(1, 38, 18), (4, 80, 30), (8, 120, 48), (16, 130, 110)],
           7: [(1, 40, 15), (4, 90, 25), (8, 140, 40), (16, 155, 120), (32, 165, 200)]}
    nlp = {1: [(1, 6, 95), (4, 7, 260)], 2: [(1, 14, 70), (4, 20, 150)], 3: [(1, 24, 55), (4, 33, 110)],
           4: [(1, 36, 42), (4, 52, 85), (8, 60, 140)], 7: [(1, 70, 28), (4, 112, 55), (8, 130, 90), (16, 140, 160)]}
    return {"cnn-a": prof("cnn-a", cnn), "nlp-a": prof("nlp-a", nlp)}


def random_workload(n: int, seed: int):
    """testfx::random_workload (fixtures.hpp:51-58)."""
    ps = two_model_store()
    normal = bool(seed % 2)
    mu, sigma = (900.0, 400.0) if normal else (6.3, 0.5)
    return ps, mp.gen_workload(n, not normal, mu, sigma, 100.0, seed, ps, backend=host_backend())


def gen(n: int, mu: float, seed: int = 4242):
    """gen_workload(n, Lognormal, mu, 0.6, 100 ms, seed, fixtures/profiles.json) (bench.hpp:125-156)."""
    ps = profiles()
    return ps, mp.gen_workload(n, True, mu, 0.6, 100.0, seed, ps, backend=host_backend())


# ---- canonical forms

def plan_key(plan) -> list:
    """A plan (list of GpuConfig) as plain lists, order preserved."""
    return [[[i.placement.slices, i.placement.start_slot, i.service_id, i.batch] for i in g.instances] for g in plan]


def fhex(x: float) -> str:
    return float(x).hex()


def comp_digest(comp) -> str:
    return hashlib.sha1(b"".join(struct.pack("<d", c) for c in comp)).hexdigest()[:16]


def plan_sha(plan_or_key) -> str:
    """sha256 (16 hex) of a plan's canonical form (plan_key), printed by both bench arms."""
    key = plan_or_key if (not plan_or_key or isinstance(plan_or_key[0], list)) else plan_key(plan_or_key)
    return hashlib.sha256(json.dumps(key, separators=(",", ":")).encode()).hexdigest()[:16]


def pool_sha(ctx) -> str:
    """Order-free digest of a context's base pool: sorted canonical rows (configs, utility
    bits, util_sum bits)."""
    rows = []
    for c in ctx.pool:
        key = [[i.placement.slices, i.placement.start_slot, i.service_id, i.batch] for i in c.config.instances]
        rows.append(json.dumps([key, [[k, v.hex()] for k, v in c.util], c.util_sum.hex()], separators=(",", ":")))
    rows.sort()
    return hashlib.sha256("\n".join(rows).encode()).hexdigest()[:16]


def load_golden(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)
