"""The C-ABI boundary: every library exports exactly what include/migplan_b200.h declares.

CPU-only: loads the libraries (no compute call reaches a GPU) and checks the product
fails loudly — MIG_ERR_DEVICE, never a silent CPU path — when no CUDA device exists.
"""
import ctypes as C
import os
import re

import pytest

import support as S
from support import abi, mp

HEADER = os.path.join(S.ROOT, "include", "migplan_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mig_[a-z0-9_]+)\s*\(", text)) - {"mig_greedy_trace_fn", "mig_mcts_trace_fn",
                                                                     "mig_ga_log_fn"})


def test_header_and_bindings_agree():
    assert header_functions() == abi.header_symbols()


def product_path():
    from paper_2109_11067_b200 import native_library_path

    return native_library_path()


@pytest.mark.parametrize("which", ["product", "oracle", "reference"])
def test_library_exports_every_symbol(which):
    path = {"product": None, "oracle": S.ORACLE_LIB, "reference": S.REF_LIB}[which]
    if which == "product":
        path = product_path()
    if not os.path.exists(path):
        pytest.skip(f"{which} library not built")
    lib = C.CDLL(path)
    missing = [f for f in header_functions() if not hasattr(lib, f)]
    assert not missing
    b = mp.Backend.load(path)
    assert b.name == which
    assert b.lib.mig_abi_version() == 1


def test_product_has_no_cpu_fallback():
    """Without a GPU the product must refuse to plan (MIG_ERR_DEVICE), not fall back."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    b = mp.Backend.load(product_path())
    ps = S.profiles()
    sv = S.fixture_services("slos_day", ps)
    with pytest.raises(mp.DeviceError):
        mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=b)


def test_product_host_entry_points_work_without_gpu():
    """Pure host entry points (rules, RNG) are usable anywhere and agree with the checker."""
    b = mp.Backend.load(product_path())
    parts = mp.enumerate_maximal_partitions(mp.PartitionRuleSet.defaults(), backend=b)
    gold = S.load_golden("partitions.json")["defaults"]
    assert [[[p.slices, p.start_slot] for p in lp.placements] for lp in parts] == gold
    r1, r2 = mp.Rng(42, backend=b), mp.Rng(42, backend=S.host_backend())
    assert [r1() for _ in range(64)] == [r2() for _ in range(64)]
    assert b.lib.mig_mix_seed(7, 1 << 20) == mp.mix_seed(7, 1 << 20)


def test_status_codes_map_to_reference_exceptions(impl):
    b = impl
    ps = S.two_model_store()
    sv = mp.validate_services([mp.ServiceSpec("a", "cnn-a", 350.0, 100.0)], ps)
    ctx = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults(), backend=b)
    with pytest.raises(mp.PlanningError):
        mp.fast_algo([0.0, 0.0], ctx)  # length mismatch (greedy.hpp:98-99)
    bad = dict(ps)
    bad["cnn-a"] = mp.ModelProfile("cnn-a", {1: [mp.ProfileEntry(4, 10.0, 5.0), mp.ProfileEntry(2, 10.0, 6.0)]})
    with pytest.raises(mp.SchemaError):
        mp.make_plan_context(sv, bad, mp.PartitionRuleSet.defaults(), backend=b)
