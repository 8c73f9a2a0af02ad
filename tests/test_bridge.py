"""The C++ drop-in bridge compiles against the reference's own headers and links the product.

Where the reference headers exist (this container) the program is compiled and linked; it is
run (GPU fast_algo and GPU-MCTS crossover vs the reference's, in-process) only with a GPU.
"""
import os
import subprocess

import pytest

import support as S

REF_INC = "/root/reference/proj/include"


def build(tmp_path):
    from paper_2109_11067_b200 import native_library_path

    lib = native_library_path()
    exe = tmp_path / "bridge_check"
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{REF_INC}", f"-I{os.path.join(S.ROOT, 'include')}",
           os.path.join(S.ROOT, "tests", "cpp", "bridge_check.cpp"), "-o", str(exe), lib,
           f"-Wl,-rpath,{os.path.dirname(lib)}", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_bridge_compiles_against_reference(tmp_path):
    exe = build(tmp_path)
    assert subprocess.run([str(exe), "--compile-only"]).returncode == 0


BRIDGE = os.path.join(S.ROOT, "oracle", "_ref", "bridge_check")


@pytest.mark.gpu
def test_bridge_drives_reference_ga_on_gpu():
    """The reference's own crossover() with GpuMctsProcedure == with its MctsProcedure (matched seed)."""
    if not os.path.exists(BRIDGE):
        pytest.skip("bridge_check not built (needs the reference headers at build time)")
    r = subprocess.run([BRIDGE], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bridge ok" in r.stdout
