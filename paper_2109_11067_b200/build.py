"""Builds the product library `_native/libmigplan_b200.so` for sm_100a (in-tree, no JIT cache).

Every translation unit is compiled by nvcc with FMA contraction disabled on both the
device (-fmad=false) and host (-ffp-contract=off) side: the FP64 score/utility bits must
equal the reference's (SURVEY §0 hazard 1).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_native")
LIB = os.path.join(OUT_DIR, "libmigplan_b200.so")
SOURCES = ["model.cpp", "kernels.cu", "topk.cu", "rollout.cu", "ga.cu", "mcts.cu", "keyrank.cu", "bf.cu", "engine.cu", "search.cpp", "capi.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-std=c++20", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-fmad=false",
         "-Xcompiler", "-fPIC,-ffp-contract=off,-O3,-Wall", f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}",
         "--expt-relaxed-constexpr"]


def _compile(src: str) -> str:
    obj = os.path.join(OUT_DIR, "obj", os.path.splitext(src)[0] + ".o")
    srcp = os.path.join(CSRC, src)
    deps = [srcp] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".hpp", ".cuh"))]
    deps.append(os.path.join(ROOT, "include", "migplan_b200.h"))
    if os.path.exists(obj) and all(os.path.getmtime(obj) >= os.path.getmtime(d) for d in deps):
        return obj
    lang = [] if src.endswith(".cu") else ["-x", "cu"]
    cmd = [NVCC, *FLAGS, *lang, "-c", srcp, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(os.path.join(OUT_DIR, "obj"), exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xlinker", "-soname=libmigplan_b200.so",
               "-o", LIB, *objs, "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    if verbose:
        print(LIB)
    return LIB


def build_variant(defines: list[str], out: str) -> str:
    """Development aid (tools/probe_ab.py): the same library with extra -D flags, built into
    `out` (objects under <out>.obj/) so kernel variants can be A/B-timed on one GPU box."""
    obj_dir = out + ".obj"
    os.makedirs(obj_dir, exist_ok=True)

    def comp(src):
        obj = os.path.join(obj_dir, os.path.splitext(src)[0] + ".o")
        lang = [] if src.endswith(".cu") else ["-x", "cu"]
        r = subprocess.run([NVCC, *FLAGS, *[f"-D{d}" for d in defines], *lang, "-c", os.path.join(CSRC, src), "-o", obj],
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(comp, SOURCES))
    r = subprocess.run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out, *objs, "-lpthread"],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return out


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "variant":  # python build.py variant OUT.so DEF1 DEF2 ...
        print(build_variant(sys.argv[3:], sys.argv[2]))
    else:
        build(verbose="-v" in sys.argv)
