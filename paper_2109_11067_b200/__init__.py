"""B200-native MIG-SERVING optimizer hot path (arXiv 2109.11067).

`migplan` mirrors the reference's C++ API (proj/include/migplan) in Python over the
C-ABI of `include/migplan_b200.h`; the compute lives in `_native/libmigplan_b200.so`
(hand-written CUDA for sm_100a + native C++ runtime).
"""
import os

_HERE = os.path.dirname(os.path.abspath(__file__))


def native_library_path() -> str:
    """Path of the product library; raises if it has not been built (no CPU fallback)."""
    p = os.environ.get("MIGPLAN_B200_LIB") or os.path.join(_HERE, "_native", "libmigplan_b200.so")
    if not os.path.exists(p):
        raise ImportError(f"libmigplan_b200.so not built ({p}); run `python -c 'import __graft_entry__ as g; g.build()'`")
    return p
