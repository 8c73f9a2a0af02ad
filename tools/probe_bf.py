"""Time brute_force_optimum: device search vs the reference (when oracle/_ref is built)."""
import sys
import time

sys.path.insert(0, "tests")
import support as S  # noqa: E402
from support import mp  # noqa: E402

BF = S.load_golden("brute_force.json")
RULES = mp.PartitionRuleSet.defaults()
prod, ref = S.product_backend(), S.ref_backend()
for name in sorted(BF):
    g = BF[name]
    if not name.startswith("gen4") and g.get("ref_wall_s", 0) < 0.05:
        continue
    ps = S.profiles() if g["store"] == "fixture" else S.two_model_store()
    sv = [mp.ServiceSpec(i, m, float.fromhex(r), float.fromhex(p)) for i, m, r, p in g["services"]]
    row = [name]
    for b in (prod, ref):
        if b is None:
            continue
        mp.brute_force_optimum(sv, ps, RULES, g["cap"], backend=b)
        t = time.perf_counter()
        dep = mp.brute_force_optimum(sv, ps, RULES, g["cap"], backend=b)
        row += [b.name, None if dep is None else len(dep.gpus), round((time.perf_counter() - t) * 1e3, 2)]
    print(*row, flush=True)
