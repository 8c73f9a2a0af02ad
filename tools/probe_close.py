"""Where an end-to-end config-#5 step's host time goes (context build / plan / stats / close),
with bench.py's NVML clock sampler running beside it (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
import support as S  # noqa: E402
from support import mp  # noqa: E402

import bench  # noqa: E402


def main():
    ps, sv = bench.load_workload("gen128_8.0_greedy")
    clocks = bench.ClockSampler(0)
    clocks.start()
    for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
        t0 = time.perf_counter()
        c = mp.make_plan_context(sv, ps, mp.PartitionRuleSet.defaults())
        t1 = time.perf_counter()
        plan = mp.fast_algo(mp.zero_completion(len(sv)), c)
        t2 = time.perf_counter()
        st = c.stats()
        t3 = time.perf_counter()
        c.close()
        t4 = time.perf_counter()
        print(f"rep {rep}: ctx {1e3*(t1-t0):.1f} plan {1e3*(t2-t1):.1f} (kernel {st['greedy_ms']:.1f}) stats {1e3*(t3-t2):.2f} "
              f"close {1e3*(t4-t3):.1f} ms, {len(plan)} GPUs", flush=True)
    clocks.stop()


if __name__ == "__main__":
    main()
