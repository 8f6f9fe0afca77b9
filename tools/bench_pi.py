"""Wall time of configs 1-2 (BASELINE.json): the paper's Π explored to depth
12 and 200 (launch- and latency-bound — ≤ 5 parents per
level — so wall time is the measure, no roofline).  Engine: snp_explore
through the C ABI (exact dedup, int32 storage); oracle: oracle_explore
(1 thread).  Prints one JSON line per (encoding, depth).
Usage: python tools/bench_pi.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1104_1824_b200 import snp  # noqa: E402
from paper_1104_1824_b200 import workloads as W  # noqa: E402


def main():
    for enc in ("simulator", "textbook"):
        w = W.pi_system(enc)
        for depth in (12, 200):
            eng = snp.System(w, count_bits=32, dedup=0)
            t0 = time.perf_counter()
            eng.explore(None, depth=depth)  # first run: includes the level buffers' first allocation
            tf = time.perf_counter() - t0
            t0 = time.perf_counter()
            tree = eng.explore(None, depth=depth)
            te = time.perf_counter() - t0
            launches = snp.snp_kernel_launches()
            t0 = time.perf_counter()
            ref = oracle.System.from_workload(w).explore(w.C0, depth=depth)
            to = time.perf_counter() - t0
            same = bool((tree.configs == ref.configs).all() and (tree.parent == ref.parent).all())
            tree.close()
            # the ABI call alone (snp_explore + snp_tree_free, no Python-side copies)
            import ctypes
            L = snp.lib()
            h = ctypes.c_void_p()
            t0 = time.perf_counter()
            st = L.snp_explore(eng._h, None, depth, ctypes.byref(h))
            ta = time.perf_counter() - t0
            L.snp_tree_free(h)
            assert st == 0
            print(json.dumps({"workload": f"Π ({enc} encoding) to depth {depth}", "configs": int(tree.num_configs),
                              "transitions": int(tree.counters.T.sum()), "engine_ms": 1e3 * te,
                              "engine_first_run_ms": 1e3 * tf, "abi_snp_explore_ms": 1e3 * ta,
                              "oracle_ms": 1e3 * to, "levels": int(tree.num_levels),
                              "level_kernels_ms": float(tree.counters.ms.sum()),
                              "equal_to_oracle": same, "kernel_launches_total": launches}))


if __name__ == "__main__":
    main()
