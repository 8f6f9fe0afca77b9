"""Measurement of BFS exploration for SN P systems with delays (SURVEY §8(f)
NEXT-3, include/snp.h ``snp_load_delay``, reading A26): a config-3-shaped
random system (m = 1024, 4 rules per neuron, out-degree 8) with 30 % of its
rules delayed by d ∈ {1, 2, 3}, uint8 storage, fingerprint dedup, thinning to
F.  Every child is materialised to key it (the delayed state is not linear in
the rule choice), so this path is bound by per-child work, not HBM.

Prints one JSON line: transitions/s over the timed levels (device time per
level from snp_advance's CUDA events), and the CPU oracle
(``oracle_explore_delay``, 1 thread) on a bounded sample of parents.
Usage: python tools/bench_delay.py [--F 65536] [--levels 6] [--warmup 2]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1104_1824_b200 import snp  # noqa: E402
from paper_1104_1824_b200 import workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1024)
    ap.add_argument("--F", type=int, default=65536)
    ap.add_argument("--levels", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--cpu-parents", type=int, default=200)
    args = ap.parse_args()
    w = W.random_system(args.m, outdeg=8, k_nd=3, seed=3, name="delay")
    rng = np.random.default_rng(3)
    delays = np.where(rng.random(w.n) < 0.3, rng.integers(1, 4, size=w.n), 0).astype(np.int32)
    L0 = W.level0_counts(w, args.F, 3).astype(np.int32)
    eng = snp.System(w, count_bits=8, dedup=1, frontier_target=args.F, keep_tree=0, delays=delays)
    eng.begin(L0)
    for _ in range(args.warmup):
        eng.advance()
    T = 0
    ms = 0.0
    levels = []
    for _ in range(args.levels):
        lc = eng.advance()
        T += lc["T"]
        ms += lc["ms"]
        levels.append({k: lc[k] for k in ("parents", "T", "n_new", "kept", "ms")})
    line = {"metric": "delayed-system transitions/s (snp_load_delay, BFS)", "value": T / (ms / 1e3),
            "unit": "transitions/s", "levels_timed": args.levels, "levels_warmup": args.warmup,
            "config": {"m": w.m, "n": w.n, "F": args.F, "delayed_rules": int((delays > 0).sum()),
                       "storage": "u8", "dedup": "fp128"}, "levels": levels}
    try:
        import oracle
        o = oracle.System.from_workload(w)
        k = args.cpu_parents
        t0 = time.perf_counter()
        r = o.explore_delay(delays, L0[:k], 1, dedup=1, count_bits=8)
        tc = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": float(r.counters.T.sum()) / tc, "unit": "transitions/s", "cores": 1,
                                "kind": "oracle",
                                "sample": f"oracle_explore_delay, {k} level-0 parents by one level: "
                                          f"{int(r.counters.T.sum())} transitions in {tc:.2f} s"}
    except Exception as ex:
        line["cpu_baseline"] = {"unavailable": str(ex)[:200]}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
