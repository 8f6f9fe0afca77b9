"""Measurement of single-path sampling (include/snp.h
``snp_sample``) on config 4's system (m = 16384, uint8 storage): W walkers
start from seeded level-0 configurations and take `steps` steps each.

Prints one JSON line: walker-steps/s through the C ABI (host int32 walkers in
and out, so the copies are inside the timed region — the call a user makes),
the device time of ``k_sample`` alone comes from an ncu launch list of this
script; and the CPU oracle (``oracle_sample``, 1 thread) on a bounded sample
of walkers, checked equal to the GPU's walkers.

Usage: python tools/bench_sample.py [--walkers 8192] [--steps 20] [--reps 3]
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
    ap.add_argument("--walkers", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cpu-walkers", type=int, default=8)
    args = ap.parse_args()
    cfg = W.CONFIGS[4]
    w = W.random_system(cfg["m"], outdeg=8, k_nd=cfg["k_nd"], seed=cfg["seed"], name="config4")
    C0 = W.level0_counts(w, args.walkers, cfg["seed"]).astype(np.int32)
    eng = snp.System(w, count_bits=8, dedup=1)
    eng.sample(C0[:64], 1, 2)  # warm-up (module load, first launch)
    times = []
    for r in range(args.reps):
        t0 = time.perf_counter()
        out, hs = eng.sample(C0, 1000 + r, args.steps)
        times.append(time.perf_counter() - t0)
    t = float(np.median(times))
    ws = args.walkers * args.steps
    line = {"metric": "sampled walker-steps/s (snp_sample, config-4 system)", "value": ws / t,
            "unit": "walker-steps/s", "walkers": args.walkers, "steps": args.steps, "ms_per_call": 1e3 * t,
            "h2d_bytes": int(C0.nbytes), "d2h_bytes": int(C0.nbytes + hs.nbytes),
            "halted": int((hs >= 0).sum()), "kernel_launches_per_call": 1}
    try:
        import oracle
        o = oracle.System.from_workload(w)
        n = args.cpu_walkers
        t0 = time.perf_counter()
        ref, _ = o.sample(C0[:n], 1000 + args.reps - 1, args.steps, count_bits=8)  # the last timed call's seed
        tc = time.perf_counter() - t0
        eq = bool((ref == out[:n]).all())
        line["cpu_baseline"] = {"value": n * args.steps / tc, "unit": "walker-steps/s", "cores": 1, "kind": "oracle",
                                "sample": f"oracle_sample, {n} walkers x {args.steps} steps in {tc:.2f} s",
                                "equal_to_gpu_walkers": eq}
    except Exception as ex:  # the oracle is test infrastructure; report why it is missing
        line["cpu_baseline"] = {"unavailable": str(ex)[:200]}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
