"""Per-level drift attribution at config 4: for each of
the bench's 25 levels, the phase times (CUDA events) next to the properties
of the frontier that select slower kernel paths — the count distribution
(K-a / K-c byte-permute tables cover counts < 16 / < 32; larger counts fold
through the compact table), T/F, the share of kept children with t != 0
(k_patch) and the overflow fixes.  Prints one JSON line per level."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1104_1824_b200 import snp  # noqa: E402
from paper_1104_1824_b200 import workloads as W  # noqa: E402


def main(levels=25, sample=8192):
    import torch
    cfg = W.CONFIGS[4]
    w = W.random_system(cfg["m"], outdeg=8, k_nd=cfg["k_nd"], seed=cfg["seed"])
    F = cfg["F"]
    eng = snp.System(w, count_bits=8, dedup=1, frontier_target=F, keep_tree=0)
    eng.set_profiling(True)
    buf = torch.empty((w.m, F), dtype=torch.uint8, device="cuda")
    snp.generate_level0_device(w, F, cfg["seed"], buf.data_ptr(), 1, snp.SNP_LAYOUT_NEURON_MAJOR, F)
    torch.cuda.synchronize()
    eng.begin(snp.configs_from_device(buf.data_ptr(), F, F, 1, snp.SNP_LAYOUT_NEURON_MAJOR))
    del buf
    torch.cuda.empty_cache()
    rng = np.random.default_rng(0)
    prev = eng.profile()
    for L in range(levels):
        Fl = eng.level_size(L)
        rows = eng.level_columns(L, np.sort(rng.choice(Fl, min(sample, Fl), replace=False)))
        c = eng.advance()
        p = eng.profile()
        _par, t, _h, _fp = eng.level_edges(L + 1, halting=False)
        blk = rows.reshape(-1, 64, w.m) if rows.shape[0] % 64 == 0 else None
        out = {"level": L, "ms": round(c["ms"], 2),
               "phase_ms": {k: round(p[k] - prev[k], 2) for k in ("expand", "keys", "dedup", "materialize")},
               "T_over_F": round(c["T"] / c["parents"], 3), "kept_t_nonzero": round(float((t != 0).mean()), 4),
               "overflow_fixes": c["overflow_fixes"],
               "count_ge16": round(float((rows >= 16).mean()), 5), "count_ge32": round(float((rows >= 32).mean()), 6),
               "count_ge128": round(float((rows >= 128).mean()), 7), "count_max": int(rows.max()),
               "count_mean": round(float(rows.mean()), 4)}
        # share of 32-lane warps (32 consecutive configurations of one neuron)
        # whose counts all stay below 16 / 32 (the register-table fast paths)
        if blk is not None:
            g = rows.reshape(-1, 32, w.m)
            out["warps_all_lt16"] = round(float((g.max(axis=1) < 16).mean()), 4)
            out["warps_all_lt32"] = round(float((g.max(axis=1) < 32).mean()), 4)
        prev = p
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
