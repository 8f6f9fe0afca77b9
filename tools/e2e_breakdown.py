"""Where the e2e time of bench.py's run_e2e goes (one B200): wall time of
snp_begin (H2D of the pinned row-major level 0 + import) and of each
snp_advance / snp_level_edges, with the transitions of each level.
Usage: python tools/e2e_breakdown.py [--steps K]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1104_1824_b200 import snp  # noqa: E402


def main():
    sys.argv = [sys.argv[0]] + sys.argv[1:]
    args = bench.parse()
    cfg, w = bench.workload_for(args)
    m, F = w.m, cfg["F"]
    wb = cfg["count_bits"] // 8
    dt = torch.uint8 if wb == 1 else torch.int32
    host = torch.empty((F, m), dtype=dt, pin_memory=True)
    chunk = max(1, (1 << 31) // (m * wb))
    tmp = torch.empty((chunk, m), dtype=dt, device="cuda")
    for r0 in range(0, F, chunk):
        n = min(chunk, F - r0)
        snp.generate_level0_device(w, n, cfg["seed"], tmp.data_ptr(), wb, snp.SNP_LAYOUT_ROW_MAJOR, m, 0, row_begin=r0)
        host[r0:r0 + n].copy_(tmp[:n])
    del tmp
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    t = time.perf_counter()
    eng = snp.System(w, count_bits=cfg["count_bits"], dedup=cfg["dedup"], frontier_target=cfg["frontier_target"],
                     keep_tree=0)
    rec = {"system_s": time.perf_counter() - t}
    c0 = snp.snp_configs(host.data_ptr(), F, m, wb, snp.SNP_LAYOUT_ROW_MAJOR, 0, 0)
    t = time.perf_counter()
    eng.begin(c0)
    rec["begin_s"] = time.perf_counter() - t
    rec["h2d_GBps"] = F * m * wb / rec["begin_s"] / 1e9
    lv = []
    for _ in range(args.steps):
        t = time.perf_counter()
        c = eng.advance()
        ta = time.perf_counter() - t
        t = time.perf_counter()
        eng.level_edges(eng.depth, pinned=True)
        te = time.perf_counter() - t
        lv.append({"T": c["T"], "advance_ms": ta * 1e3, "edges_ms": te * 1e3})
    rec["levels"] = lv
    rec["T_sum"] = sum(x["T"] for x in lv)
    tot = rec["begin_s"] + sum(x["advance_ms"] + x["edges_ms"] for x in lv) / 1e3
    rec["e2e_transitions_per_s"] = rec["T_sum"] / tot
    eng.close()
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
