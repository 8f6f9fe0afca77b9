#!/usr/bin/env python
"""bench.py — config transitions/s of the batched SNP transition step on B200.

One "step" = one BFS level of the hot path (applicability,
Ψ + scan, mixed-radix decode + child fingerprints, dedup + thinning, C + S·M
for the kept children) over the whole frontier of BASELINE.json config 4
(random SNP system m = 16384 neurons, n = 65536 rules, out-degree 8,
frontier F = 2^22, uint8 counts, 128-bit fingerprint dedup, 20 levels).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]

value       Σ T over the K timed levels ÷ their device time (CUDA events on the
            engine's stream, inputs resident in HBM).
e2e         the same metric through the public C ABI from a pinned HOST level 0
            (row-major uint8, H2D inside the timed region) with the per-level
            result (edges + fingerprints of the new frontier) read back.
roofline    dominant kernel phase: algorithmic bytes ÷ its
            CUDA-event time, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline  the CPU oracle (oracle/, as it stands: oracle_explore_par with
            one thread per host core) on a bounded sample of the same workload.
--impl reference  the oracle as the reference arm (this tier has no reference
            code): each step = the oracle on a bounded sample of the workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1104_1824_b200 import workloads as W  # noqa: E402

METRIC = "config transitions/s (C+S·M) at 1/2/4/8 B200; % HBM roofline"
UNIT = "transitions/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=17)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[3, 4, 5],
                    help="BASELINE.json configs[k-1]; 5 is an 8-GPU workload (use --F for a 1-GPU slice)")
    ap.add_argument("--F", type=int, default=0, help="override frontier size (testing only)")
    ap.add_argument("--m", type=int, default=0, help="override neuron count (testing only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dist", action="store_true", help="use the multi-GPU driver even on 1 GPU (testing)")
    return ap.parse_args()


def workload_for(args):
    cfg = dict(W.CONFIGS[args.config])
    if args.F:
        cfg["F"] = args.F
        cfg["frontier_target"] = args.F
    if args.m:
        cfg["m"] = args.m
    w = W.random_system(cfg["m"], outdeg=8, k_nd=cfg["k_nd"], seed=cfg["seed"], name=f"config{args.config}")
    return cfg, w


def config_json(args, cfg, w, K):
    bytes_per = cfg["count_bits"] // 8
    return {
        "workload": f"config{args.config}: random SNP system m={w.m} n={w.n} outdeg 8 k_nd={cfg['k_nd']}, "
                    f"frontier F={cfg['F']} (thinning target), {cfg['depth']} levels",
        "m": w.m, "n": w.n, "F": cfg["F"], "storage": f"u{cfg['count_bits']}" if bytes_per < 4 else "i32",
        "dedup": "fp128" if cfg["dedup"] else "exact", "levels_warmup": args.warmup, "levels_timed": K,
        "l2": f"inputs > L2: each level reads a {w.m * cfg['F'] * bytes_per / 1e9:.1f} GB frontier (L2 = 126 MB)",
        "seed": cfg["seed"],
    }


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for ln in open(self.path):
            f = [x.strip() for x in ln.split(",")]
            if len(f) >= 9:
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


KERNEL_OF = {"expand": "K-a k_expand_tc (tensor cores) + k_nd_pass, else k_expand_q / k_expand_t", "materialize": "K-c k_materialize_bs + k_patch",
             "dedup": "K-d k_dedup..k_compact", "keys": "K-b k_child_keys"}


def ncu_traffic(kernel_phase, config):
    """dram bytes per launch of the dominant kernel from the committed ncu
    summary (profiles/ncu_summary.json) when it was captured on this
    workload (its "config"), else None."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        d = json.load(open(path))
        if int(d.get("config", 4)) != int(config):
            return None
        return d["kernels"][kernel_phase]["dram_bytes_per_launch"]
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline and the reference arm)
# ---------------------------------------------------------------------------
def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def oracle_sample(w, cfg, rows_begin, n_rows, threads):
    """the oracle (oracle_explore_par: children of each parent on `threads`
    host threads, decisions in canonical order) expanding n_rows level-0
    parents of the workload by one level; returns (T, seconds)."""
    import oracle
    sysw = oracle.System.from_workload(w)
    L0 = W.level0_counts(w, n_rows, cfg["seed"], row_begin=rows_begin)
    t0 = time.perf_counter()
    run = sysw.explore_par(L0, depth=1, dedup=cfg["dedup"], count_bits=cfg["count_bits"], n_threads=threads)
    dt = time.perf_counter() - t0
    assert run.status == 0, run.error
    T = int(run.counters.T.sum())
    run.close()
    return T, dt


def calibrate_rows(w, cfg, target_s, threads):
    n0 = 4 * threads
    T, dt = oracle_sample(w, cfg, 0, n0, threads)
    per_row = max(dt / n0, 1e-5)
    return max(n0, min(1 << 17, int(target_s / per_row)))


def cpu_baseline(w, cfg, target_s=12.0):
    cores = host_cores()
    rows = calibrate_rows(w, cfg, target_s, cores)
    T, dt = oracle_sample(w, cfg, 0, rows, cores)
    return {"value": T / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"oracle BFS (C++ oracle/ oracle_explore_par, {cores} threads on {cores} host cores, "
                      f"{cpu_model()}) expanding {rows} level-0 parents of the same workload by one level: "
                      f"{T} transitions in {dt:.1f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg, w = workload_for(args)
    cores = host_cores()
    rows = calibrate_rows(w, cfg, 2.0, cores)
    for i in range(args.warmup):
        oracle_sample(w, cfg, i * rows, rows, cores)
    Ts, dts = [], []
    for i in range(args.steps):
        T, dt = oracle_sample(w, cfg, (args.warmup + i) * rows, rows, cores)
        Ts.append(T)
        dts.append(dt)
    value = sum(Ts) / sum(dts)
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(dts) / len(dts),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
           "data": "synthetic", "config": config_json(args, cfg, w, args.steps),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                            "sample": f"each step: oracle BFS (oracle_explore_par, {cores} threads, {cpu_model()}) "
                                      f"expanding {rows} level-0 parents by one level"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# native arm
# ---------------------------------------------------------------------------
def step_bytes(c, m, w_bytes):
    """SURVEY §8(d-3) algorithmic bytes of one level: parents read once, kept
    children written once, one 32-B probe per transition, 48 B per kept key."""
    return c["parents"] * m * w_bytes + c["kept"] * m * w_bytes + c["T"] * 32 + c["kept"] * 48


def run_native(args, rank, world):
    import torch
    from paper_1104_1824_b200 import snp

    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local_rank)
    snp.set_device(local_rank)  # libsnp.so's own CUDA runtime: the same GPU
    dev = torch.device("cuda", local_rank)
    dist = None
    use_dist = world > 1 or args.dist
    if use_dist:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    cfg, w = workload_for(args)
    m, F = w.m, cfg["F"]
    wb = cfg["count_bits"] // 8
    eng = snp.System(w, count_bits=cfg["count_bits"], dedup=cfg["dedup"], frontier_target=cfg["frontier_target"],
                     keep_tree=0)
    stream = torch.cuda.current_stream()
    eng.set_stream(stream.cuda_stream)
    eng.set_profiling(True)
    # level 0 generated on the device (inputs resident in HBM); rank r holds rows [lo, hi)
    if use_dist:
        from paper_1104_1824_b200 import dist as D
        lo, hi = D.level0_slice(F, rank, world)
        runner = D.DistExplorer(eng)  # the library's NCCL communicator; every exchange inside snp_dist_advance
    else:
        lo, hi, runner = 0, F, eng
    Fl = hi - lo
    buf = torch.empty((m, max(Fl, 1)), dtype=torch.uint8 if wb == 1 else torch.int32, device=dev)
    if Fl:
        snp.generate_level0_device(w, Fl, cfg["seed"], buf.data_ptr(), wb, snp.SNP_LAYOUT_NEURON_MAJOR, Fl,
                                   stream.cuda_stream, row_begin=lo)
    runner.begin(snp.configs_from_device(buf.data_ptr(), Fl, max(Fl, 1), wb, snp.SNP_LAYOUT_NEURON_MAJOR))
    del buf
    torch.cuda.empty_cache()
    digest_at = {}  # run digest after `steps` levels, compared with the e2e run's (same levels from the same level 0)
    for _ in range(args.warmup):
        runner.advance()
        if eng.depth == args.steps and not use_dist:
            digest_at[args.steps] = eng.summary()[2]
    prof0 = eng.profile()
    launches0 = snp.snp_kernel_launches()
    clocks = Clocks(torch.cuda.current_device())
    clocks.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    levels, lvl_prof = [], []
    for _ in range(args.steps):
        levels.append(runner.advance())
        if not use_dist:
            lvl_prof.append(eng.profile())  # cumulative phase times: per-level deltas below (drift attribution)
            if eng.depth == args.steps:
                digest_at[args.steps] = eng.summary()[2]  # a host read of the running sum: no device work
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = e0.elapsed_time(e1)
    if dist:  # max over ranks
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    launches = snp.snp_kernel_launches() - launches0
    prof1 = eng.profile()
    phase_ms = {k: prof1[k] - prof0[k] for k in prof1}
    T_sum = sum(c["T"] for c in levels)
    value = T_sum / (elapsed_ms / 1e3)
    peak, peak_src = measured_peak()
    # per-phase algorithmic bytes of THIS rank's kernels
    par = [c.get("parents_local", c["parents"]) for c in levels]
    kep = [c.get("kept_local", c["kept"]) for c in levels]
    Tl = [c.get("T_local", c["T"]) for c in levels]
    alg = {
        "expand": sum(x * m * wb for x in par),
        # K-c reads each parent row once and writes each kept child once
        "materialize": sum(x * m * wb + k * m * wb for x, k in zip(par, kep)),
        "dedup": sum(t * 32 + k * 48 for t, k in zip(Tl, kep)),
        "keys": sum(t * 16 for t in Tl),
    }
    dom = max(("expand", "materialize", "dedup", "keys"), key=lambda k: phase_ms.get(k, 0.0))
    achieved = alg[dom] / (phase_ms[dom] / 1e3) / 1e9 if phase_ms[dom] > 0 else 0.0
    sb = sum(p_ * m * wb + k * m * wb + t * 32 + k * 48 for p_, k, t in zip(par, kep, Tl))
    n_conf, T_total, digest = runner.summary()
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": f"u{8 * wb}" if wb < 4 else "i32", "data": "synthetic",
        "config": {**config_json(args, cfg, w, args.steps),
                   "parallelism": f"hash-partitioned dedup over {world} GPU(s): keys all-to-all over NCCL issued by "
                                  f"libsnp.so (snp_dist_advance), frontier range-partitioned and rebalanced"
                   if use_dist else "1 GPU"},
        "roofline": {"bound": "hbm", "kernel": f"phase '{dom}' ({KERNEL_OF.get(dom, dom)})",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ncu_traffic(dom, args.config), "peak_source": peak_src},
        "step_roofline": {"algorithmic_GB_per_step_per_gpu": sb / len(levels) / 1e9,
                          "achieved_per_gpu": sb / (elapsed_ms / 1e3) / 1e9,
                          "frac": sb / (elapsed_ms / 1e3) / 1e9 / peak},
        "phase_ms_per_step": {**{k: v / args.steps for k, v in phase_ms.items()},
                              "other": elapsed_ms / args.steps - sum(phase_ms.values()) / args.steps},
        "levels": [{k: c[k] for k in ("parents", "halting", "T", "n_new", "kept")} | {"ms": round(c["ms"], 3)}
                   | ({"phase_ms": {k: round(lvl_prof[i][k] - (lvl_prof[i - 1] if i else prof0)[k], 3)
                                    for k in ("expand", "keys", "dedup", "materialize")}} if lvl_prof else {})
                   for i, c in enumerate(levels)],
        "digest": f"{digest:016x}", "gpu_launches": launches, "clocks": clk,
    }
    eng.close()
    del eng, runner
    torch.cuda.empty_cache()
    if not args.no_e2e:
        out["e2e"] = run_e2e(args, cfg, w, snp, torch, rank, world, dist if use_dist else None,
                             digest_at.get(args.steps))
    if not args.no_cpu and rank == 0 and world == 1:
        out["cpu_baseline"] = cpu_baseline(w, cfg)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, cfg, w, snp, torch, rank=0, world=1, dist=None, device_digest=None):
    """The user's call path: level 0 from a pinned HOST buffer (row-major;
    snp_begin, or snp_dist_start with this rank's slice), then per level
    snp_advance / snp_dist_advance and the new level's edges + fingerprints
    read back into pinned host buffers.  N > 1: each rank its slice, wall
    time between barriers, max over ranks; value = all ranks' transitions."""
    m, F = w.m, cfg["F"]
    wb = cfg["count_bits"] // 8
    dt = torch.uint8 if wb == 1 else torch.int32
    lo, hi = (F * rank // world, F * (rank + 1) // world)
    Fl = hi - lo
    try:
        host = torch.empty((max(Fl, 1), m), dtype=dt, pin_memory=True)
    except Exception as e:  # pinned allocation failed
        return {"value": None, "unit": UNIT, "error": f"pinned host buffer: {e}"}
    # fill the host buffer with the same level 0 (device generator, chunked D2H; setup, untimed)
    chunk = max(1, (1 << 31) // (m * wb))
    tmp = torch.empty((chunk, m), dtype=dt, device="cuda")
    for r0 in range(0, Fl, chunk):
        n = min(chunk, Fl - r0)
        snp.generate_level0_device(w, n, cfg["seed"], tmp.data_ptr(), wb, snp.SNP_LAYOUT_ROW_MAJOR, m, 0,
                                   row_begin=lo + r0)
        host[r0:r0 + n].copy_(tmp[:n])
    # this box's pinned host -> device copy rate (context for the e2e number: level 0 is H2D-bound)
    nb = min(Fl, max(1, (4 << 30) // (m * wb)))
    probe = torch.empty((nb, m), dtype=dt, device="cuda")
    probe.copy_(host[:nb], non_blocking=True)
    torch.cuda.synchronize()
    tp = time.perf_counter()
    probe.copy_(host[:nb], non_blocking=True)
    torch.cuda.synchronize()
    box_h2d = nb * m * wb / (time.perf_counter() - tp) / 1e9
    del tmp, probe
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    eng = snp.System(w, count_bits=cfg["count_bits"], dedup=cfg["dedup"], frontier_target=cfg["frontier_target"],
                     keep_tree=0)
    runner = eng
    if dist is not None:
        from paper_1104_1824_b200 import dist as D
        runner = D.DistExplorer(eng)
    c0 = snp.snp_configs(host.data_ptr(), Fl, m, wb, snp.SNP_LAYOUT_ROW_MAJOR, 0, 0)
    eng.reserve_edges(2 * (F // world) + 1024)  # pinned result buffers, like the pinned input: allocated before timing
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    runner.begin(c0)
    t_begin = time.perf_counter() - t0
    T_sum = 0
    d2h = 0
    t_adv = t_edges = 0.0
    for _ in range(args.steps):
        ta = time.perf_counter()
        c = runner.advance()
        tb = time.perf_counter()
        T_sum += c["T"]
        parent, t, _h, fp = eng.level_edges(eng.depth, pinned=True, halting=False)
        d2h += parent.nbytes + t.nbytes + fp.nbytes
        t_adv += tb - ta
        t_edges += time.perf_counter() - tb
    dt_s = time.perf_counter() - t0
    e2e_digest = runner.summary()[2]
    if dist is not None:
        tt = torch.tensor([dt_s, d2h], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
        dt_s, d2h = float(tt[0].item()), int(tt[1].item())
    eng.close()
    del host
    return {"value": T_sum / dt_s, "unit": UNIT, "h2d_bytes_per_step": F * m * wb // args.steps,
            "d2h_bytes_per_step": d2h // args.steps,
            "digest": f"{e2e_digest:016x}",
            "digest_equal_device_run": (None if device_digest is None else e2e_digest == device_digest),
            "breakdown_s": {"begin (level-0 H2D + import + dedup)": round(t_begin, 4), "advance": round(t_adv, 4),
                            "edges D2H": round(t_edges, 4), "total": round(dt_s, 4),
                            "h2d_GBps_through_begin": round(Fl * m * wb / t_begin / 1e9, 2),
                            "box_pinned_h2d_GBps (torch copy, 4 GB)": round(box_h2d, 2)},
            "note": ("snp_begin" if world == 1 else f"snp_dist_start ({world} ranks, one host slice each)") +
                    "(pinned host row-major level 0) + K x (advance + snp_level_edges D2H into pinned buffers); "
                    "wall clock around synchronous ABI calls" + (", max over ranks" if world > 1 else "")}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus if args.gpus else 1))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_native(args, rank, world)


if __name__ == "__main__":
    main()
