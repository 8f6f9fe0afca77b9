"""Parity at the stated sizes of BASELINE.json configs 3, 4 and 5 (SURVEY
§8(d-4), §8(d-6)), the CUDA engine through the C ABI against the oracle:

* config 4 (m = 16384, F = 2^22, uint8, fp128 dedup, thinning to F) in the
  launch configuration bench.py times, through all 25 levels of the driver's
  ``--steps 20 --warmup 5`` run: per level >= 1000 kept children recomputed
  one by one by the oracle from their parents (at least a third with t != 0,
  the k_patch path), their fingerprints, Ψ and the validity of the sibling
  set, plus properties that hold at any size;
* config 3 (m = 1024, F = 2^20, int32, exact dedup, 10 levels) in full: every
  level's counters, every configuration's (parent, t, fingerprint, halting)
  and the run digest against oracle_explore_par, plus sampled rows;
* config 5 scaled down as SURVEY §8(d-6) prescribes (m = 4096, F = 10^5,
  k_nd = 7, 20 levels) in full, and one level of the full-width system
  (m = 65536) with sampled parents."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
from paper_1104_1824_b200 import workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
THREADS = len(os.sched_getaffinity(0))


def level0_host(w, F, seed, dtype=np.int32, chunk=1 << 14):
    out = np.empty((F, w.m), dtype)
    for r0 in range(0, F, chunk):
        n = min(chunk, F - r0)
        out[r0:r0 + n] = W.level0_counts(w, n, seed, row_begin=r0, dtype=dtype)
    return out


def device_level0(snp, w, F, seed, wb):
    import torch
    buf = torch.empty((w.m, F), dtype=torch.uint8 if wb == 1 else torch.int32, device="cuda")
    snp.generate_level0_device(w, F, seed, buf.data_ptr(), wb, snp.SNP_LAYOUT_NEURON_MAJOR, F)
    torch.cuda.synchronize()
    return buf


def check_sampled_children(eng, osys, L, rng, n_children, min_nonzero_t):
    """kept children of level L+1 against the oracle, recomputed one by one
    from their parents (level L, still on the device)."""
    parent, t, _h, fp = eng.level_edges(L + 1, halting=False)
    K = len(parent)
    nz = np.nonzero(t != 0)[0]
    z = np.nonzero(t == 0)[0]
    n_nz = min(len(nz), max(min_nonzero_t, n_children // 2))
    pick = np.concatenate([rng.choice(nz, n_nz, replace=False) if n_nz else np.zeros(0, np.int64),
                           rng.choice(z, min(len(z), n_children - n_nz), replace=False)])
    pick = np.sort(pick)
    par_rows = eng.level_columns(L, parent[pick])
    child_rows = eng.level_columns(L + 1, pick)
    psi_of = {}

    def expected(k):  # the oracle, one sampled child (ctypes releases the GIL: host threads run in parallel)
        q = pick[k]
        psi, _S, Cn = osys.children(par_rows[k], cap=int(t[q]) + 1)
        return psi, Cn[int(t[q])], oracle.fingerprint(Cn[int(t[q])])

    with ThreadPoolExecutor(THREADS) as ex:
        res = list(ex.map(expected, range(len(pick))))
    for k, q in enumerate(pick):
        psi, child, f = res[k]
        assert (child == child_rows[k]).all()
        assert f == (int(fp[q][0]), int(fp[q][1]))
        psi_of[int(parent[q])] = psi
    # siblings kept from one parent: distinct t < Ψ(parent), tag order
    for p, psi in psi_of.items():
        ts = t[parent == p]
        assert len(ts) <= psi and len(set(ts.tolist())) == len(ts) and (ts < psi).all()
        assert (np.diff(ts.astype(np.int64)) > 0).all()
    return len(pick), int((t[pick] != 0).sum()), K


def test_config4_sampled_parity_all_timed_levels():
    from paper_1104_1824_b200 import snp
    cfg = W.CONFIGS[4]
    w = W.random_system(cfg["m"], outdeg=8, k_nd=cfg["k_nd"], seed=cfg["seed"])
    m, F = w.m, cfg["F"]
    eng = snp.System(w, count_bits=8, dedup=1, frontier_target=cfg["frontier_target"], keep_tree=0)
    buf = device_level0(snp, w, F, cfg["seed"], 1)
    eng.begin(snp.configs_from_device(buf.data_ptr(), F, F, 1, snp.SNP_LAYOUT_NEURON_MAJOR))
    del buf
    import torch
    torch.cuda.empty_cache()
    osys = oracle.System.from_workload(w)
    rng = np.random.default_rng(4)
    idx0 = np.sort(rng.choice(F, 32, replace=False))
    got0 = eng.level_columns(0, idx0)
    exp0 = np.stack([W.level0_counts(w, 1, cfg["seed"], row_begin=int(i))[0] for i in idx0])
    assert (got0 == exp0).all()
    seen = set(map(tuple, eng.level_edges(0, halting=False)[3].tolist()))
    assert len(seen) == eng.level_size(0)
    checked = []
    for L in range(25):                                           # bench: --warmup 5 --steps 20
        c = eng.advance()
        assert c["parents"] == eng.level_size(L) and c["kept"] <= c["n_new"] <= c["T"]
        parent, t, _h, fp = eng.level_edges(L + 1, halting=False)
        pinned = eng.level_edges(L + 1, pinned=True, halting=False)   # the e2e path's pinned buffers
        for a, b in zip((parent, t, fp), (pinned[0], pinned[1], pinned[3])):
            assert a.shape == b.shape and (a == b).all()
        assert (np.diff(parent) >= 0).all()                       # tag order
        keys = list(map(tuple, fp.tolist()))
        assert len(set(keys)) == len(keys) and not (set(keys) & seen)   # new, no repeats (A6)
        seen.update(keys)
        # thinning (A19): kept = N_new if N_new <= F, else ~F (every kept key below τ)
        if c["n_new"] > F:
            tau = oracle.thinning_tau(F, c["n_new"])
            assert c["tau"] == tau
            sample = fp[rng.choice(len(fp), 2000, replace=False)]
            assert all(oracle.fmix64(int(a)) < tau for a in sample[:, 0])
        n, n_nz, K = check_sampled_children(eng, osys, L, rng, 1000, 330)
        assert n >= 1000 and n_nz >= 330
        checked.append((n, n_nz, c["overflow_fixes"]))
    eng.close()
    print("config 4 sampled children per level (n, t != 0, overflow fixes):", checked)


def test_config3_full_size_exact():
    from paper_1104_1824_b200 import snp
    cfg = W.CONFIGS[3]
    w = W.random_system(cfg["m"], outdeg=8, k_nd=cfg["k_nd"], seed=cfg["seed"])
    F, depth = cfg["F"], cfg["depth"]
    eng = snp.System(w, count_bits=32, dedup=0, frontier_target=F, keep_tree=1)
    buf = device_level0(snp, w, F, cfg["seed"], 4)
    tree = eng.explore(snp.configs_from_device(buf.data_ptr(), F, F, 4, snp.SNP_LAYOUT_NEURON_MAJOR), depth=depth)
    del buf
    L0 = level0_host(w, F, cfg["seed"])
    ref = oracle.System.from_workload(w).explore_par(L0, depth, dedup=0, count_bits=32, frontier_target=F,
                                                     n_threads=THREADS)
    del L0
    assert ref.status == 0, ref.error
    assert tree.level_offsets.tolist() == ref.level_offsets.tolist()
    for a, b in (("T", "T"), ("new", "new"), ("kept", "kept")):
        assert getattr(tree.counters, a).tolist() == getattr(ref.counters, b).tolist()
    assert (tree.parent == ref.parent).all() and (tree.t == ref.t).all()
    assert (tree.fp == ref.fp).all() and (tree.halting == ref.halting).all()
    rng = np.random.default_rng(3)
    for L in range(tree.num_levels):
        lo, hi = tree.level_offsets[L], tree.level_offsets[L + 1]
        idx = np.sort(rng.choice(hi - lo, min(512, hi - lo), replace=False))
        assert (eng.level_columns(L, idx) == ref.rows(lo + idx)).all()
    assert tree.num_configs > 10 * F // 2
    ref.close()
    eng.close()


def test_config5_scaled_full():
    from paper_1104_1824_b200 import snp
    cfg = W.CONFIGS[5]
    w = W.random_system(4096, outdeg=8, k_nd=cfg["k_nd"], seed=cfg["seed"])
    F, depth = 100_000, 20
    L0 = level0_host(w, F, cfg["seed"])
    eng = snp.System(w, count_bits=8, dedup=1, frontier_target=F, keep_tree=1)
    tree = eng.explore(L0, depth=depth)
    ref = oracle.System.from_workload(w).explore_par(L0, depth, dedup=1, count_bits=8, frontier_target=F,
                                                     n_threads=THREADS)
    assert ref.status == 0, ref.error
    assert int(ref.counters.T[0]) > 20 * F                          # high nondeterminism (mean Ψ ≈ 32)
    assert tree.level_offsets.tolist() == ref.level_offsets.tolist()
    assert tree.counters.T.tolist() == ref.counters.T.tolist()
    assert tree.counters.new.tolist() == ref.counters.new.tolist()
    assert (tree.parent == ref.parent).all() and (tree.t == ref.t).all()
    assert (tree.fp == ref.fp).all() and (tree.halting == ref.halting).all()
    rng = np.random.default_rng(5)
    for L in range(tree.num_levels):
        lo, hi = tree.level_offsets[L], tree.level_offsets[L + 1]
        idx = np.sort(rng.choice(hi - lo, min(256, hi - lo), replace=False))
        assert (eng.level_columns(L, idx) == ref.rows(lo + idx)).all()
    ref.close()
    eng.close()


def test_config5_full_width_sampled():
    """config 5's per-GPU slice shape (m = 65536, k_nd = 7) on one GPU, F =
    2^16: one level, sampled children recomputed by the oracle."""
    from paper_1104_1824_b200 import snp
    cfg = W.CONFIGS[5]
    w = W.random_system(cfg["m"], outdeg=8, k_nd=cfg["k_nd"], seed=cfg["seed"])
    F = 1 << 16
    eng = snp.System(w, count_bits=8, dedup=1, frontier_target=F, keep_tree=0)
    buf = device_level0(snp, w, F, cfg["seed"], 1)
    eng.begin(snp.configs_from_device(buf.data_ptr(), F, F, 1, snp.SNP_LAYOUT_NEURON_MAJOR))
    del buf
    osys = oracle.System.from_workload(w)
    rng = np.random.default_rng(55)
    for L in range(2):
        c = eng.advance()
        assert c["T"] > 20 * c["parents"]
        n, n_nz, _K = check_sampled_children(eng, osys, L, rng, 300, 150)
        assert n >= 300
    eng.close()
