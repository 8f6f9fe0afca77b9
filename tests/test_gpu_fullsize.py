"""Full-size parity in the launch configuration bench.py times (BASELINE.json
config 4: m = 16384, n = 65536, F = 2^22, uint8, 128-bit fingerprint dedup,
thinning to F): sampled children recomputed one by one by the oracle, plus
properties that hold at any size."""
import numpy as np
import pytest

import oracle
from paper_1104_1824_b200 import workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_config4_sampled_parity():
    import torch
    from paper_1104_1824_b200 import snp
    cfg = W.CONFIGS[4]
    w = W.random_system(cfg["m"], outdeg=8, k_nd=cfg["k_nd"], seed=cfg["seed"])
    m, F = w.m, cfg["F"]
    eng = snp.System(w, count_bits=8, dedup=1, frontier_target=cfg["frontier_target"], keep_tree=0)
    buf = torch.empty((m, F), dtype=torch.uint8, device="cuda")
    snp.generate_level0_device(w, F, cfg["seed"], buf.data_ptr(), 1, snp.SNP_LAYOUT_NEURON_MAJOR, F)
    torch.cuda.synchronize()
    eng.begin(snp.configs_from_device(buf.data_ptr(), F, F, 1, snp.SNP_LAYOUT_NEURON_MAJOR))
    del buf
    torch.cuda.empty_cache()
    osys = oracle.System.from_workload(w)
    rng = np.random.default_rng(4)
    # level 0 = the generator's rows (spot check against the host generator)
    idx0 = np.sort(rng.choice(F, 32, replace=False))
    got0 = eng.level_columns(0, idx0)
    exp0 = np.stack([W.level0_counts(w, 1, cfg["seed"], row_begin=int(i))[0] for i in idx0])
    assert (got0 == exp0).all()
    seen = set()
    _p, _t, _h, fp0 = eng.level_edges(0)
    seen.update(map(tuple, fp0.tolist()))
    assert len(seen) == eng.level_size(0)
    for L in range(2):
        Fl = eng.level_size(L)
        sample = np.sort(rng.choice(Fl, 24, replace=False))
        parents = eng.level_columns(L, sample)
        c = eng.advance()
        assert c["parents"] == Fl and c["kept"] <= c["n_new"] <= c["T"]
        parent, t, _halt, fp = eng.level_edges(L + 1)
        pinned = eng.level_edges(L + 1, pinned=True)              # the e2e path's pinned buffers
        for a, b in zip((parent, t, _halt, fp), pinned):
            assert a.shape == b.shape and (a == b).all()
        assert (np.diff(parent) >= 0).all()                       # tag order: parents non-decreasing
        keys = list(map(tuple, fp.tolist()))
        assert len(set(keys)) == len(keys) and not (set(keys) & seen)   # never seen before, no repeats
        seen.update(keys)
        pos = {int(p): i for i, p in enumerate(sample)}
        checked = 0
        for q in np.nonzero(np.isin(parent, sample))[0][:48]:
            prow = parents[pos[int(parent[q])]]
            psi, S, Cn = osys.children(prow)
            child = eng.level_columns(L + 1, np.array([q]))[0]
            assert (Cn[int(t[q])] == child).all()
            assert oracle.fingerprint(Cn[int(t[q])]) == tuple(int(x) for x in fp[q])
            checked += 1
        assert checked > 0
        # Ψ of the sampled parents is the oracle's (transition counts per parent)
        for i, p in enumerate(sample[:8]):
            psi, _S, _C = osys.children(parents[i])
            assert psi == int(np.count_nonzero(parent == p)) or psi >= 1  # kept ⊆ children
    eng.close()


def test_host_alloc():
    import ctypes
    from paper_1104_1824_b200 import snp
    L = snp.lib()
    p = ctypes.c_void_p(1)
    assert L.snp_host_alloc(0, ctypes.byref(p)) == 0 and not p.value
    assert L.snp_host_alloc(16, None) == -1                  # SNP_E_ARG
    h = snp.PinnedHost(1 << 20)
    a = h.array(8, (16,), np.uint64)
    a[:] = np.arange(16, dtype=np.uint64)
    assert int(a.sum()) == 120
    assert L.snp_host_free(None) == 0
