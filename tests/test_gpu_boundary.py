"""GPU tests of the §8(b) boundary calls added in round 2, through the C ABI
against the oracle: snp_spiking_vector / snp_level_spiking_vectors
("generate the succeeding C_k's and their corresponding S_k's"),
snp_frontier_copy, snp_level_all_edges (reading A17, Fig. 4),
the tree/system lifetime, the k_expand_tc width bound and the chunked level-0
upload."""
import gc

import numpy as np
import pytest

import oracle
from paper_1104_1824_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def snp():
    from paper_1104_1824_b200 import snp as _snp
    return _snp


def _global_rows(tree):
    return {tuple(c): i for i, c in enumerate(tree.configs.tolist())}


@pytest.mark.parametrize("case", ["pi", "tiny3", "tiny8", "random_thin", "random_exact", "generated"])
def test_all_edges_match_oracle(snp, case):
    kw = {}
    if case == "pi":
        w, L0, depth, dedup, bits, tgt = W.pi_system("simulator"), None, 8, 0, 32, 0
    elif case.startswith("tiny"):
        w = W.tiny_random_system(int(case[4:]))
        L0, depth, dedup, bits, tgt = None, 5, 1, 32, 0
    elif case == "random_thin":
        w = W.random_system(200, outdeg=8, k_nd=6, seed=11)
        L0, depth, dedup, bits, tgt = W.level0_counts(w, 300, 11), 3, 1, 8, 250
    elif case == "random_exact":
        w = W.random_system(120, outdeg=6, k_nd=5, seed=12)
        L0, depth, dedup, bits, tgt = W.level0_counts(w, 200, 12), 3, 0, 16, 150
    else:  # generated numbers: terminal transitions reach nothing (-1)
        w, L0, depth, dedup, bits, tgt = W.pi_system("textbook"), None, 12, 0, 32, 0
        kw = {"out_rule": 3}
    eng = snp.System(w, count_bits=bits, dedup=dedup, frontier_target=tgt, keep_all_edges=1, **kw)
    tree = eng.explore(L0, depth=depth)
    osys = oracle.System.from_workload(w)
    ref = osys.explore(w.C0 if L0 is None else L0, depth=depth, dedup=dedup, count_bits=bits, frontier_target=tgt,
                       **({"out_rule": kw["out_rule"]} if kw else {}))
    assert ref.status == 0
    assert tree.level_offsets.tolist() == ref.level_offsets.tolist()
    for L in range(1, tree.num_levels):
        parent, t, r = eng.level_all_edges(L)
        assert r.tolist() == ref.edge_ref[L - 1].tolist()
        # (parent, t) enumerate every transition of level L-1 in tag order
        psi = np.bincount(parent, minlength=tree.level_offsets[L] - tree.level_offsets[L - 1])
        assert psi.sum() == len(r) == ref.counters.T[L - 1]
        assert (t == np.concatenate([np.arange(k) for k in psi]).astype(np.uint64)).all() if len(r) else True


def test_all_edges_off_is_state_error(snp):
    w = W.pi_system("simulator")
    eng = snp.System(w)
    eng.explore(None, depth=2)
    with pytest.raises(snp.SnpError) as e:
        eng.level_all_edges(1)
    assert e.value.status == snp.SNP_E_STATE


def test_spiking_vector_of_a_configuration(snp):
    # C0 = <2,1,1> of Π has the two spiking vectors 10110, 01110
    w = W.pi_system("simulator")
    eng = snp.System(w, count_bits=8)
    assert "".join(map(str, eng.spiking_vector([2, 1, 1], 0))) == "10110"
    assert "".join(map(str, eng.spiking_vector([2, 1, 1], 1))) == "01110"
    with pytest.raises(snp.SnpError) as e:
        eng.spiking_vector([2, 1, 1], 2)          # t >= Ψ = 2
    assert e.value.status == snp.SNP_E_ARG
    with pytest.raises(snp.SnpError) as e:
        eng.spiking_vector([1, 0, 0], 0)          # halting: no spiking vector (reading A5)
    assert e.value.status == snp.SNP_E_ARG
    # random systems: every t of sampled configurations = the oracle's S_t
    wr = W.random_system(500, outdeg=8, k_nd=6, seed=3)
    er = snp.System(wr, count_bits=8)
    osys = oracle.System.from_workload(wr)
    L0 = W.level0_counts(wr, 12, 3)
    for C in L0:
        psi, S, _C = osys.children(C)
        for t in sorted({0, psi - 1, psi // 2}):
            assert (er.spiking_vector(C, t) == S[t]).all()


def test_level_spiking_vectors_without_keep_tree(snp):
    w = W.random_system(300, outdeg=8, k_nd=6, seed=4)
    L0 = W.level0_counts(w, 256, 4)
    eng = snp.System(w, count_bits=8, dedup=1, frontier_target=300, keep_tree=0)
    osys = oracle.System.from_workload(w)
    eng.begin(L0)
    for L in (1, 2, 3):
        prev = eng.frontier_copy()[0]                # parents of level L (the current frontier)
        eng.advance()
        C, parent, t = eng.frontier_copy()
        idx = np.arange(0, len(C), 7)
        S = eng.level_spiking_vectors(L, idx)
        for k, q in enumerate(idx):
            _psi, So, Co = osys.children(prev[parent[q]])
            assert (S[k] == So[t[q]]).all() and (Co[t[q]] == C[q]).all()
    with pytest.raises(snp.SnpError) as e:
        eng.level_spiking_vectors(2, [0])            # its parent level was released (keep_tree = 0)
    assert e.value.status == snp.SNP_E_STATE


def test_frontier_copy_matches_tree(snp):
    w = W.random_system(150, outdeg=6, k_nd=5, seed=6)
    L0 = W.level0_counts(w, 100, 6)
    eng = snp.System(w, count_bits=16, dedup=0, frontier_target=120)
    tree = eng.explore(L0, depth=3)
    C, parent, t = eng.frontier_copy()
    lo = tree.level_offsets[-2]
    assert (C == tree.level(tree.num_levels - 1)).all()
    assert (parent == tree.parent[lo:]).all() and (t == tree.t[lo:]).all()


def test_tree_outlives_system(snp):
    w = W.random_system(64, outdeg=4, k_nd=4, seed=8)
    L0 = W.level0_counts(w, 50, 8)
    eng = snp.System(w, count_bits=8, dedup=1)
    tree = eng.explore(L0, depth=2)
    ref = oracle.System.from_workload(w).explore(L0, depth=2, dedup=1, count_bits=8)
    eng.close()                                      # snp_system_free: the tree keeps the system alive
    del eng
    gc.collect()
    assert (tree.configs == ref.configs).all()
    assert tree.spiking_vectors(1).shape[0] == tree.level_offsets[2] - tree.level_offsets[1]
    tree.close()


def test_level_edges_halting_of_unexpanded_level(snp):
    w = W.pi_system("simulator")
    eng = snp.System(w)
    eng.begin(None)
    eng.advance()
    with pytest.raises(snp.SnpError) as e:
        eng.level_edges(1)                           # level 1 is not classified yet
    assert e.value.status == snp.SNP_E_STATE
    parent, t, h, fp = eng.level_edges(1, halting=False)
    assert h is None and parent.tolist() == [0, 0]
    assert eng.level_edges(0)[2].tolist() == [0]     # level 0 was expanded: its flags are known


def test_pinned_views_survive_regrowth_and_close(snp):
    w = W.random_system(64, outdeg=4, k_nd=5, seed=9)
    L0 = W.level0_counts(w, 40, 9)
    eng = snp.System(w, count_bits=8, dedup=1, keep_tree=1)
    eng.explore(L0, depth=3)
    p1, t1, _h, fp1 = eng.level_edges(1, pinned=True, halting=False)
    keep = (p1.copy(), fp1.copy())
    eng.reserve_edges(10 * eng.level_size(3) + 1000)  # replaces the pinned block
    big = eng.level_edges(3, pinned=True, halting=False)
    eng.close()
    del eng
    gc.collect()
    assert (p1 == keep[0]).all() and (fp1 == keep[1]).all()   # old views still own their memory
    assert big[0].shape[0] > 0


def test_tc_expand_width_bound(snp):
    """k_expand_tc's s32 accumulators are exact only for m <= 2^19 (DESIGN.md
    §7): one neuron more and the CUDA-core K-a runs, still equal to the oracle."""
    m = (1 << 19) + 64
    w = W.random_system(m, outdeg=2, k_nd=2, seed=13)
    eng = snp.System(w, count_bits=8, dedup=1, frontier_target=24)
    assert eng.kernel_paths == 0
    L0 = W.level0_counts(w, 12, 13)
    tree = eng.explore(L0, depth=1)
    ref = oracle.System.from_workload(w).explore(L0, depth=1, dedup=1, count_bits=8, frontier_target=24)
    assert tree.level_offsets.tolist() == ref.level_offsets.tolist()
    assert (tree.fp == ref.fp).all() and (tree.parent == ref.parent).all() and (tree.t == ref.t).all()


def test_chunked_level0_upload(snp, monkeypatch):
    """snp_begin's multi-chunk host upload (two staging buffers, event
    ping-pong): >= 3 chunks and a partial last chunk, against the oracle."""
    w = W.random_system(256, outdeg=8, k_nd=5, seed=14)
    F = 64 * 7 + 19
    L0 = W.level0_counts(w, F, 14).astype(np.uint8)
    monkeypatch.setenv("SNP_UPLOAD_CHUNK_BYTES", str(64 * 2 * 256))   # 128 rows per chunk: 4 chunks
    eng = snp.System(w, count_bits=8, dedup=1, frontier_target=F)
    tree = eng.explore(L0, depth=2)
    ref = oracle.System.from_workload(w).explore(L0.astype(np.int32), depth=2, dedup=1, count_bits=8,
                                                 frontier_target=F)
    assert (tree.configs == ref.configs).all() and (tree.fp == ref.fp).all()
    assert tree.counters.T.tolist() == ref.counters.T.tolist()


def test_host_alloc(snp):
    import ctypes
    L = snp.lib()
    p = ctypes.c_void_p(1)
    assert L.snp_host_alloc(0, ctypes.byref(p)) == 0 and not p.value
    assert L.snp_host_alloc(16, None) == -1                  # SNP_E_ARG
    h = snp.PinnedHost(1 << 20)
    a = h.array(8, (16,), np.uint64)
    a[:] = np.arange(16, dtype=np.uint64)
    del h                                                    # the view keeps the block alive
    gc.collect()
    assert int(a.sum()) == 120
    assert L.snp_host_free(None) == 0
