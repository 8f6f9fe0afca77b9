"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle on
identical seeded inputs.  Integer work ⇒ bit-exact: same configurations in
the same order, same (parent, t) edges, halting flags, fingerprints and
per-level counters."""
import numpy as np
import pytest

import oracle
from paper_1104_1824_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def snp():
    from paper_1104_1824_b200 import snp as _snp
    return _snp


def assert_same_tree(tree, ref, check_configs=True):
    assert ref.status == 0, ref.error
    assert tree.level_offsets.tolist() == ref.level_offsets.tolist()
    if check_configs:
        assert (tree.configs == ref.configs).all()
    assert (tree.parent == ref.parent).all()
    assert (tree.t == ref.t).all()
    assert (tree.halting == ref.halting).all()
    assert (tree.fp == ref.fp).all()
    assert tree.counters.T.tolist() == ref.counters.T.tolist()
    assert tree.counters.new.tolist() == ref.counters.new.tolist()
    assert tree.counters.kept.tolist() == ref.counters.kept.tolist()


# ---- config 1 / 2: the paper's Π ------------------------------------------
@pytest.mark.parametrize("enc", ["simulator", "textbook"])
@pytest.mark.parametrize("dedup", [0, 1])
@pytest.mark.parametrize("bits", [8, 16, 32])
def test_pi_config1(snp, enc, dedup, bits):
    w = W.pi_system(enc)
    tree = snp.System(w, count_bits=bits, dedup=dedup).explore(None, depth=12)
    ref = oracle.System.from_workload(w).explore(w.C0, depth=12, dedup=dedup, count_bits=bits)
    assert_same_tree(tree, ref)


def test_pi_worked_example(snp):
    w = W.pi_system("simulator")
    tree = snp.System(w).explore(None, depth=1)
    assert ["".join(map(str, s)) for s in tree.spiking_vectors(1)] == ["10110", "01110"]
    assert tree.level(1).tolist() == [[2, 1, 2], [1, 1, 2]]


def test_pi_config2_depth200(snp):
    w = W.pi_system("simulator")
    tree = snp.System(w, count_bits=8).explore(None, depth=200)
    ref = oracle.System.from_workload(w).explore(w.C0, depth=200, count_bits=8)
    assert_same_tree(tree, ref)
    assert tree.num_configs == 1000 and int(tree.counters.T.sum()) == 2779


def test_pi_overflow_uint8(snp):
    w = W.pi_system("simulator")
    with pytest.raises(snp.SnpError) as e:
        snp.System(w, count_bits=8).explore(None, depth=300)
    assert e.value.status == snp.SNP_E_OVERFLOW


def test_transition_budget(snp):
    w = W.pi_system("simulator")
    with pytest.raises(snp.SnpError) as e:
        snp.System(w, max_transitions=3).explore(None, depth=5)
    assert e.value.status == snp.SNP_E_CAPACITY


def test_halting_root(snp):
    w = W.pi_system("simulator")
    tree = snp.System(w).explore(np.array([[1, 0, 0]], np.int32), depth=5)
    assert tree.num_configs == 1 and tree.halting.tolist() == [1]


def test_invalid_system_rejected(snp):
    w = W.pi_system("simulator")
    bad = W.Workload(**{**w.__dict__})
    bad.val = w.val.copy()
    bad.val[0] = -2  # M[0][0] != -c
    with pytest.raises(snp.SnpError) as e:
        snp.System(bad)
    assert e.value.status == snp.SNP_E_INVALID_SYSTEM


def test_spiking_vectors_match_oracle(snp):
    w = W.random_system(40, outdeg=4, k_nd=8, seed=5)
    L0 = W.level0_counts(w, 50, 5)
    tree = snp.System(w).explore(L0, depth=2)
    sys_o = oracle.System.from_workload(w)
    for L in (1, 2):
        S = tree.spiking_vectors(L)
        prev = tree.level(L - 1)
        lo = tree.level_offsets[L]
        for q in range(0, S.shape[0], max(1, S.shape[0] // 40)):
            _psi, So, Co = sys_o.children(prev[tree.parent[lo + q]])
            assert (S[q] == So[tree.t[lo + q]]).all()
            assert (Co[tree.t[lo + q]] == tree.configs[lo + q]).all()


# ---- tiny random systems (every rule kind, p up to 2, empty neurons) -------
@pytest.mark.parametrize("seed", range(0, 400, 4))
def test_tiny_random(snp, seed):
    w = W.tiny_random_system(seed)
    dedup = seed % 2
    tree = snp.System(w, count_bits=32, dedup=dedup).explore(None, depth=5)
    ref = oracle.System.from_workload(w).explore(w.C0, depth=5, dedup=dedup)
    assert_same_tree(tree, ref)


# ---- random systems shaped like configs 3-5, scaled to oracle size ---------
@pytest.mark.parametrize("kernels", ["kc_global_e", "kc_tc"])
def test_random_parity_global_emit_words(snp, monkeypatch, kernels):
    monkeypatch.setenv("SNP_KERNELS", kernels)
    for m, F, bits, dedup in [(300, 700, 16, 0), (1024, 900, 8, 1)]:
        w = W.random_system(m, outdeg=8, k_nd=5, seed=m + 3)
        L0 = W.level0_counts(w, F, m + 3)
        tree = snp.System(w, count_bits=bits, dedup=dedup, frontier_target=F).explore(L0, depth=3)
        ref = oracle.System.from_workload(w).explore(L0, depth=3, dedup=dedup, count_bits=bits, frontier_target=F)
        assert_same_tree(tree, ref)


@pytest.mark.parametrize("m,F,depth,bits,dedup,target", [
    (64, 513, 4, 8, 1, 0),          # ragged F (not a multiple of 4 / 128)
    (300, 1000, 3, 16, 0, 700),     # thinning, exact dedup
    (1024, 600, 2, 32, 0, 900),     # config 3 shape (m = 1024, int32, exact)
    (1024, 1500, 3, 8, 1, 1500),    # config 4 dtype/dedup at m = 1024
    (2048, 257, 2, 8, 1, 0),        # m spanning many emit words
])
def test_random_system_parity(snp, m, F, depth, bits, dedup, target):
    w = W.random_system(m, outdeg=8, k_nd=5, seed=m + F)
    L0 = W.level0_counts(w, F, m + F)
    tree = snp.System(w, count_bits=bits, dedup=dedup, frontier_target=target).explore(L0, depth=depth)
    ref = oracle.System.from_workload(w).explore(L0, depth=depth, dedup=dedup, count_bits=bits,
                                                 frontier_target=target)
    assert_same_tree(tree, ref)


@pytest.mark.parametrize("kernels", ["", "expand_t", "kc_global_e", "no_tc", "kc_tc", "kc_tc,kc_global_e"])
def test_uint8_large_counts(snp, monkeypatch, kernels):
    """uint8 storage with counts well above the 32-entry register tables, so
    the table-fallback paths of K-a and K-c run; SNP_KERNELS=expand_t selects
    the 8-configurations-per-lane K-a instead of the 4-per-lane one,
    kc_global_e the K-c variant that gathers emit words from global memory,
    kc_tc the K-c whose output permutation runs on the tensor cores (level 1
    has > 8 sectors of children per block: its per-lane byte fallback)."""
    monkeypatch.setenv("SNP_KERNELS", kernels)
    w = W.random_system(700, outdeg=8, k_nd=5, seed=77)
    rng = np.random.default_rng(77)
    L0 = rng.integers(0, 72, size=(900, w.m)).astype(np.int32)
    L0[::7] = W.level0_counts(w, 900, 77)[::7]  # some rows in the usual range
    tree = snp.System(w, count_bits=8, dedup=1, frontier_target=800).explore(L0, depth=3)
    ref = oracle.System.from_workload(w).explore(L0, depth=3, dedup=1, count_bits=8, frontier_target=800)
    assert_same_tree(tree, ref)


@pytest.mark.parametrize("kernels", ["", "no_tc"])
def test_tc_expand_selected_and_equal(snp, monkeypatch, kernels):
    """The tensor-core K-a (k_expand_tc) is the path for uint8 systems of the
    generator family and for Π; SNP_KERNELS=no_tc runs the CUDA-core K-a.
    Both give the oracle's tree (ragged F: a partial last 128-configuration
    tile and a partial 64-configuration block; m not a multiple of 64)."""
    monkeypatch.setenv("SNP_KERNELS", kernels)
    want = 0 if kernels else snp.SNP_PATH_TC_EXPAND
    w = W.random_system(1000, outdeg=8, k_nd=6, seed=5)
    L0 = W.level0_counts(w, 1100, 5)
    L0[3::11] += 300  # 16/32-bit storage: counts >= 256 (the exact per-count lookups of the NARROW K-a)
    for bits in (8, 16, 32):
        L = L0 if bits > 8 else W.level0_counts(w, 1100, 5)
        eng = snp.System(w, count_bits=bits, dedup=1, frontier_target=1000)
        assert eng.kernel_paths == want
        tree = eng.explore(L, depth=4)
        ref = oracle.System.from_workload(w).explore(L, depth=4, dedup=1, count_bits=bits, frontier_target=1000)
        assert_same_tree(tree, ref)
    pi = W.pi_system("simulator")
    assert snp.System(pi, count_bits=8, dedup=0).kernel_paths == want
    assert snp.System(pi, count_bits=32, dedup=0).kernel_paths == want  # int32 storage: the NARROW TC K-a


def test_tc_expand_declined_when_not_applicable(snp):
    """k_expand_tc needs c <= 15, p <= 1 and at most 64 possibly
    nondeterministic neurons; otherwise the CUDA-core K-a runs (and agrees)."""
    w = W.random_system(300, outdeg=8, k_nd=80, seed=31)  # 80 ND neurons > 64
    L0 = W.level0_counts(w, 200, 31)
    L0[:, w.meta["nd_neurons"]] = 0  # below threshold at first: Ψ stays small for 3 levels
    eng = snp.System(w, count_bits=8, dedup=1, frontier_target=300)
    assert eng.kernel_paths == 0
    tree = eng.explore(L0, depth=3)
    ref = oracle.System.from_workload(w).explore(L0, depth=3, dedup=1, count_bits=8, frontier_target=300)
    assert_same_tree(tree, ref)
    w2 = W.random_system(200, outdeg=8, k_nd=3, seed=32)
    w2.rules[w2.rules[:, 0] == 5, 2] += 20  # neuron 5: thresholds and consumption above 15
    w2.rules[w2.rules[:, 0] == 5, 4] += 20
    w2 = W.Workload(name="bigc", m=w2.m, rules=w2.rules, row_ptr=w2.row_ptr,
                    col=w2.col, val=np.where(w2.val < 0, -w2.rules[np.repeat(np.arange(w2.n), np.diff(w2.row_ptr)), 4],
                                             w2.val).astype(np.int32),
                    C0=w2.C0, level0_range=w2.level0_range)
    eng2 = snp.System(w2, count_bits=8, dedup=1, frontier_target=300)
    assert eng2.kernel_paths == 0
    L0 = W.level0_counts(w2, 150, 32)
    L0[:, 5] = 30
    tree = eng2.explore(L0, depth=3)
    ref = oracle.System.from_workload(w2).explore(L0, depth=3, dedup=1, count_bits=8, frontier_target=300)
    assert_same_tree(tree, ref)


def test_config5_shape_parity(snp):
    """Config 5's system family at full width (m = 65536, n = 262144, k_nd = 7:
    mean Ψ ≈ 38 children per parent), scaled-down frontier, bit-exact."""
    cfg = W.CONFIGS[5]
    w = W.random_system(cfg["m"], outdeg=8, k_nd=cfg["k_nd"], seed=cfg["seed"])
    L0 = W.level0_counts(w, 64, cfg["seed"])
    tree = snp.System(w, count_bits=8, dedup=1, frontier_target=64).explore(L0, depth=2)
    ref = oracle.System.from_workload(w).explore(L0, depth=2, dedup=1, count_bits=8, frontier_target=64)
    assert ref.counters.T[0] > 20 * 64
    assert_same_tree(tree, ref)


def test_level0_duplicates_and_neuron_major_input(snp):
    w = W.random_system(100, outdeg=5, k_nd=4, seed=9)
    L0 = W.level0_counts(w, 200, 9)
    L0 = np.concatenate([L0, L0[:37], L0[5:9]])  # duplicates keep their first occurrence
    for dedup in (0, 1):
        ref = oracle.System.from_workload(w).explore(L0, depth=2, dedup=dedup)
        eng = snp.System(w, dedup=dedup)
        assert_same_tree(eng.explore(L0, depth=2), ref)
        nm = np.ascontiguousarray(L0.T.astype(np.uint16))
        c, keep = snp.configs_from_host(nm, layout=snp.SNP_LAYOUT_NEURON_MAJOR)
        assert_same_tree(eng.explore(c, depth=2), ref)


def test_level0_out_of_range(snp):
    w = W.random_system(50, seed=1)
    L0 = W.level0_counts(w, 10, 1)
    L0[3, 7] = 300
    with pytest.raises(snp.SnpError) as e:
        snp.System(w, count_bits=8).explore(L0, depth=1)
    assert e.value.status == snp.SNP_E_OVERFLOW


def _boundary_system():
    # σ0 (nondeterministic): a a*/a -> a (to σ1)  or  a a* -> λ ;  σ1 never fires.
    rules = np.array([[0, W.PERIODIC, 1, 1, 1, 1], [0, W.PERIODIC, 1, 1, 1, 0], [1, W.EXACT, 0, 0, 1, 1]], np.int32)
    M = np.array([[-1, 1], [-1, 0], [0, -1]], np.int32)
    return rules, M


def test_overflow_boundary_exact(snp):
    """Base child (first rules) overflows uint8 at σ1 (255 + 1) while the ND
    alternative (forget) stays at 255: only the kept child decides (reading
    A16).  Thinning to F = 1 picks one of the two by fingerprint; the seed is
    chosen with the oracle so that the in-range child is the kept one."""
    rules, M = _boundary_system()
    osys = oracle.System.from_dense(rules, M)
    L0 = np.array([[1, 255]], np.int32)
    chosen = None
    for s in range(200):
        ref = osys.explore(L0, depth=1, dedup=1, count_bits=8, frontier_target=1, seeds=(s, s + 7))
        if ref.status == 0 and ref.level(1).tolist() == [[0, 255]]:
            chosen = s
            break
    assert chosen is not None
    w = W.Workload(name="boundary", m=2, rules=rules, row_ptr=np.array([0, 2, 3, 4], np.int64),
                   col=np.array([0, 1, 0, 1], np.int32), val=np.array([-1, 1, -1, -1], np.int32), C0=L0[0],
                   level0_range=np.array([2, 256], np.int32))
    assert (w.dense_M() == M).all()
    tree = snp.System(w, count_bits=8, dedup=1, frontier_target=1, fp_seed=(chosen, chosen + 7)).explore(L0, depth=1)
    assert_same_tree(tree, ref)
    # without thinning both children are kept: the overflowing one is an error in both
    ref2 = osys.explore(L0, depth=1, dedup=1, count_bits=8)
    assert ref2.status == oracle.OR_E_OVERFLOW
    with pytest.raises(snp.SnpError) as e:
        snp.System(w, count_bits=8, dedup=1).explore(L0, depth=1)
    assert e.value.status == snp.SNP_E_OVERFLOW


def test_psi_capacity(snp):
    # 16 nondeterministic neurons above threshold: Ψ up to 4^16 per parent → budget error
    w = W.random_system(48, outdeg=12, k_nd=16, seed=21)
    L0 = np.full((4, 48), 14, np.int32)
    with pytest.raises(snp.SnpError) as e:
        snp.System(w, count_bits=8, dedup=1, max_transitions=1 << 20).explore(L0, depth=1)
    assert e.value.status == snp.SNP_E_CAPACITY


def test_incremental_api_and_digest(snp):
    w = W.random_system(256, outdeg=8, k_nd=5, seed=3)
    L0 = W.level0_counts(w, 400, 3)
    eng = snp.System(w, count_bits=8, dedup=1, frontier_target=500, keep_tree=0)
    eng.begin(L0)
    for _ in range(3):
        eng.advance()
    n, T, digest = eng.summary()
    ref = oracle.System.from_workload(w).explore(L0, depth=3, dedup=1, count_bits=8, frontier_target=500)
    assert n == len(ref.configs) and T == int(ref.counters.T.sum())
    assert digest == run_digest(ref)
    # the current level's counts are retained and match the oracle
    lvl = ref.level(3)
    idx = np.arange(0, len(lvl), 7)
    assert (eng.level_columns(3, idx) == lvl[idx]).all()


M64 = (1 << 64) - 1


def _fmix(k):
    k ^= k >> 33
    k = (k * 0xFF51AFD7ED558CCD) & M64
    k ^= k >> 33
    k = (k * 0xC4CEB9FE1A85EC53) & M64
    k ^= k >> 33
    return k


def run_digest(ref):
    """DESIGN.md §5 digest, computed here from the oracle's tree."""
    d = 0
    for L in range(ref.num_levels):
        lo = ref.level_offsets[L]
        for q in range(ref.level_offsets[L + 1] - lo):
            i = lo + q
            z = _fmix((L << 40) ^ q)
            z = _fmix(z ^ int(ref.fp[i][0]))
            z = _fmix(z ^ int(ref.fp[i][1]))
            z = _fmix(z ^ ((int(ref.parent[i]) + 1) & M64))
            z = _fmix(z ^ int(ref.t[i]))
            d = (d + z) & M64
    return d


def test_device_level0_generator_matches_host(snp):
    import torch
    w = W.random_system(300, seed=4)
    F = 1000
    buf = torch.empty((w.m, F), dtype=torch.uint8, device="cuda")
    snp.generate_level0_device(w, F, 77, buf.data_ptr(), 1, snp.SNP_LAYOUT_NEURON_MAJOR, F)
    torch.cuda.synchronize()
    host = W.level0_counts(w, F, 77, dtype=np.uint8)
    assert (buf.cpu().numpy().T == host).all()


def test_generic_neurons(snp):
    """Neurons the outcome tables cannot hold (> 15 rules; an EXACT exponent
    beyond the table width) take the rule-by-rule path inside the same kernels."""
    rng = np.random.default_rng(1)
    m = 40
    out = [np.sort(rng.choice([j for j in range(m) if j != s], 5, replace=False)) for s in range(m)]
    rules = []
    for s in range(m):
        if s == 3:
            for x in range(20):
                rules.append([s, W.PERIODIC, 2 + x, 3, 1 + x % 3, x % 2])
        elif s == 7:
            rules += [[s, W.EXACT, 700, 0, 5, 1], [s, W.PERIODIC, 2, 1, 1, 1]]
        else:
            rules.append([s, W.PERIODIC, 2, 1, 2, 1])
    rules = np.array(rules, np.int32)
    row_ptr, col, val = W._csr_from_rows(W.matrix_rows_from_rules(rules, out))
    C0 = rng.integers(0, 8, m).astype(np.int32)
    C0[3] = 30
    C0[7] = 700
    w = W.Workload("generic", m, rules, row_ptr, col, val, C0, np.full(m, 8, np.int32))
    for bits in (16, 32):
        for dedup in (0, 1):
            tree = snp.System(w, count_bits=bits, dedup=dedup, frontier_target=300).explore(None, depth=4)
            ref = oracle.System.from_workload(w).explore(C0, depth=4, dedup=dedup, count_bits=bits,
                                                         frontier_target=300)
            assert_same_tree(tree, ref)


# ---- the single-CTA small-frontier path (k_small_bfs) against the big path ---
@pytest.mark.parametrize("case", ["pi_sim", "pi_text", "tiny", "random_thin", "random_exact16", "grow"])
def test_small_path_equals_big_path(snp, monkeypatch, case):
    """k_small_bfs runs whole levels of small frontiers in one launch; the
    multi-kernel path (SNP_SMALL=0) and the oracle give the same tree."""
    kw, L0, depth = {}, None, 12
    if case == "pi_sim":
        w, depth = W.pi_system("simulator"), 60
    elif case == "pi_text":
        w = W.pi_system("textbook")
    elif case == "tiny":
        w = W.tiny_random_system(17)
        kw = dict(dedup=1)
    elif case == "random_thin":
        w = W.random_system(40, outdeg=4, k_nd=6, seed=2)
        L0, depth, kw = W.level0_counts(w, 30, 2), 6, dict(count_bits=8, dedup=1, frontier_target=40)
    elif case == "random_exact16":
        w = W.random_system(30, outdeg=4, k_nd=5, seed=3)
        L0, depth, kw = W.level0_counts(w, 20, 3), 5, dict(count_bits=16, dedup=0, frontier_target=100)
    else:  # frontier outgrows SMALL_F / SMALL_T: the levels move to the big path mid-run
        w = W.random_system(64, outdeg=6, k_nd=8, seed=4)
        L0, depth, kw = W.level0_counts(w, 8, 4), 4, dict(count_bits=8, dedup=1)
    monkeypatch.setenv("SNP_SMALL", "1")
    small = snp.System(w, **kw).explore(L0, depth=depth)
    monkeypatch.setenv("SNP_SMALL", "0")
    big = snp.System(w, **kw).explore(L0, depth=depth)
    ref = oracle.System.from_workload(w).explore(w.C0 if L0 is None else L0, depth=depth,
                                                 **{k: v for k, v in kw.items()})
    assert_same_tree(small, ref)
    assert_same_tree(big, ref)
    assert small.counters.halting.tolist() == big.counters.halting.tolist()


@pytest.mark.parametrize("bits", [16, 32])
@pytest.mark.parametrize("cap", ["", "16"])
def test_wide_counts_narrow_kc(snp, monkeypatch, bits, cap):
    """16/32-bit storage: K-c computes x in bytes (NARROW) and rewrites every
    x outside [0, 255] exactly (the overflow list); counts far above 255 take
    the per-parent exact fallback; SNP_OVF_CAP=16 overflows the list so the
    level is materialised again in full width.  Also SNP_KERNELS=kc_wide_exact
    (full width from the start).  Every variant gives the oracle's tree."""
    monkeypatch.setenv("SNP_OVF_CAP", cap)
    w = W.random_system(700, outdeg=8, k_nd=5, seed=91)
    rng = np.random.default_rng(91)
    L0 = W.level0_counts(w, 900, 91)
    L0[::5] = rng.integers(0, 900, size=L0[::5].shape)  # some rows far above one byte
    L0[1::9] += 240                                        # x near the byte boundary
    dedup = 0 if bits == 32 else 1
    for kern in ["", "kc_wide_exact"]:
        monkeypatch.setenv("SNP_KERNELS", kern)
        tree = snp.System(w, count_bits=bits, dedup=dedup, frontier_target=800).explore(L0, depth=3)
        ref = oracle.System.from_workload(w).explore(L0, depth=3, dedup=dedup, count_bits=bits, frontier_target=800)
        assert_same_tree(tree, ref)


@pytest.mark.parametrize("batch", ["", "1"])
def test_exact_dedup_verification(snp, monkeypatch, batch):
    """dedup = 0 compares every key match as full configurations: both
    verification paths (one CTA per match; SNP_VERIFY_BATCH=1 the batched
    two-pass one) agree with the oracle on a config-3-shaped system, and with
    6-bit child keys (SNP_KERNELS=fp_weak, tests only) distinct children
    share keys and the verification reports a collision (reading A18)."""
    monkeypatch.setenv("SNP_VERIFY_BATCH", batch)
    monkeypatch.setenv("SNP_SMALL", "0")
    w = W.random_system(1024, outdeg=8, k_nd=5, seed=123)
    L0 = W.level0_counts(w, 700, 123)
    tree = snp.System(w, count_bits=32, dedup=0, frontier_target=900).explore(L0, depth=3)
    ref = oracle.System.from_workload(w).explore(L0, depth=3, dedup=0, count_bits=32, frontier_target=900)
    assert_same_tree(tree, ref)
    monkeypatch.setenv("SNP_KERNELS", "fp_weak")
    with pytest.raises(snp.SnpError) as ei:
        snp.System(w, count_bits=32, dedup=0, frontier_target=900).explore(L0, depth=3)
    assert ei.value.status == snp.SNP_E_COLLISION


@pytest.mark.parametrize("bits", [8, 16])
@pytest.mark.parametrize("target", [40, 150, 1100])
def test_sparse_and_dense_kept_windows(snp, bits, target):
    """K-c's per-block child windows from nearly empty (a few kept children
    per 64-parent block: no whole 4-child quad, partial quads only) to more
    than 16 whole quads (whole store passes plus a tail pass)."""
    w = W.random_system(300, outdeg=8, k_nd=6, seed=321)
    L0 = W.level0_counts(w, 1000, 321)
    tree = snp.System(w, count_bits=bits, dedup=1, frontier_target=target).explore(L0, depth=3)
    ref = oracle.System.from_workload(w).explore(L0, depth=3, dedup=1, count_bits=bits, frontier_target=target)
    assert_same_tree(tree, ref)
