"""Oracle pins that do not come from Π: brute force on tiny random systems,
invariants of eq. (2), closed-form special cases, fingerprint linearity and
the thinning threshold.  CPU only."""
import numpy as np
import pytest

import oracle
from oracle import brute
from paper_1104_1824_b200 import workloads as W

SEEDS = range(300)


def _sys(w):
    return oracle.System.from_workload(w)


@pytest.mark.parametrize("seed", SEEDS)
def test_children_match_bruteforce(seed):
    """Mixed-radix enumeration = brute-force validity over
    all 2^n vectors; same children; plus invariants."""
    w = W.tiny_random_system(seed)
    M = w.dense_M()
    sys_ = _sys(w)
    rng = np.random.default_rng(seed)
    for C in [w.C0] + [rng.integers(0, 7, size=w.m).astype(np.int32) for _ in range(3)]:
        psi, S, Cn = sys_.children(C)
        bf = brute.children(w.rules.tolist(), M.tolist(), [int(x) for x in C])
        assert sorted(tuple(int(x) for x in s) for s in S) == sorted(s for s, _ in bf)
        assert sorted(tuple(int(x) for x in c) for c in Cn) == sorted(c for _, c in bf)
        tmp, d = sys_.applicability(C)
        halting = brute.is_halting(w.rules.tolist(), [int(x) for x in C])
        # child count = Π max(1, d_s), and 0 iff halting (readings A3, A5)
        assert psi == (0 if halting else int(np.prod(np.maximum(d, 1))))
        assert (psi == 0) == (d.max(initial=0) == 0)
        outdeg = np.zeros(w.m, np.int64)
        for s, _j in w.synapses:
            outdeg[s] += 1
        for t in range(psi):
            s_vec = S[t].astype(np.int64)
            # one rule per neuron with d_s > 0, none otherwise
            fired_per_neuron = np.bincount(w.rules[:, 0], weights=s_vec, minlength=w.m) if w.n else np.zeros(w.m)
            assert (fired_per_neuron == (d > 0)).all()
            # C' = C + S·M exactly; C' >= 0
            assert (Cn[t] == C.astype(np.int64) + s_vec @ M.astype(np.int64)).all()
            assert (Cn[t] >= 0).all()
            # spike-sum conservation: Σ C' - Σ C = Σ_{r∈S} (p_r·outdeg(σ(r)) - c_r)
            delta = sum(int(w.rules[r, 5]) * int(outdeg[w.rules[r, 0]]) - int(w.rules[r, 4])
                        for r in range(w.n) if s_vec[r])
            assert int(Cn[t].sum()) - int(C.sum()) == delta
        # mixed-radix order: first neuron with d>0 most significant
        keys = []
        for t in range(psi):
            key = []
            for s in range(w.m):
                rs = [r for r in range(w.n) if w.rules[r, 0] == s and tmp[r] > 0]
                key += [rs.index(r) for r in rs if S[t][r]]
            keys.append(tuple(key))
        assert keys == sorted(keys)


@pytest.mark.parametrize("seed", range(0, 300, 3))
@pytest.mark.parametrize("dedup", [0, 1])
def test_bfs_levels_match_bruteforce(seed, dedup):
    w = W.tiny_random_system(seed)
    levels, transitions = brute.bfs_levels(w.rules.tolist(), w.dense_M().tolist(), w.C0.tolist(), 4)
    run = _sys(w).explore(w.C0, depth=4, dedup=dedup)
    assert run.status == 0
    for d, lev in enumerate(levels):
        assert {tuple(int(x) for x in c) for c in run.level(d)} == lev
    assert int(run.counters.T.sum()) == transitions
    allc = [tuple(c) for c in run.configs]
    assert len(allc) == len(set(allc))  # no configuration appears twice
    for i in range(len(allc)):
        assert run.halting[i] == brute.is_halting(w.rules.tolist(), list(allc[i]))


@pytest.mark.parametrize("seed", range(40))
def test_tree_edges_reproduce_children(seed):
    """(parent, t) recorded per configuration regenerate it; parents appear in
    discovery order and t increases within a parent (reading A7)."""
    w = W.tiny_random_system(seed)
    sys_ = _sys(w)
    run = sys_.explore(w.C0, depth=4)
    for L in range(1, run.num_levels):
        prev = run.level(L - 1)
        lo = run.level_offsets[L]
        tags = []
        for q, C in enumerate(run.level(L)):
            p, t = int(run.parent[lo + q]), int(run.t[lo + q])
            _psi, _S, Cn = sys_.children(prev[p])
            assert (Cn[t] == C).all()
            tags.append((p, t))
        assert tags == sorted(tags)


def test_splitmix64_known_vector():
    # SplitMix64 seeded with 0 first outputs 0xE220A8397B1DCDAF (public test vector);
    # fp of the unit vector e_0 with seed 0 is that value | 1.
    e0 = np.zeros(4, np.int64)
    e0[0] = 1
    f0, _ = oracle.fingerprint(e0, seeds=(0, 0))
    assert f0 == 0xE220A8397B1DCDAF | 1


_M64 = (1 << 64) - 1


def _rotl64(x, r):
    return ((x << r) | (x >> (64 - r))) & _M64


def _murmur3_x64_128(key: bytes, seed: int, fmix) -> bytes:
    """MurmurHash3_x64_128 (Austin Appleby, public domain), written out here
    with the ORACLE's fmix64 as its finalizer: the oracle's thinning key and
    owner hash (readings A19, §8(e)) are exactly MurmurHash3's fmix64, so a
    wrong constant or shift in oracle.cpp:fmix64 breaks the published
    verification value below."""
    n = len(key)
    h1 = h2 = seed
    c1, c2 = 0x87C37B91114253D5, 0x4CF5AD432745937F
    nb = n // 16
    for i in range(nb):
        k1 = int.from_bytes(key[16 * i:16 * i + 8], "little")
        k2 = int.from_bytes(key[16 * i + 8:16 * i + 16], "little")
        k1 = (_rotl64((k1 * c1) & _M64, 31) * c2) & _M64
        h1 ^= k1
        h1 = (((_rotl64(h1, 27) + h2) & _M64) * 5 + 0x52DCE729) & _M64
        k2 = (_rotl64((k2 * c2) & _M64, 33) * c1) & _M64
        h2 ^= k2
        h2 = (((_rotl64(h2, 31) + h1) & _M64) * 5 + 0x38495AB5) & _M64
    tail, r = key[16 * nb:], n & 15
    k1 = k2 = 0
    if r > 8:
        for i in range(r - 1, 7, -1):
            k2 ^= tail[i] << (8 * (i - 8))
        h2 ^= (_rotl64((k2 * c2) & _M64, 33) * c1) & _M64
    if r > 0:
        for i in range(min(r, 8) - 1, -1, -1):
            k1 ^= tail[i] << (8 * i)
        h1 ^= (_rotl64((k1 * c1) & _M64, 31) * c2) & _M64
    h1 ^= n
    h2 ^= n
    h1 = (h1 + h2) & _M64
    h2 = (h2 + h1) & _M64
    h1, h2 = fmix(h1), fmix(h2)
    h1 = (h1 + h2) & _M64
    h2 = (h2 + h1) & _M64
    return h1.to_bytes(8, "little") + h2.to_bytes(8, "little")


def test_fmix64_pinned_by_murmur3_verification_value():
    """Pin of oracle fmix64 (oracle.cpp; thinning key A19, owner hash §8(e))
    against published values, not against another copy of itself:
      * SMHasher's VerificationTest for MurmurHash3_x64_128 (key i = bytes
        0..i-1 hashed with seed 256 - i, i = 0..255; the 4096 hash bytes hashed
        with seed 0; first 4 bytes little-endian) = 0x6384BA69 — the value
        SMHasher's hash table lists for "Murmur3F";
      * MurmurHash3_x64_128("The quick brown fox jumps over the lazy dog", 0)
        = 6c1b07bc7bbc4be3 47939ac4a93c437a (the widely quoted test vector);
      * fmix64(0) = 0 (every step maps 0 to 0)."""
    fmix = lambda k: int(oracle.fmix64(k))
    key = bytes(range(256))
    hashes = b"".join(_murmur3_x64_128(key[:i], 256 - i, fmix) for i in range(256))
    final = _murmur3_x64_128(hashes, 0, fmix)
    assert int.from_bytes(final[:4], "little") == 0x6384BA69
    assert _murmur3_x64_128(b"The quick brown fox jumps over the lazy dog", 0, fmix).hex() == \
        "6c1b07bc7bbc4be347939ac4a93c437a"
    assert fmix(0) == 0
    # a typo in either multiplier or shift breaks the verification value
    bad = lambda k: (fmix(k) ^ (k >> 40)) & _M64
    assert int.from_bytes(_murmur3_x64_128(hashes, 0, bad)[:4], "little") != 0x6384BA69


@pytest.mark.parametrize("seed", range(30))
def test_fingerprint_linearity(seed):
    # H(C + S·M) = H(C) + Σ_{r∈S} H(M_r) mod 2^64 (reading A18)
    w = W.tiny_random_system(seed)
    M = w.dense_M().astype(np.int64)
    sys_ = _sys(w)
    psi, S, Cn = sys_.children(w.C0)
    hC = oracle.fingerprint(w.C0.astype(np.int64))
    hr = [oracle.fingerprint(M[r]) for r in range(w.n)]
    for t in range(psi):
        exp = [hC[0], hC[1]]
        for r in range(w.n):
            if S[t][r]:
                exp = [(exp[0] + hr[r][0]) % 2**64, (exp[1] + hr[r][1]) % 2**64]
        assert tuple(exp) == oracle.fingerprint(Cn[t])


def test_thinning_tau_exact():
    for F, n in [(1, 2), (3, 7), (1 << 20, (1 << 20) + 1), (4194304, 16777000), (10**7, 3 * 10**8 + 17)]:
        assert oracle.thinning_tau(F, n) == (F << 64) // n


@pytest.mark.parametrize("seed", range(20))
def test_thinning_keeps_fingerprint_prefix(seed):
    """Reading A19: with a cap F < N_new, level 1 keeps exactly the new
    children with fmix64(fp0) < τ, in tag order; dropped ones are not visited."""
    w = W.random_system(24, outdeg=3, k_nd=6, seed=seed)
    L0 = W.level0_counts(w, 40, seed)
    sys_ = _sys(w)
    full = sys_.explore(L0, depth=1, dedup=1)
    n_new = int(full.counters.new[0])
    F = max(1, n_new // 3)
    thin = sys_.explore(L0, depth=1, dedup=1, frontier_target=F)
    tau = oracle.thinning_tau(F, n_new) if n_new > F else 1 << 64
    lvl = full.level(1)
    fps = full.fp[full.level_offsets[1]:full.level_offsets[2]]
    keep = [i for i in range(len(lvl)) if oracle.fmix64(int(fps[i][0])) < tau]
    assert (thin.level(1) == lvl[keep]).all()
    assert int(thin.counters.kept[0]) == len(keep)


def test_special_case_deterministic_single_path():
    # all d_s <= 1 → Ψ = 1: a plain textbook simulation (one path)
    w = W.random_system(16, outdeg=3, k_nd=0, seed=7)
    run = _sys(w).explore(w.C0, depth=15)
    assert (np.diff(run.level_offsets) <= 1).all()
    assert (run.counters.T <= 1).all()


def test_special_case_halting_root():
    # C0 with no applicable rule: the tree is {C0}, T = 0
    w = W.pi_system("simulator")
    run = _sys(w).explore(np.array([1, 0, 0], np.int32), depth=5)
    assert len(run.configs) == 1 and run.halting.tolist() == [1] and int(run.counters.T.sum()) == 0


@pytest.mark.parametrize("i,j,c,n0", [(2, 3, 3, 20), (0, 1, 2, 9), (1, 2, 1, 11)])
def test_special_case_single_periodic_rule(i, j, c, n0):
    # m = 1, one PERIODIC(i, j) rule consuming c: C0, C0-c, C0-2c, ... while the regex matches
    rules = np.array([[0, W.PERIODIC, i, j, c, 1]], np.int32)
    sys_ = oracle.System.from_dense(rules, np.array([[-c]]))
    run = sys_.explore(np.array([n0], np.int32), depth=50)
    exp = [n0]
    while True:
        v = exp[-1]
        if v >= i and (v - i) % j == 0 and v >= c:
            exp.append(v - c)
        else:
            break
    assert run.configs[:, 0].tolist() == exp


def test_overflow_and_capacity_errors():
    w = W.pi_system("simulator")
    s = _sys(w)
    r = s.explore(w.C0, depth=300, count_bits=8)   # the ≥-Π reaches 256 at depth 255
    assert r.status == oracle.OR_E_OVERFLOW
    r = s.explore(w.C0, depth=5, max_transitions=3)
    assert r.status == oracle.OR_E_CAPACITY


def test_validation_rejects_bad_systems():
    w = W.pi_system("simulator")
    M = w.dense_M()
    bad = M.copy()
    bad[0, 0] = -2          # M[r][σ(r)] != -c
    with pytest.raises(oracle.OracleError):
        oracle.System.from_dense(w.rules, bad)
    bad = M.copy()
    bad[1, 1] = 0           # rule 2 lacks the synapse (1,2) that its sibling rule 1 has
    with pytest.raises(oracle.OracleError):
        oracle.System.from_dense(w.rules, bad)
    rules = w.rules.copy()
    rules[[0, 2]] = rules[[2, 0]]  # not grouped by neuron
    with pytest.raises(oracle.OracleError):
        oracle.System.from_dense(rules, M[[2, 1, 0, 3, 4]])
