"""Oracle pins for SURVEY §8(f) NEXT-2 — general unary regular expressions.

The paper's rules use E = a^k (form (b-3)) and names general
regular expressions as future work.  Every regular language
over {a} is ultimately periodic, so the UNARY rule kind carries its
membership bits below t + P and repeats with period P above (oracle.cpp
``regex_matches``).  Pinned here against Python's own regular-expression
engine (``re.fullmatch`` on a^v) — applicability, all children of random
configurations (via the 2^n brute force of PAPER.md:111-113) — and against
the EXACT / PERIODIC kinds re-encoded as UNARY (identical trees).  CPU only."""
import re

import numpy as np
import pytest

import oracle
from oracle import brute
from paper_1104_1824_b200 import workloads as W


RE_MAX = 40  # Python's backtracking engine is exponential on long a^v for some (x|y)* forms


def _re_app(w):
    rx = w.meta["regex"]
    return lambda r, v: re.fullmatch(rx[r], "a" * v) is not None and v >= int(w.rules[r][4])


@pytest.mark.parametrize("seed", range(120))
def test_unary_applicability_and_children_match_python_re(seed):
    w = W.tiny_unary_system(seed)
    o = oracle.System.from_workload(w)
    app = _re_app(w)
    M = w.dense_M().tolist()
    rng = np.random.default_rng(seed)
    # the length-set builder agrees with Python's re on short strings ...
    for r, rx in enumerate(w.meta["regex"]):
        mem = W.unary_lengths(rx, 300)
        assert mem[:RE_MAX] == [re.fullmatch(rx, "a" * v) is not None for v in range(RE_MAX)]
    # ... and the oracle's ultimately periodic membership agrees with it to 299
    mem = [W.unary_lengths(rx, 300) for rx in w.meta["regex"]]
    for v in range(300):
        C = np.full(w.m, v, np.int32)
        tmp, d = o.applicability(C)
        for r in range(w.n):
            assert (tmp[r] > 0) == (mem[r][v] and v >= int(w.rules[r][4])), (seed, r, v, w.meta["regex"][r])
    for C in [w.C0] + [rng.integers(0, 12, size=w.m).astype(np.int32) for _ in range(4)]:  # counts < RE_MAX
        psi, S, Cn = o.children(C)
        bf = brute.children(w.rules.tolist(), M, [int(x) for x in C], app_fn=app)
        assert sorted(tuple(int(x) for x in s) for s in S) == sorted(s for s, _ in bf)
        assert sorted(tuple(int(x) for x in c) for c in Cn) == sorted(c for _, c in bf)


@pytest.mark.parametrize("seed", range(40))
def test_unary_bfs_matches_bruteforce_levels(seed):
    w = W.tiny_unary_system(seed)
    run = oracle.System.from_workload(w).explore(w.C0, depth=6)
    if run.status != 0:
        pytest.skip("capacity")
    app = _re_app(w)
    M = w.dense_M().tolist()
    seen = {tuple(int(x) for x in w.C0)}
    level = [tuple(int(x) for x in w.C0)]
    for d in range(1, run.num_levels):
        nxt = []
        for C in level:
            for _S, Cn in brute.children(w.rules.tolist(), M, list(C), app_fn=app):
                if Cn not in seen and Cn not in nxt:
                    nxt.append(Cn)
        seen |= set(nxt)
        assert {tuple(int(x) for x in c) for c in run.level(d)} == set(nxt)
        level = nxt


@pytest.mark.parametrize("enc", ["simulator", "textbook"])
def test_exact_and_periodic_equal_their_unary_encoding(enc):
    w = W.pi_system(enc)
    a = oracle.System.from_workload(w).explore(w.C0, depth=20)
    b = oracle.System.from_workload(W.as_unary(w)).explore(w.C0, depth=20)
    assert (a.configs == b.configs).all() and (a.parent == b.parent).all() and (a.t == b.t).all()


def test_random_system_unary_encoding():
    w = W.random_system(64, outdeg=8, k_nd=4, seed=5)
    L0 = W.level0_counts(w, 40, 5)
    a = oracle.System.from_workload(w).explore(L0, depth=3, dedup=1, count_bits=8)
    b = oracle.System.from_workload(W.as_unary(w)).explore(L0, depth=3, dedup=1, count_bits=8)
    assert a.status == b.status == 0
    assert (a.configs == b.configs).all() and (a.fp == b.fp).all()


def test_unary_validation():
    w = W.tiny_unary_system(1)
    bad = w.rules.copy()
    bad[0, 3] = 0  # period 0
    with pytest.raises(oracle.OracleError):
        oracle.System(w.m, bad, w.row_ptr, w.col, w.val, w.re_bits)
    with pytest.raises(oracle.OracleError):  # UNARY without membership rows
        oracle.System(w.m, w.rules, w.row_ptr, w.col, w.val, None)
