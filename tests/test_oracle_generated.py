"""Oracle pins for SURVEY §8(f) NEXT-1 — generated numbers.

The result of a computation of a generating SNP system is the number of steps
between the first two spikes its output neuron sends to the environment
(PAPER.md:89 `out`; Π "generates all numbers in N - {1}" and
"this generated set is the result of the computation").  The oracle computes
the set by a BFS over the augmented state (C, A), A = steps since the first
output spike (oracle.cpp ``oracle_explore_gen``).  It is pinned here against

* an independent path enumerator (``brute.generated_numbers_paths``: every
  computation path of length T, no dedup, no mixed-radix decoding, no
  augmented state) on Π and on tiny random systems;
* the paper's claim for Π: N − {1}, i.e. {2, …, T−1} within T
  steps under the textbook encoding (reading A1; the simulator encoding also
  generates 1), up to T = 200 (config 2);
* the structure of the augmented state (A = 0 until the first output spike,
  then the level distance to it). CPU only.
"""
import numpy as np
import pytest

import oracle
from oracle import brute
from paper_1104_1824_b200 import workloads as W


def _numbers_brute(w, out_rule, T):
    return brute.generated_numbers_paths(w.rules.tolist(), w.dense_M().tolist(), [int(x) for x in w.C0],
                                         out_rule, T)


@pytest.mark.parametrize("enc", ["textbook", "simulator"])
@pytest.mark.parametrize("T", [1, 2, 3, 5, 8, 12, 16])
def test_pi_numbers_match_path_enumeration(enc, T):
    w = W.pi_system(enc)
    run = oracle.System.from_workload(w).explore(w.C0, depth=T, out_rule=w.meta["out_rule"])
    assert run.status == 0
    assert run.numbers == _numbers_brute(w, w.meta["out_rule"], T)


@pytest.mark.parametrize("enc,lo", [("textbook", 2), ("simulator", 1)])
def test_pi_generates_N_minus_1_to_depth_200(enc, lo):
    # config 2 (BASELINE.json): Π to depth 200; PAPER.md:99 — N − {1} (textbook)
    w = W.pi_system(enc)
    run = oracle.System.from_workload(w).explore(w.C0, depth=200, out_rule=w.meta["out_rule"])
    assert run.status == 0
    assert run.numbers == set(range(lo, 200))
    if enc == "textbook":
        assert len(run.numbers) == 198


def test_augmented_column_semantics():
    """A = 0 on every state whose path has no output spike yet; after the first
    spike at step t1 the state at level k carries A = k − t1; no stored state
    has a second spike behind it (those children are terminal)."""
    w = W.pi_system("textbook")
    out = w.meta["out_rule"]
    o = oracle.System.from_workload(w)
    run = o.explore(w.C0, depth=30, out_rule=out)
    lev = np.searchsorted(run.level_offsets, np.arange(len(run.configs)), side="right") - 1
    for q in range(len(run.configs)):
        L = lev[q]
        a = int(run.configs[q, -1])
        assert 0 <= a <= L
        if L == 0:
            assert a == 0
            continue
        parent = run.configs[run.level_offsets[L - 1] + run.parent[q]]
        pa = int(parent[-1])
        # the spiking vector that produced q from its parent
        psi, S, Cn = o.children(parent[:-1].astype(np.int32))
        t = int(run.t[q])
        fired = bool(S[t][out])
        assert (Cn[t] == run.configs[q, :-1]).all()
        assert not (pa >= 1 and fired)
        assert a == (pa + 1 if pa >= 1 else (1 if fired else 0))


def test_no_output_rule_is_the_plain_tree():
    w = W.pi_system("simulator")
    o = oracle.System.from_workload(w)
    a = o.explore(w.C0, depth=12)
    b = o.explore(w.C0, depth=12, out_rule=None)
    assert (a.configs == b.configs).all() and a.numbers == b.numbers == set()


@pytest.mark.parametrize("chunk", range(10))
def test_tiny_random_numbers_match_path_enumeration(chunk):
    """200 tiny random systems × every spiking rule as the output rule, T = 10
    (about 80 of the ≈590 cases generate at least one number)."""
    T, nonempty = 10, 0
    for seed in range(20 * chunk, 20 * chunk + 20):
        w = W.tiny_random_system(seed, m_max=4, rules_max=3, count_max=6)
        for out in [r for r in range(w.n) if int(w.rules[r][5]) > 0]:
            run = oracle.System.from_workload(w).explore(w.C0, depth=T, out_rule=out)
            if run.status != 0:
                continue
            assert run.numbers == _numbers_brute(w, out, T), (seed, out)
            nonempty += bool(run.numbers)
            # the same set under fingerprint dedup (reading A18)
            run1 = oracle.System.from_workload(w).explore(w.C0, depth=T, out_rule=out, dedup=1)
            assert run1.numbers == run.numbers
    assert nonempty > 0
