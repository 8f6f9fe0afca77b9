"""Oracle pins for SURVEY §8(f) NEXT-4 — single-path sampling with an input
spike train (Def. 1 `in`).  Each walker follows one
computation path, taking the child t = u mod Ψ (counter-based u, reading A25)
in Alg. 2's enumeration order; the input neuron receives train[k] spikes at
step k.  Pinned against the 2^n brute force (every step lands on a valid
child), uniformity of t over the children, the BFS tree of deterministic
systems (one path), and the closed form of a rule-less input neuron."""
import numpy as np
import pytest

import oracle
from oracle import brute
from paper_1104_1824_b200 import workloads as W


def _path(o, C0, seed, steps, w=0, **kw):
    """configurations after 0..steps steps of walker w (prefix property)."""
    out = [np.array(C0, np.int64)]
    for k in range(1, steps + 1):
        C = np.tile(np.asarray(C0, np.int32), (w + 1, 1))
        Ck, hs = o.sample(C, seed, k, **kw)
        out.append(Ck[w].astype(np.int64))
    return out


@pytest.mark.parametrize("seed", range(40))
def test_every_step_is_a_valid_child(seed):
    w = W.tiny_random_system(seed, m_max=4, rules_max=3, count_max=6)
    o = oracle.System.from_workload(w)
    M = w.dense_M().tolist()
    path = _path(o, w.C0, seed, 8, w=seed % 3)
    for a, b in zip(path, path[1:]):
        kids = {c for _, c in brute.children(w.rules.tolist(), M, [int(x) for x in a])}
        if not kids:  # halting: the walker stays
            assert (a == b).all()
        else:
            assert tuple(int(x) for x in b) in kids


def test_choice_is_uniform_over_children():
    # one step of 24000 walkers from a configuration with Ψ = 12 children
    w = W.random_system(16, outdeg=3, k_nd=3, seed=2)
    o = oracle.System.from_workload(w)
    C = None
    for s in range(2000):
        cand = W.level0_counts(w, 1, 100 + s)[0]
        psi, S, Cn = o.children(cand)
        if psi >= 8:
            C = cand
            break
    assert C is not None
    psi, S, Cn = o.children(C)
    Wn = 3000 * psi
    out, hs = o.sample(np.tile(C, (Wn, 1)), 12345, 1)
    idx = {tuple(int(x) for x in c): i for i, c in enumerate(Cn)}
    counts = np.bincount([idx[tuple(int(x) for x in r)] for r in out], minlength=psi)
    chi2 = float(((counts - Wn / psi) ** 2 / (Wn / psi)).sum())
    assert chi2 < psi + 6 * np.sqrt(2 * psi) + 10  # far inside any sane rejection region
    assert (counts > 0).all()


def test_deterministic_system_sample_equals_bfs():
    w = W.random_system(40, outdeg=4, k_nd=0, seed=9)
    o = oracle.System.from_workload(w)
    run = o.explore(w.C0, depth=30)
    L = run.num_levels
    assert all(run.level_offsets[i + 1] - run.level_offsets[i] <= 1 for i in range(L))
    path = _path(o, w.C0, 7, L - 1)
    for d in range(L):
        if run.level_offsets[d + 1] > run.level_offsets[d]:
            assert (run.level(d)[0] == path[d]).all()


def test_input_neuron_closed_form():
    # Π with σ1 as the input neuron: every step is a valid child plus train[k]
    # spikes at σ1
    w = W.pi_system("simulator")
    rules = w.rules
    o = oracle.System.from_workload(w)
    train = np.array([1, 0, 2, 1, 0, 0, 3], np.int32)
    M = w.dense_M().tolist()
    for seed in range(5):
        path = _path(o, w.C0, seed, 7, input_neuron=0, train=train)
        for k, (a, b) in enumerate(zip(path, path[1:])):
            kids = {c for _, c in brute.children(rules.tolist(), M, [int(x) for x in a])} or {tuple(int(x) for x in a)}
            shifted = {tuple(c[j] + (int(train[k]) if j == 0 else 0) for j in range(w.m)) for c in kids}
            assert tuple(int(x) for x in b) in shifted
    # a rule-less, synapse-less input neuron just accumulates the train
    from paper_1104_1824_b200.workloads import Workload
    acc = Workload(name="acc", m=1, rules=np.zeros((0, 6), np.int32), row_ptr=np.zeros(1, np.int64),
                   col=np.zeros(0, np.int32), val=np.zeros(0, np.int32), C0=np.array([3], np.int32),
                   level0_range=np.array([4], np.int32))
    oa = oracle.System.from_workload(acc)
    out, hs = oa.sample(np.array([[3]], np.int32), 1, 10, input_neuron=0, train=train)
    assert out[0, 0] == 3 + train.sum() and hs[0] == len(train)
