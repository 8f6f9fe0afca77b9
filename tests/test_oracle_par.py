"""Pins of oracle_explore_par (oracle.cpp) — the parent-parallel form of the
BFS used for configs 3 and 5 at their stated sizes — against oracle_explore,
the sequential definition (itself pinned to the paper's worked example, the
printed run, brute force and closed forms in test_oracle_*.py): identical
trees (level sizes, parents, t, fingerprints, halting flags, rows, counters)
on the shapes of the parity suite, for every thread count."""
import numpy as np
import pytest

import oracle
from paper_1104_1824_b200 import workloads as W


def _same(a, b):
    assert a.status == b.status == 0, (a.error, b.error)
    assert a.level_offsets.tolist() == b.level_offsets.tolist()
    assert (a.parent == b.parent).all() and (a.t == b.t).all()
    assert (a.fp == b.fp).all() and (a.halting == b.halting).all()
    assert a.counters.T.tolist() == b.counters.T.tolist()
    assert a.counters.new.tolist() == b.counters.new.tolist()
    assert a.counters.kept.tolist() == b.counters.kept.tolist()
    assert (b.rows(np.arange(len(a.configs))) == a.configs).all()


@pytest.mark.parametrize("m,F,depth,bits,dedup,target,threads", [
    (64, 513, 4, 8, 1, 0, 3),
    (300, 1000, 3, 16, 0, 700, 4),
    (1024, 600, 2, 32, 0, 900, 8),
    (400, 800, 4, 8, 1, 800, 2),
    (40, 300, 6, 32, 0, 0, 5),
])
def test_par_equals_sequential_random(m, F, depth, bits, dedup, target, threads):
    w = W.random_system(m, outdeg=8 if m > 8 else 3, k_nd=5, seed=m + F)
    L0 = W.level0_counts(w, F, m + F)
    s = oracle.System.from_workload(w)
    a = s.explore(L0, depth, dedup=dedup, count_bits=bits, frontier_target=target)
    b = s.explore_par(L0, depth, dedup=dedup, count_bits=bits, frontier_target=target, n_threads=threads)
    _same(a, b)


@pytest.mark.parametrize("seed", range(0, 60, 3))
def test_par_equals_sequential_tiny(seed):
    w = W.tiny_random_system(seed)
    s = oracle.System.from_workload(w)
    for dedup in (0, 1):
        a = s.explore(w.C0, 6, dedup=dedup)
        b = s.explore_par(w.C0, 6, dedup=dedup, n_threads=1 + seed % 4)
        if a.status != 0:
            assert b.status == a.status
            continue
        _same(a, b)


def test_par_pi_closed_form():
    w = W.pi_system("simulator")
    b = oracle.System.from_workload(w).explore_par(w.C0, 200, count_bits=8, n_threads=4)
    assert b.level_offsets[-1] == 1000 and int(b.counters.T.sum()) == 2779   # SURVEY §8(c) closed forms


def test_par_errors_match():
    w = W.pi_system("simulator")
    s = oracle.System.from_workload(w)
    assert s.explore_par(w.C0, 300, count_bits=8).status == oracle.OR_E_OVERFLOW
    assert s.explore_par(w.C0, 5, max_transitions=3).status == oracle.OR_E_CAPACITY
