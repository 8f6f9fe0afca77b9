"""Oracle pins for SURVEY §8(f) NEXT-3 — SN P systems WITH delays (reading
A26: a rule E/a^c -> a^p; d fired at step t emits at t + d and keeps its
neuron closed at t .. t+d-1, spikes sent to a closed neuron are lost).  The
state is [C | τ | π] (width 3m).  Pinned against:
  * the delay-free tree when every d = 0 (the paper's eq. (2) semantics);
  * an independent brute force (every subset of rules, an event list of
    emissions, synapses read from the dense M) on tiny random systems with
    random delays and random closed neurons;
  * closed forms: a delayed chain delivers after d + 1 steps; a spike sent to
    a closed neuron is lost; a closed neuron alone still has one child."""

import numpy as np
import pytest

import oracle
from paper_1104_1824_b200 import workloads as W
from paper_1104_1824_b200.workloads import Workload


def _matches(rule, v):
    _, kind, a, b, c, _ = rule
    if kind == W.EXACT:
        ok = v == a
    else:
        ok = v >= a and (v - a) % b == 0
    return ok and v >= c


def brute_children_delay(rules, M, delays, X):
    """Set of child states by brute force over every subset of rules."""
    n, m = len(rules), len(M[0]) if M else 0
    C, tau, pi = list(X[:m]), list(X[m:2 * m]), list(X[2 * m:])
    targets = [sorted({j for r in range(n) if rules[r][0] == s for j in range(m) if j != s and M[r][j] != 0})
               for s in range(m)]
    app = [tau[rules[r][0]] == 0 and _matches(rules[r], C[rules[r][0]]) for r in range(n)]
    open_with_rules = {rules[r][0] for r in range(n) if app[r]}
    if not open_with_rules and all(t == 0 for t in tau):
        return set()  # halting
    kids = set()
    for mask in range(1 << n):
        chosen = [r for r in range(n) if mask >> r & 1]
        if any(not app[r] for r in chosen):
            continue
        neurons = [rules[r][0] for r in chosen]
        if len(set(neurons)) != len(neurons) or set(neurons) != open_with_rules:
            continue
        Cn, tn, pn = list(C), list(tau), list(pi)
        events = []
        for s in range(m):
            if tau[s] >= 1:
                tn[s] = tau[s] - 1
                if tn[s] == 0:
                    events.append((s, pi[s]))
                    pn[s] = 0
        for r in chosen:
            s, _, _, _, c, p = rules[r]
            Cn[s] -= c
            if delays[r] == 0:
                events.append((s, p))
            else:
                tn[s], pn[s] = delays[r], p
        for s, k in events:
            for j in targets[s]:
                if tn[j] == 0:
                    Cn[j] += k
        kids.add(tuple(Cn + tn + pn))
    return kids


@pytest.mark.parametrize("enc", ["simulator", "textbook"])
@pytest.mark.parametrize("dedup", [0, 1])
def test_zero_delays_is_the_delay_free_tree(enc, dedup):
    w = W.pi_system(enc)
    o = oracle.System.from_workload(w)
    a = o.explore_delay(np.zeros(w.n, np.int32), w.C0, 15, dedup=dedup)
    b = o.explore(w.C0, 15, dedup=dedup)
    assert a.status == b.status == 0
    assert (a.level_offsets == b.level_offsets).all()
    assert (a.configs[:, :w.m] == b.configs).all() and (a.configs[:, w.m:] == 0).all()
    assert (a.parent == b.parent).all() and (a.t == b.t).all() and (a.halting == b.halting).all()
    assert (a.fp == b.fp).all()  # zero tails add nothing to the fingerprint
    assert (a.counters.T == b.counters.T).all()


def test_zero_delays_random_system_with_thinning():
    w = W.random_system(60, outdeg=5, k_nd=4, seed=3)
    o = oracle.System.from_workload(w)
    L0 = W.level0_counts(w, 40, 3)
    a = o.explore_delay(np.zeros(w.n, np.int32), L0, 4, dedup=1, count_bits=8, frontier_target=50)
    b = o.explore(L0, 4, dedup=1, count_bits=8, frontier_target=50)
    assert (a.configs[:, :w.m] == b.configs).all() and (a.level_offsets == b.level_offsets).all()
    assert (a.counters.kept == b.counters.kept).all()


@pytest.mark.parametrize("seed", range(150))
def test_children_match_brute_force(seed):
    w = W.tiny_random_system(seed, m_max=4, rules_max=3, count_max=5)
    rng = np.random.default_rng(seed + 77)
    delays = rng.integers(0, 3, size=w.n).astype(np.int32)
    M = w.dense_M().tolist()
    o = oracle.System.from_workload(w)
    for trial in range(4):
        C = rng.integers(0, 6, size=w.m)
        tau = np.where(rng.random(w.m) < 0.3, rng.integers(1, 3, size=w.m), 0)
        pi = np.where(tau > 0, rng.integers(0, 3, size=w.m), 0)
        X = np.concatenate([C, tau, pi]).astype(np.int32)
        psi, S, Y = o.children_delay(delays, X)
        kids = brute_children_delay(w.rules.tolist(), M, delays.tolist(), X.tolist())
        assert {tuple(int(v) for v in y) for y in Y} == kids
        assert psi == len(Y) and psi >= len(kids)  # distinct choices may coincide
        # each spiking vector: one rule per open neuron with an applicable rule
        for srow in S:
            fired = [w.rules[r][0] for r in range(w.n) if srow[r]]
            assert len(fired) == len(set(fired))
            assert all(tau[s] == 0 for s in fired)


def _chain(d):
    # σ0 (1 spike, a -> a; d) -> σ1 (no rules)
    rules = np.array([[0, W.EXACT, 1, 0, 1, 1]], np.int32)
    rows = W.matrix_rows_from_rules(rules, [np.array([1]), np.array([], np.int64)])
    rp, col, val = W._csr_from_rows(rows)
    return Workload(name=f"chain{d}", m=2, rules=rules, row_ptr=rp, col=col, val=val,
                    C0=np.array([1, 0], np.int32), level0_range=np.array([2, 1], np.int32))


@pytest.mark.parametrize("d", [0, 1, 2, 5])
def test_delayed_chain_delivers_after_d_plus_1_steps(d):
    w = _chain(d)
    o = oracle.System.from_workload(w)
    r = o.explore_delay(np.array([d], np.int32), w.C0, 20)
    assert r.status == 0
    sizes = np.diff(r.level_offsets)
    assert (sizes[:d + 2] == 1).all() and sizes[d + 2:].sum() == 0  # one path, d + 1 steps
    last = r.configs[-1]
    assert list(last) == [0, 1, 0, 0, 0, 0] and r.halting[-1] == 1
    assert all(r.halting[:-1] == 0)
    for k in range(1, d + 1):  # while closed: τ counts down from d, π = 1 pending
        assert list(r.configs[k]) == [0, 0, d - k + 1, 0, 1, 0]


def test_spike_to_a_closed_neuron_is_lost():
    # σ0 (1 spike, a -> a; 0) -> σ1 (1 spike, a -> a; D) -> σ2 (no rules)
    def system(D):
        rules = np.array([[0, W.EXACT, 1, 0, 1, 1], [1, W.PERIODIC, 1, 1, 1, 1]], np.int32)
        rows = W.matrix_rows_from_rules(rules, [np.array([1]), np.array([2]), np.array([], np.int64)])
        rp, col, val = W._csr_from_rows(rows)
        return Workload(name="lost", m=3, rules=rules, row_ptr=rp, col=col, val=val,
                        C0=np.array([1, 1, 0], np.int32), level0_range=np.array([2, 2, 1], np.int32))
    w = system(2)
    o = oracle.System.from_workload(w)
    r = o.explore_delay(np.array([0, 2], np.int32), w.C0, 10)
    # step 1: σ1 closes (τ = 2) so σ0's spike is lost; step 3: σ1 emits into σ2
    assert [list(c) for c in r.configs] == [[1, 1, 0, 0, 0, 0, 0, 0, 0], [0, 0, 0, 0, 2, 0, 0, 1, 0],
                                            [0, 0, 0, 0, 1, 0, 0, 1, 0], [0, 0, 1, 0, 0, 0, 0, 0, 0]]
    assert list(r.halting) == [0, 0, 0, 1]
    # without the delay σ1 keeps the spike and fires twice
    r0 = o.explore_delay(np.array([0, 0], np.int32), w.C0, 10)
    assert [list(c[:3]) for c in r0.configs] == [[1, 1, 0], [0, 1, 1], [0, 0, 2]]


def test_closed_neuron_alone_has_one_child():
    w = _chain(3)
    o = oracle.System.from_workload(w)
    psi, S, Y = o.children_delay(np.array([3], np.int32), np.array([0, 0, 2, 0, 1, 0], np.int32))
    assert psi == 1 and S.sum() == 0 and list(Y[0]) == [0, 0, 1, 0, 1, 0]
    psi, S, Y = o.children_delay(np.array([3], np.int32), np.array([0, 0, 0, 0, 0, 0], np.int32))
    assert psi == 0  # nothing open can fire, nothing closed: halting


def test_overflow_applies_to_clock_and_pending_columns():
    w = _chain(300)
    o = oracle.System.from_workload(w)
    r = o.explore_delay(np.array([300], np.int32), w.C0, 3, count_bits=8)
    assert r.status == oracle.OR_E_OVERFLOW  # τ = 300 does not fit uint8
    r = o.explore_delay(np.array([300], np.int32), w.C0, 3, count_bits=16)
    assert r.status == 0
