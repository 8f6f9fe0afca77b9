"""GPU parity for SURVEY §8(f) NEXT-3 — SN P systems with delays
(include/snp.h ``snp_load_delay``, reading A26).  The engine explores states
[C | τ | π] (width 3m); the oracle (``oracle_explore_delay``, pinned in
tests/test_oracle_delay.py) does the same BFS on the CPU.  Bit-exact: the same
trees (states, parents, t, halting, fingerprints, per-level counters)."""
import numpy as np
import pytest

import oracle
from paper_1104_1824_b200 import workloads as W
from paper_1104_1824_b200.workloads import Workload

from test_gpu_parity import assert_same_tree

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def snp():
    from paper_1104_1824_b200 import snp as _snp
    return _snp


def _wide(L0, m):
    L0 = np.atleast_2d(np.asarray(L0, np.int32))
    return np.hstack([L0, np.zeros((L0.shape[0], 2 * m), np.int32)])


def _check(snp, w, delays, L0, depth, bits=32, target=0):
    eng = snp.System(w, count_bits=bits, dedup=1, frontier_target=target, delays=delays)
    assert eng.width == 3 * w.m
    tree = eng.explore(L0, depth=depth)
    ref = oracle.System.from_workload(w).explore_delay(delays, L0, depth, dedup=1, count_bits=bits,
                                                       frontier_target=target)
    assert_same_tree(tree, ref)
    return tree


@pytest.mark.parametrize("enc", ["simulator", "textbook"])
@pytest.mark.parametrize("bits", [8, 32])
def test_pi_zero_delays_is_the_delay_free_tree(snp, enc, bits):
    w = W.pi_system(enc)
    tree = _check(snp, w, np.zeros(w.n, np.int32), _wide(w.C0, w.m), 12, bits)
    plain = snp.System(w, count_bits=bits, dedup=1).explore(None, depth=12)
    assert (tree.configs[:, :w.m] == plain.configs).all() and (tree.configs[:, w.m:] == 0).all()
    assert (tree.fp == plain.fp).all()


@pytest.mark.parametrize("enc", ["simulator", "textbook"])
def test_pi_with_delays(snp, enc):
    w = W.pi_system(enc)
    for delays in ([1, 0, 0, 2, 0], [0, 2, 1, 0, 1], [3, 3, 3, 3, 3]):
        _check(snp, w, np.array(delays, np.int32), _wide(w.C0, w.m), 14)


@pytest.mark.parametrize("seed", range(80))
def test_tiny_random_systems(snp, seed):
    w = W.tiny_random_system(seed, m_max=5, rules_max=3, count_max=6)
    rng = np.random.default_rng(seed + 5)
    delays = rng.integers(0, 3, size=w.n).astype(np.int32)
    L0 = _wide(rng.integers(0, 6, size=(3, w.m)), w.m)
    _check(snp, w, delays, L0, 6, bits=8 if seed % 2 else 32)


def test_random_system_with_thinning(snp):
    w = W.random_system(200, outdeg=8, k_nd=6, seed=21)
    rng = np.random.default_rng(21)
    delays = np.where(rng.random(w.n) < 0.3, rng.integers(1, 4, size=w.n), 0).astype(np.int32)
    L0 = _wide(W.level0_counts(w, 120, 21), w.m)
    _check(snp, w, delays, L0, 4, bits=8, target=150)


def test_lost_spike_closed_form(snp):
    rules = np.array([[0, W.EXACT, 1, 0, 1, 1], [1, W.PERIODIC, 1, 1, 1, 1]], np.int32)
    rows = W.matrix_rows_from_rules(rules, [np.array([1]), np.array([2]), np.array([], np.int64)])
    rp, col, val = W._csr_from_rows(rows)
    w = Workload(name="lost", m=3, rules=rules, row_ptr=rp, col=col, val=val,
                 C0=np.array([1, 1, 0], np.int32), level0_range=np.array([2, 2, 1], np.int32))
    tree = _check(snp, w, np.array([0, 2], np.int32), _wide(w.C0, 3), 10)
    assert [list(c) for c in tree.configs] == [[1, 1, 0, 0, 0, 0, 0, 0, 0], [0, 0, 0, 0, 2, 0, 0, 1, 0],
                                               [0, 0, 0, 0, 1, 0, 0, 1, 0], [0, 0, 1, 0, 0, 0, 0, 0, 0]]
    assert list(tree.halting) == [0, 0, 0, 1]


def test_clock_overflow_and_state_errors(snp):
    rules = np.array([[0, W.EXACT, 1, 0, 1, 1]], np.int32)
    rows = W.matrix_rows_from_rules(rules, [np.array([1]), np.array([], np.int64)])
    rp, col, val = W._csr_from_rows(rows)
    w = Workload(name="chain", m=2, rules=rules, row_ptr=rp, col=col, val=val,
                 C0=np.array([1, 0], np.int32), level0_range=np.array([2, 1], np.int32))
    with pytest.raises(snp.SnpError) as ex:  # τ = 300 does not fit uint8
        snp.System(w, count_bits=8, dedup=1, delays=np.array([300], np.int32)).explore(None, depth=3)
    assert ex.value.status == snp.SNP_E_OVERFLOW
    with pytest.raises(snp.SnpError) as ex:
        snp.System(w, count_bits=8, dedup=0, delays=np.array([1], np.int32))
    assert ex.value.status == snp.SNP_E_ARG
    with pytest.raises(snp.SnpError) as ex:
        snp.System(w, count_bits=8, dedup=1, delays=np.array([-1], np.int32))
    assert ex.value.status == snp.SNP_E_ARG
    eng = snp.System(w, count_bits=8, dedup=1, delays=np.array([1], np.int32))
    with pytest.raises(snp.SnpError) as ex:
        eng.sample(np.array([[1, 0]], np.int32), 1, 2)
    assert ex.value.status == snp.SNP_E_STATE


def test_wide_system_takes_the_global_scratch_kernels(snp):
    """m = 2000: the per-warp shared-memory step data (16·m B × 8 warps) does
    not fit, so the kernels that recompute per column run; same tree."""
    w = W.random_system(2000, outdeg=8, k_nd=4, seed=8)
    rng = np.random.default_rng(8)
    delays = np.where(rng.random(w.n) < 0.2, rng.integers(1, 3, size=w.n), 0).astype(np.int32)
    _check(snp, w, delays, _wide(W.level0_counts(w, 30, 8), w.m), 3, bits=8, target=40)
