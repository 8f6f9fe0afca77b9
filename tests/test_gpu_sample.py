"""GPU parity for SURVEY §8(f) NEXT-4 — single-path sampling with an input
spike train (include/snp.h ``snp_sample``; Def. 1 `in`, PAPER.md:89;
PAPER.md:240).  Each walker takes the child t = u mod Ψ (counter-based u,
reading A25) in Alg. 2's enumeration order, then the input neuron receives
train[k] spikes.  The oracle (``oracle_sample``) is pinned in
tests/test_oracle_sample.py; here the engine must agree with it exactly:
the same final configurations, the same halting steps, the same errors."""
import numpy as np
import pytest

import oracle
from paper_1104_1824_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def snp():
    from paper_1104_1824_b200 import snp as _snp
    return _snp


def _both(snp, w, C, seed, steps, bits=32, **kw):
    """(engine result or status, oracle result or status) on the same walkers."""
    try:
        e = snp.System(w, count_bits=bits, dedup=0).sample(C, seed, steps, **kw)
    except snp.SnpError as ex:
        e = ex.status
    try:
        o = oracle.System.from_workload(w).sample(C, seed, steps, count_bits=bits, **kw)
    except oracle.OracleError as ex:
        o = ex.status
    return e, o


def _assert_same(e, o):
    if isinstance(o, int) or isinstance(e, int):
        assert e == o, (e, o)
        return
    assert (e[0] == o[0]).all(), np.argwhere(e[0] != o[0])[:5]
    assert (e[1] == o[1]).all()


@pytest.mark.parametrize("enc", ["simulator", "textbook"])
@pytest.mark.parametrize("with_input", [False, True])
def test_pi_walkers(snp, enc, with_input):
    w = W.pi_system(enc)
    C = np.tile(w.C0, (97, 1))
    kw = dict(input_neuron=0, train=np.array([1, 0, 2, 0, 0, 1], np.int32)) if with_input else {}
    for seed in range(4):
        e, o = _both(snp, w, C, seed, 40, **kw)
        _assert_same(e, o)
    if enc == "textbook" and not with_input:
        assert (e[1] >= 0).all()  # the textbook Π always halts (at (1,0,0))


@pytest.mark.parametrize("seed", range(60))
def test_tiny_random_systems(snp, seed):
    w = W.tiny_random_system(seed, m_max=5, rules_max=3, count_max=6)
    rng = np.random.default_rng(seed)
    C = rng.integers(0, 7, size=(13, w.m)).astype(np.int32)
    kw = {}
    if seed % 2:
        kw = dict(input_neuron=int(seed % w.m), train=rng.integers(0, 3, size=5).astype(np.int32))
    e, o = _both(snp, w, C, 1000 + seed, 12, bits=8 if seed % 3 == 0 else 32, **kw)
    _assert_same(e, o)


@pytest.mark.parametrize("m,bits", [(300, 8), (1000, 32)])
def test_random_system_walkers(snp, m, bits):
    w = W.random_system(m, outdeg=8, k_nd=6, seed=m)
    C = W.level0_counts(w, 211, m).astype(np.int32)
    e, o = _both(snp, w, C, 77, 25, bits=bits, input_neuron=3, train=np.arange(7, dtype=np.int32) % 3)
    _assert_same(e, o)
    assert not isinstance(e, int)


def test_config5_width_walkers(snp):
    """config 5's system family at full width (m = 65536, k_nd = 7)."""
    w = W.random_system(65536, outdeg=8, k_nd=7, seed=5)
    C = W.level0_counts(w, 40, 5).astype(np.int32)
    e, o = _both(snp, w, C, 5, 4, bits=8)
    _assert_same(e, o)
    assert not isinstance(e, int)


def test_overflow_and_capacity(snp):
    # two neurons feeding each other 2 spikes per spike consumed: +1 per step,
    # so uint8 storage overflows after 254 steps on every path
    rules = np.array([[0, W.PERIODIC, 1, 1, 1, 2], [1, W.PERIODIC, 1, 1, 1, 2]], np.int32)
    rows = W.matrix_rows_from_rules(rules, [np.array([1]), np.array([0])])
    row_ptr, col, val = W._csr_from_rows(rows)
    wg = W.Workload(name="grow", m=2, rules=rules, row_ptr=row_ptr, col=col, val=val,
                    C0=np.array([1, 1], np.int32), level0_range=np.array([2, 2], np.int32))
    e, o = _both(snp, wg, np.tile(wg.C0, (3, 1)), 1, 400, bits=8)
    assert e == o == snp.SNP_E_OVERFLOW
    e, o = _both(snp, wg, np.tile(wg.C0, (3, 1)), 1, 200, bits=8)  # 201 spikes: fits
    _assert_same(e, o)
    assert (e[0] == 201).all()
    # 64 neurons with two applicable rules each: Ψ = 2^64 > 2^62
    m = 64
    rules = np.array([[s, W.PERIODIC, 1, 1, 1, 1] for s in range(m)] + [[s, W.PERIODIC, 1, 1, 2, 1] for s in range(m)],
                     np.int32)
    rules = rules[np.argsort(rules[:, 0], kind="stable")]
    out_targets = [np.array([(s + 1) % m]) for s in range(m)]
    rows = W.matrix_rows_from_rules(rules, out_targets)
    row_ptr, col, val = W._csr_from_rows(rows)
    wc = W.Workload(name="cap", m=m, rules=rules, row_ptr=row_ptr, col=col, val=val,
                    C0=np.full(m, 3, np.int32), level0_range=np.full(m, 4, np.int32))
    e, o = _both(snp, wc, wc.C0[None, :], 1, 2)
    assert e == o == snp.SNP_E_CAPACITY


def test_bad_arguments(snp):
    w = W.pi_system("simulator")
    eng = snp.System(w, count_bits=8, dedup=0)
    with pytest.raises(snp.SnpError) as ex:
        eng.sample(np.tile(w.C0, (2, 1)), 1, 3, input_neuron=3)  # neuron index out of range
    assert ex.value.status == snp.SNP_E_ARG
    with pytest.raises(snp.SnpError) as ex:
        eng.sample(np.array([[2, 1, 300]], np.int32), 1, 3)  # count beyond uint8
    assert ex.value.status == snp.SNP_E_ARG
    C, hs = eng.sample(np.zeros((0, 3), np.int32), 1, 3)
    assert C.shape == (0, 3) and hs.shape == (0,)


def test_large_rule_values_take_the_warp_kernel(snp):
    """a rule with p > 255 cannot use the shared-memory (c, p) bytes of
    k_sample_cta: the warp-per-walker kernel runs and must agree too."""
    rules = np.array([[0, W.PERIODIC, 1, 1, 1, 300], [1, W.PERIODIC, 1, 1, 1, 2], [1, W.PERIODIC, 2, 1, 2, 1]],
                     np.int32)
    rows = W.matrix_rows_from_rules(rules, [np.array([1]), np.array([0])])
    row_ptr, col, val = W._csr_from_rows(rows)
    wg = W.Workload(name="bigp", m=2, rules=rules, row_ptr=row_ptr, col=col, val=val,
                    C0=np.array([1, 1], np.int32), level0_range=np.array([2, 2], np.int32))
    for seed in range(3):
        e, o = _both(snp, wg, np.tile(wg.C0, (17, 1)), seed, 12, bits=32, input_neuron=1,
                     train=np.array([1, 0, 3], np.int32))
        _assert_same(e, o)
