"""GPU parity for SURVEY §8(f) NEXT-2 — general unary regular expressions
(SNP_RE_UNARY, include/snp.h; PAPER.md:419 future work).  The engine's table
builder and generic kernels evaluate the ultimately periodic membership rows;
results must be bit-identical to the oracle (itself pinned to Python's re
engine in tests/test_oracle_unary.py)."""
import numpy as np
import pytest

import oracle
from paper_1104_1824_b200 import workloads as W

from test_gpu_parity import assert_same_tree

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def snp():
    from paper_1104_1824_b200 import snp as _snp
    return _snp


@pytest.mark.parametrize("chunk", range(4))
@pytest.mark.parametrize("bits,dedup", [(8, 1), (16, 0), (32, 0)])
def test_tiny_unary_systems(snp, chunk, bits, dedup):
    for seed in range(30 * chunk, 30 * chunk + 30):
        w = W.tiny_unary_system(seed)
        ref = oracle.System.from_workload(w).explore(w.C0, depth=8, dedup=dedup, count_bits=bits)
        eng = snp.System(w, count_bits=bits, dedup=dedup)
        if ref.status != 0:
            with pytest.raises(snp.SnpError):
                eng.explore(None, depth=8)
        else:
            assert_same_tree(eng.explore(None, depth=8), ref)
        eng.close()


@pytest.mark.parametrize("enc", ["simulator", "textbook"])
def test_pi_unary_encoding(snp, enc):
    w = W.pi_system(enc)
    u = W.as_unary(w)
    a = snp.System(w, count_bits=8).explore(None, depth=40)
    b = snp.System(u, count_bits=8).explore(None, depth=40)
    ref = oracle.System.from_workload(u).explore(w.C0, depth=40, count_bits=8)
    assert_same_tree(b, ref)
    assert (a.configs == b.configs).all() and (a.fp == b.fp).all()


def test_random_system_unary_fast_kernels(snp):
    """The uint8 fast path (tables, byte-permute lookups, bit-sliced K-c) with
    every rule given as a UNARY membership row, thinning on."""
    w = W.as_unary(W.random_system(512, outdeg=8, k_nd=6, seed=33))
    L0 = W.level0_counts(w, 600, 33)
    tree = snp.System(w, count_bits=8, dedup=1, frontier_target=800).explore(L0, depth=4)
    ref = oracle.System.from_workload(w).explore(L0, depth=4, dedup=1, count_bits=8, frontier_target=800)
    assert_same_tree(tree, ref)


def test_unary_generated_numbers(snp):
    """NEXT-1 and NEXT-2 together: Π's output rule given as a unary regex."""
    w = W.as_unary(W.pi_system("textbook"))
    out = w.meta["out_rule"]
    eng = snp.System(w, out_rule=out)
    tree = eng.explore(None, depth=60)
    ref = oracle.System.from_workload(w).explore(w.C0, depth=60, out_rule=out)
    assert_same_tree(tree, ref)
    assert eng.generated_numbers() == ref.numbers == set(range(2, 60))
