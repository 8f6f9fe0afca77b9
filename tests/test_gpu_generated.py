"""GPU parity for SURVEY §8(f) NEXT-1 — generated numbers.

The engine explores the augmented state (C, A) (include/snp.h "Generated
numbers"; A = steps since the first output spike, PAPER.md:89 `out`, 95-99)
and records the numbers; the oracle (``oracle_explore_gen``) does the same BFS
on the CPU.  Bit-exact: the same augmented trees (configurations with the A
column, parents, t, halting, fingerprints, counters) and the same numbers."""
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


@pytest.mark.parametrize("enc", ["textbook", "simulator"])
@pytest.mark.parametrize("dedup", [0, 1])
@pytest.mark.parametrize("bits", [8, 32])
def test_pi_generated_numbers_depth_200(snp, enc, dedup, bits):
    # config 2 (BASELINE.json): Π to depth 200 — N − {1}
    w = W.pi_system(enc)
    out = w.meta["out_rule"]
    eng = snp.System(w, count_bits=bits, dedup=dedup, out_rule=out)
    assert eng.width == w.m + 1
    tree = eng.explore(None, depth=200)
    ref = oracle.System.from_workload(w).explore(w.C0, depth=200, dedup=dedup, count_bits=bits, out_rule=out)
    assert_same_tree(tree, ref)
    assert eng.generated_numbers() == ref.numbers == set(range(2 if enc == "textbook" else 1, 200))
    eng.close()


@pytest.mark.parametrize("T", [1, 2, 3, 7, 12])
def test_pi_generated_numbers_small_depths(snp, T):
    w = W.pi_system("textbook")
    out = w.meta["out_rule"]
    eng = snp.System(w, out_rule=out)
    tree = eng.explore(None, depth=T)
    ref = oracle.System.from_workload(w).explore(w.C0, depth=T, out_rule=out)
    assert_same_tree(tree, ref)
    assert eng.generated_numbers() == ref.numbers
    # begin() clears the numbers of the previous exploration
    eng.explore(None, depth=1)
    assert eng.generated_numbers() == set()
    eng.close()


@pytest.mark.parametrize("chunk", range(4))
def test_tiny_random_generated_numbers(snp, chunk):
    T, nonempty = 10, 0
    for seed in range(25 * chunk, 25 * chunk + 25):
        w = W.tiny_random_system(seed, m_max=4, rules_max=3, count_max=6)
        for out in [r for r in range(w.n) if int(w.rules[r][5]) > 0][:2]:
            ref = oracle.System.from_workload(w).explore(w.C0, depth=T, out_rule=out, dedup=1, count_bits=16)
            if ref.status != 0:
                continue
            eng = snp.System(w, count_bits=16, dedup=1, out_rule=out)
            tree = eng.explore(None, depth=T)
            assert_same_tree(tree, ref)
            assert eng.generated_numbers() == ref.numbers, (seed, out)
            nonempty += bool(ref.numbers)
            eng.close()
    assert nonempty > 0


def test_random_system_fast_kernels_with_output(snp):
    """A config-3-shaped system (uint8 fast kernels: K-a tables, bit-sliced K-c,
    ND patches) with an output rule on a nondeterministic neuron, thinning on."""
    w = W.random_system(256, outdeg=8, k_nd=6, seed=21)
    nd = w.meta["nd_neurons"][0]
    out = int(np.nonzero(w.rules[:, 0] == nd)[0][0])
    L0 = W.level0_counts(w, 200, 21)
    eng = snp.System(w, count_bits=8, dedup=1, frontier_target=300, out_rule=out)
    tree = eng.explore(L0, depth=6)
    ref = oracle.System.from_workload(w).explore(L0, depth=6, dedup=1, count_bits=8, frontier_target=300,
                                                 out_rule=out)
    assert_same_tree(tree, ref)
    assert eng.generated_numbers() == ref.numbers
    assert ref.numbers  # the output neuron does spike twice within 6 steps
    eng.close()
