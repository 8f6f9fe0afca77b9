"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): Π (configs 1-2 shapes), 50 tiny random systems, a m = 1024
uint8 system through the tensor-core K-a (k_expand_tc) and the bit-sliced
K-c (k_materialize_bs, also its tensor-core permutation variant), a 32-bit
exact-dedup system (NARROW K-a / K-c, k_verify_m), plus the delay, sampling
and generated-number kernels.  Each result is checked against the oracle so a kernel that misbehaves
under the tool also fails here.  usage: compute-sanitizer --tool T python tools/sanitize_workload.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_1104_1824_b200 import snp  # noqa: E402
from paper_1104_1824_b200 import workloads as W  # noqa: E402


def same(tree, ref):
    assert ref.status == 0
    assert tree.level_offsets.tolist() == ref.level_offsets.tolist()
    assert (tree.configs == ref.configs).all() and (tree.fp == ref.fp).all()


def main():
    pi = W.pi_system("simulator")
    same(snp.System(pi, count_bits=8, dedup=1).explore(None, depth=30),
         oracle.System.from_workload(pi).explore(pi.C0, depth=30, dedup=1, count_bits=8))
    for seed in range(50):
        w = W.tiny_random_system(seed)
        same(snp.System(w, dedup=seed % 2).explore(None, depth=4),
             oracle.System.from_workload(w).explore(w.C0, depth=4, dedup=seed % 2))
    w = W.random_system(1024, outdeg=8, k_nd=6, seed=5)
    L0 = W.level0_counts(w, 300, 5)
    eng = snp.System(w, count_bits=8, dedup=1, frontier_target=300)
    assert eng.kernel_paths == snp.SNP_PATH_TC_EXPAND
    same(eng.explore(L0, depth=3), oracle.System.from_workload(w).explore(L0, depth=3, dedup=1, count_bits=8,
                                                                          frontier_target=300))
    # 32-bit counts, exact dedup: NARROW K-a / K-c and the per-match verification
    w3 = W.random_system(1024, outdeg=8, k_nd=5, seed=123)
    L3 = W.level0_counts(w3, 300, 123)
    L3[::7] += 300
    same(snp.System(w3, count_bits=32, dedup=0, frontier_target=400).explore(L3, depth=3),
         oracle.System.from_workload(w3).explore(L3, depth=3, dedup=0, count_bits=32, frontier_target=400))
    # the tensor-core output permutation variant of K-c (opt-in)
    os.environ["SNP_KERNELS"] = "kc_tc"
    same(snp.System(w, count_bits=8, dedup=1, frontier_target=300).explore(L0, depth=3),
         oracle.System.from_workload(w).explore(L0, depth=3, dedup=1, count_bits=8, frontier_target=300))
    os.environ["SNP_KERNELS"] = ""
    wg = W.pi_system("textbook")
    assert snp.System(wg, out_rule=3).explore(None, depth=20) is not None
    ws = W.random_system(200, outdeg=6, k_nd=5, seed=7)
    snp.System(ws, count_bits=8).sample(W.level0_counts(ws, 64, 7), seed=1, steps=5)
    print("sanitize workload OK")


if __name__ == "__main__":
    main()
