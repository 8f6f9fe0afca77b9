"""Diagnostic: how far apart are the parents of 4 consecutive kept children?
K-c builds each 4-child output word with byte permutes of the parent x row
when the 4 parents lie in a 16-byte window (else 4 byte loads).  Runs 4
levels of config 4's system at F = 2^16 and prints the fraction of quads
whose parents fit 8/16/24/32-byte windows (measured: 88 % / 99.8 % / 100 %).
Usage (GPU): python tools/quad_windows.py"""
import numpy as np, sys
sys.path.insert(0, '.')
from paper_1104_1824_b200 import snp, workloads as W
cfg = W.CONFIGS[4]
w = W.random_system(cfg["m"], outdeg=8, k_nd=cfg["k_nd"], seed=cfg["seed"])
F = 1 << 16
L0 = W.level0_counts(w, F, 4).astype(np.uint8)
eng = snp.System(w, count_bits=8, dedup=1, frontier_target=F, keep_tree=0)
eng.begin(L0)
for _ in range(4): eng.advance()
L = eng.depth
par, t, halt = eng.level_edges(L)[:3]
par = np.asarray(par, np.int64)
K = len(par)
blk = par // 64
# quads fully inside one parent block's child range
q = np.arange(0, K - 3, 4)
same = (blk[q] == blk[q + 3])
span = par[q + 3] - (par[q] // 4) * 4
print("K", K, "quads", len(q), "same-block", same.mean())
for lim in (8, 16, 24, 32):
    print(lim, "window ok", ((span < lim) & same).sum() / same.sum())
