"""Seeded synthetic inputs shared by the oracle tests and the CUDA engine.

This module holds NO arithmetic of the method (no applicability, no spiking
vectors, no transitions, no dedup).  It only builds input systems — rules,
synapses and the spiking transition matrix M_Π of Def. 2 —
and level-0 configurations:

* ``pi_system(encoding)`` — the paper's N−{1} generator Π (PAPER.md:97-103,
  M_Π eq. (1), rule exponents eqs. (4)/(6) PAPER.md:212, 221,
  C0 = <2,1,1> PAPER.md:109) in the two encodings of reading A1:
  ``"simulator"`` (every rule a^k a*, which reproduces the printed run,
  PAPER.md:378-408) and ``"textbook"`` (every rule exactly a^k, Def. 1).
* ``random_system(...)`` — random systems shaped like SURVEY §8(d-4): ``R``
  rules per neuron, out-degree ``outdeg`` synapses, a few nondeterministic
  neurons; all p ∈ {0, 1} as in Π.
* ``level0_counts(...)`` — level-0 frontiers from a counter-based generator
  (splitmix64 of seed ⊕ (p·m + s)), so the GPU input generator in
  ``csrc/workload_gen.cu`` produces bit-identical data on the device.

The recipe is stated in DESIGN.md §4.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

EXACT, PERIODIC, UNARY = 0, 1, 2
MASK64 = (1 << 64) - 1


@dataclass
class Workload:
    """An SNP system in the ABI's terms (rules n×6, M_Π as CSR)."""
    name: str
    m: int
    rules: np.ndarray            # int32 n×6: neuron, kind, a, b, consumed, produced
    row_ptr: np.ndarray          # int64 n+1
    col: np.ndarray              # int32 nnz
    val: np.ndarray              # int32 nnz
    C0: np.ndarray               # int32 m
    level0_range: np.ndarray     # int32 m: level-0 counts are U{0 .. range-1}
    synapses: list = field(default_factory=list)   # (s, j) pairs, 0-based
    meta: dict = field(default_factory=dict)
    re_bits: np.ndarray | None = None  # uint64 n×4: membership rows of UNARY rules (kind 2)

    @property
    def n(self) -> int:
        return int(self.rules.shape[0])

    def dense_M(self) -> np.ndarray:
        M = np.zeros((self.n, self.m), np.int32)
        for r in range(self.n):
            for e in range(self.row_ptr[r], self.row_ptr[r + 1]):
                M[r, self.col[e]] = self.val[e]
        return M


def _csr_from_rows(rows):
    row_ptr = np.zeros(len(rows) + 1, np.int64)
    cols, vals = [], []
    for r, entries in enumerate(rows):
        for j, v in sorted(entries):
            cols.append(j)
            vals.append(v)
        row_ptr[r + 1] = len(cols)
    return row_ptr, np.array(cols, np.int32), np.array(vals, np.int32)


def matrix_rows_from_rules(rules: np.ndarray, out_targets) -> list:
    """Def. 2: row r has -c at σ(r) and +p at every j with
    (σ(r), j) ∈ syn (reading A11: each out-neighbour receives p)."""
    rows = []
    for r in range(rules.shape[0]):
        s, _k, _a, _b, c, p = (int(x) for x in rules[r])
        entries = [(s, -c)]
        if p > 0:
            entries += [(int(j), p) for j in out_targets[s]]
        rows.append(entries)
    return rows


# ---------------------------------------------------------------------------
# Π — the paper's only workload
# ---------------------------------------------------------------------------
PI_M = np.array([[-1, 1, 1], [-2, 1, 1], [1, -1, 1], [0, 0, -1], [0, 0, -2]], np.int32)  # eq. (1)
PI_R_EXPONENTS = [[2, 2], [1], [1, 2]]  # eq. (6), the file r of eq. (4)
PI_C0 = np.array([2, 1, 1], np.int32)
PI_SYN = [(0, 1), (0, 2), (1, 0), (1, 2)]  # syn = {(1,2),(1,3),(2,1),(2,3)}


def pi_system(encoding: str = "simulator") -> Workload:
    """Π with rules {neuron, regex, consumed, produced} derived from eqs. (1),
    (4): the r value is E's exponent and consumption comes from M (reading A2);
    produced p = the off-diagonal entry (1 for rules 1-4, to the environment
    for rule 4 (reading A12); 0 for the forgetting rule 5)."""
    if encoding not in ("simulator", "textbook"):
        raise ValueError(encoding)
    rules = []
    r = 0
    for s, exps in enumerate(PI_R_EXPONENTS):
        for k in exps:
            c = -int(PI_M[r, s])
            p = 0 if r == 4 else 1
            if encoding == "simulator":
                rules.append([s, PERIODIC, k, 1, c, p])  # a^k a* (reading A1)
            else:
                rules.append([s, EXACT, k, 0, c, p])     # a^k
            r += 1
    rules = np.array(rules, np.int32)
    rows = [[(j, int(PI_M[r, j])) for j in range(3) if PI_M[r, j] != 0] for r in range(5)]
    row_ptr, col, val = _csr_from_rows(rows)
    return Workload(name=f"pi-{encoding}", m=3, rules=rules, row_ptr=row_ptr, col=col, val=val,
                    C0=PI_C0.copy(), level0_range=np.array([3, 3, 3], np.int32), synapses=list(PI_SYN),
                    meta={"encoding": encoding, "out_neuron": 2, "out_rule": 3})


# ---------------------------------------------------------------------------
# random systems
# ---------------------------------------------------------------------------
def random_system(m: int, outdeg: int = 8, k_nd: int = 3, seed: int = 0, name: str = "") -> Workload:
    """Deterministic neurons (threshold θ ~ U{6..10}): four rules
    PERIODIC(i=θ+x, j=4), x = 0..3, consuming c_x ∈ [θ+x-2, θ+x], p = 1 —
    exactly one is applicable iff n >= θ.  Nondeterministic neurons copy σ1's
    pattern in Π (two rules with the same language, different consumption)
    plus a spike-vs-forget overlap like σ3 under the simulator reading:
      a^θ a*/a^(θ-2) -> a,  a^θ a*/a^θ -> a,  a^(θ+1) a* -> λ,
      a^(θ+2) (a^2)*/a^(θ-1) -> a
    giving 2-4 applicable rules once n >= θ.  Each neuron has ``outdeg``
    distinct out-synapses chosen uniformly among the other neurons."""
    assert m >= 2 and outdeg <= m - 1
    rng = np.random.Generator(np.random.PCG64(seed))
    theta = rng.integers(6, 11, size=m)
    out_targets = []
    for s in range(m):
        t = rng.choice(m - 1, size=outdeg, replace=False)
        t = np.where(t >= s, t + 1, t)
        out_targets.append(np.sort(t))
    nd = set(int(x) for x in rng.choice(m, size=min(k_nd, m), replace=False)) if k_nd > 0 else set()
    cons_jitter = rng.integers(0, 3, size=(m, 4))
    rules = []
    for s in range(m):
        th = int(theta[s])
        if s in nd:
            rules += [[s, PERIODIC, th, 1, th - 2, 1],
                      [s, PERIODIC, th, 1, th, 1],
                      [s, PERIODIC, th + 1, 1, th + 1, 0],
                      [s, PERIODIC, th + 2, 2, th - 1, 1]]
        else:
            for x in range(4):
                rules.append([s, PERIODIC, th + x, 4, th + x - int(cons_jitter[s, x]), 1])
    rules = np.array(rules, np.int32)
    rows = matrix_rows_from_rules(rules, out_targets)
    row_ptr, col, val = _csr_from_rows(rows)
    syn = [(s, int(j)) for s in range(m) for j in out_targets[s]]
    w = Workload(name=name or f"random-m{m}-s{seed}", m=m, rules=rules, row_ptr=row_ptr, col=col, val=val,
                 C0=np.zeros(m, np.int32), level0_range=(theta + 4).astype(np.int32), synapses=syn,
                 meta={"seed": seed, "outdeg": outdeg, "k_nd": k_nd, "nd_neurons": sorted(nd)})
    w.C0 = level0_counts(w, 1, seed)[0].astype(np.int32)
    return w


def tiny_random_system(seed: int, m_max: int = 5, rules_max: int = 3, count_max: int = 6) -> Workload:
    """Tiny random systems for property tests: arbitrary mixes of EXACT and
    PERIODIC rules, forgetting rules, random synapses, random C0."""
    rng = np.random.Generator(np.random.PCG64(1_000_003 + seed))
    m = int(rng.integers(1, m_max + 1))
    out_targets = []
    for s in range(m):
        others = [j for j in range(m) if j != s]
        k = int(rng.integers(0, len(others) + 1)) if others else 0
        out_targets.append(np.sort(rng.choice(others, size=k, replace=False)) if k else np.zeros(0, np.int64))
    rules = []
    for s in range(m):
        for _ in range(int(rng.integers(0 if s else 1, rules_max + 1))):
            kind = int(rng.integers(0, 2))
            a = int(rng.integers(0, 4))
            b = int(rng.integers(1, 4)) if kind == PERIODIC else 0
            c = int(rng.integers(1, 4))
            p = int(rng.integers(0, 3))
            rules.append([s, kind, a, b, c, p])
    rules = np.array(rules, np.int32).reshape(-1, 6)
    rows = matrix_rows_from_rules(rules, out_targets)
    row_ptr, col, val = _csr_from_rows(rows)
    C0 = rng.integers(0, count_max + 1, size=m).astype(np.int32)
    return Workload(name=f"tiny-{seed}", m=m, rules=rules, row_ptr=row_ptr, col=col, val=val, C0=C0,
                    level0_range=np.full(m, count_max + 1, np.int32),
                    synapses=[(s, int(j)) for s in range(m) for j in out_targets[s]], meta={"seed": seed})


# ---------------------------------------------------------------------------
# level-0 frontiers (reading A20): counter-based so host and device agree
# ---------------------------------------------------------------------------
def _splitmix64_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def level0_seed_key(seed: int) -> int:
    return int(_splitmix64_np(np.array([seed & MASK64], np.uint64))[0])


def level0_counts(w: Workload, F: int, seed: int, row_begin: int = 0, dtype=np.int32) -> np.ndarray:
    """Rows [row_begin, row_begin+F) of the level-0 frontier: count(p, s) =
    (splitmix64(key ⊕ (p·m + s)) >> 32) mod level0_range[s], key =
    splitmix64(seed).  Row-major (F × m)."""
    key = np.uint64(level0_seed_key(seed))
    m = w.m
    p = np.arange(row_begin, row_begin + F, dtype=np.uint64)[:, None]
    s = np.arange(m, dtype=np.uint64)[None, :]
    with np.errstate(over="ignore"):
        v = _splitmix64_np(key ^ (p * np.uint64(m) + s))
    return ((v >> np.uint64(32)) % w.level0_range.astype(np.uint64)[None, :]).astype(dtype)


# ---------------------------------------------------------------------------
# named configurations (BASELINE.json "configs")
# ---------------------------------------------------------------------------
CONFIGS = {
    1: dict(kind="pi", depth=12, dedup=0, count_bits=32, frontier_target=0),
    2: dict(kind="pi", depth=200, dedup=0, count_bits=32, frontier_target=0),
    3: dict(kind="random", m=1024, k_nd=3, seed=3, F=1 << 20, depth=10, dedup=0, count_bits=32,
            frontier_target=1 << 20),
    4: dict(kind="random", m=16384, k_nd=3, seed=4, F=1 << 22, depth=20, dedup=1, count_bits=8,
            frontier_target=1 << 22),
    5: dict(kind="random", m=65536, k_nd=7, seed=5, F=10_000_000, depth=20, dedup=1, count_bits=8,
            frontier_target=10_000_000),
}


# ---------------------------------------------------------------------------
# general unary regular expressions
# ---------------------------------------------------------------------------
def unary_lengths(regex: str, vmax: int) -> list:
    """Membership of a^v (v < vmax) in L(regex) for the small grammar of
    ``random_unary_regex`` (literal a^k, (?:xy), (?:x|y), (?:x)*), by the set
    of achievable lengths — an input builder, no SNP arithmetic."""
    def parse(i):
        # returns (set of lengths, next index); grammar: seq of atoms
        lens = {0}
        while i < len(regex) and regex[i] not in "|)":
            if regex[i] == "a":
                lens = {x + 1 for x in lens if x + 1 < vmax}
                i += 1
            elif regex.startswith("(?:", i):
                alts = set()
                i += 3
                while True:
                    sub, i = parse(i)
                    alts |= sub
                    if regex[i] == "|":
                        i += 1
                        continue
                    break
                assert regex[i] == ")"
                i += 1
                if i < len(regex) and regex[i] == "*":
                    i += 1
                    star = {0}
                    frontier = {0}
                    while frontier:
                        frontier = {x + y for x in frontier for y in alts if x + y < vmax} - star
                        star |= frontier
                    alts = star
                lens = {x + y for x in lens for y in alts if x + y < vmax}
            else:
                raise ValueError(regex)
        return lens, i

    lens, i = parse(0)
    assert i == len(regex)
    return [v in lens for v in range(vmax)]


def unary_bits_from_regex(regex: str, vmax: int = 600):
    """(t, P, row) of the UNARY rule kind for a regular expression over {a}:
    membership of a^v for v < vmax (``unary_lengths``), and (t, P) the
    smallest threshold + period (t + P <= 256) from which the membership
    sequence repeats through vmax.  row = 4 uint64, bit v = a^v ∈ L for
    v < t + P.  An input builder only: no applicability is computed here."""
    mem = unary_lengths(regex, vmax)
    best = None
    for P in range(1, 129):
        for t in range(0, 257 - P):
            if all(mem[v] == mem[v + P] for v in range(t, vmax - P)):
                if best is None or t + P < best[0] + best[1]:
                    best = (t, P)
                break
    if best is None:
        raise ValueError(f"{regex!r}: no period <= 128 with t + P <= 256 found below {vmax}")
    t, P = best
    row = np.zeros(4, np.uint64)
    for v in range(t + P):
        if mem[v]:
            row[v // 64] |= np.uint64(1) << np.uint64(v % 64)
    return t, P, row


def random_unary_regex(rng, depth: int = 3, star_ok: bool = True) -> str:
    """A random regular expression over {a}: literals a^k, concatenation,
    alternation and Kleene star (no star inside a star, so Python's backtracking
    ``re`` engine stays fast on the test-side pin)."""
    if depth == 0 or rng.random() < 0.3:
        return "a" * int(rng.integers(0, 4))
    op = int(rng.integers(0, 3 if star_ok else 2)) if star_ok else int(rng.integers(1, 3))
    if op == 0:
        return f"(?:{random_unary_regex(rng, depth - 1, False)})*"
    x = random_unary_regex(rng, depth - 1, star_ok)
    y = random_unary_regex(rng, depth - 1, star_ok)
    return f"(?:{x}{y})" if op == 1 else f"(?:{x}|{y})"


def tiny_unary_system(seed: int, m_max: int = 4, rules_max: int = 3, count_max: int = 8) -> Workload:
    """Tiny random systems whose rules carry random unary regexes (kind UNARY);
    meta["regex"][r] is rule r's expression (the pin: Python's re engine)."""
    w = tiny_random_system(seed, m_max=m_max, rules_max=rules_max, count_max=count_max)
    rng = np.random.Generator(np.random.PCG64(7_000_003 + seed))
    rules = w.rules.copy()
    bits = np.zeros((w.n, 4), np.uint64)
    regexes = []
    for r in range(w.n):
        rx = random_unary_regex(rng)
        t, P, row = unary_bits_from_regex(rx)
        rules[r, 1], rules[r, 2], rules[r, 3] = UNARY, t, P
        bits[r] = row
        regexes.append(rx)
    w.rules = rules
    w.re_bits = bits
    w.name = f"tiny-unary-{seed}"
    w.meta = dict(w.meta, regex=regexes)
    return w


def as_unary(w: Workload) -> Workload:
    """The same system with every EXACT / PERIODIC rule re-encoded as a UNARY
    rule of the same language (a^k = threshold k+1, period 1, bit k;
    a^i(a^j)* = threshold i, period j, bit i)."""
    rules = w.rules.copy()
    bits = np.zeros((w.n, 4), np.uint64)
    for r in range(w.n):
        kind, a, b = int(rules[r, 1]), int(rules[r, 2]), int(rules[r, 3])
        if kind == EXACT:
            t, P, members = a + 1, 1, [a]
        elif kind == PERIODIC:
            t, P, members = a, b, [a]
        else:
            continue
        if t + P > 256:
            raise ValueError("exponent too large for the UNARY encoding")
        for v in members:
            bits[r, v // 64] |= np.uint64(1) << np.uint64(v % 64)
        rules[r, 1], rules[r, 2], rules[r, 3] = UNARY, t, P
    return Workload(name=w.name + "-unary", m=w.m, rules=rules, row_ptr=w.row_ptr, col=w.col, val=w.val,
                    C0=w.C0.copy(), level0_range=w.level0_range, synapses=w.synapses, meta=dict(w.meta),
                    re_bits=bits)
