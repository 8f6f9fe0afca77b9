"""Pure-Python brute-force SNP semantics for tiny systems (TEST INFRASTRUCTURE).

Independent of ``oracle.cpp``: it never decodes a mixed-radix index.  It
enumerates every 0/1 vector of length n ("We can have all the possible vectors
composed of 0s and 1s with length equal to the number of rules, but have only
some of them be valid") and keeps the valid ones: every
chosen rule is applicable, at most one rule per neuron is chosen
(PAPER.md:93), and every neuron with an applicable rule uses exactly one
(maximal parallelism; reading A4).  Children are C + S·M computed
with dense Python integer arithmetic (eq. 2).
"""
from __future__ import annotations

from itertools import product

EXACT, PERIODIC = 0, 1


def rule_applicable(rule, v: int) -> bool:
    """a^v ∈ L(E) and v >= c (regex kinds: reading A1)."""
    neuron, kind, a, b, c, p = (int(x) for x in rule)
    if kind == EXACT:
        in_lang = v == a
    else:
        in_lang = v >= a and (v - a) % b == 0
    return in_lang and v >= c


def valid_spiking_vectors(rules, C, app_fn=None):
    """All valid S ∈ {0,1}^n for configuration C, as tuples (any order).
    app_fn(r, v): applicability of rule r at v spikes (default: the EXACT /
    PERIODIC kinds above; tests pass Python-regex membership for UNARY)."""
    n = len(rules)
    app_fn = app_fn or (lambda r, v: rule_applicable(rules[r], v))
    app = [app_fn(r, C[int(rules[r][0])]) for r in range(n)]
    neurons = sorted({int(r[0]) for r in rules})
    out = []
    for S in product((0, 1), repeat=n):
        if any(S[r] and not app[r] for r in range(n)):
            continue
        ok = True
        for s in neurons:
            chosen = sum(S[r] for r in range(n) if int(rules[r][0]) == s)
            has_app = any(app[r] for r in range(n) if int(rules[r][0]) == s)
            if chosen > 1 or (has_app and chosen != 1):
                ok = False
                break
        if ok:
            out.append(S)
    return out


def apply(M, C, S):
    """Eq. (2): C' = C + S·M with M dense (n rows × m columns)."""
    m = len(C)
    return tuple(C[j] + sum(S[r] * M[r][j] for r in range(len(S))) for j in range(m))


def children(rules, M, C, app_fn=None):
    """All (S, C') pairs.  A halting configuration (no applicable rule) has no
    children: the all-zero vector would only reproduce C (reading A5,
    stopping criterion 1)."""
    if is_halting(rules, C, app_fn):
        return []
    return [(S, apply(M, C, S)) for S in valid_spiking_vectors(rules, C, app_fn)]


def is_halting(rules, C, app_fn=None) -> bool:
    app_fn = app_fn or (lambda r, v: rule_applicable(rules[r], v))
    return not any(app_fn(r, C[int(rules[r][0])]) for r in range(len(rules)))


def bfs_levels(rules, M, C0, depth: int):
    """Level sets of the BFS tree with global dedup (as Python sets)."""
    seen = {tuple(C0)}
    levels = [{tuple(C0)}]
    transitions = 0
    for _ in range(depth):
        nxt = set()
        for C in levels[-1]:
            for _S, Cn in children(rules, M, C):
                transitions += 1
                if Cn not in seen:
                    nxt.add(Cn)
        seen |= nxt
        if not nxt:
            break
        levels.append(nxt)
    return levels, transitions


def generated_numbers_paths(rules, M, C0, out_rule: int, T: int):
    """Numbers generated within T steps: along every computation path, the
    distance t2 - t1 between the first two steps at which the output neuron's
    spiking rule ``out_rule`` fires (the result of Π is the
    set of numbers it generates).  Exhaustive path enumeration (tiny T)."""
    found = set()

    def walk(C, step, t1):
        if step >= T:
            return
        for S, Cn in children(rules, M, C):
            fired = S[out_rule] == 1
            if fired and t1 is not None:
                found.add(step - t1)
                continue
            walk(Cn, step + 1, step if fired else t1)

    walk(tuple(C0), 0, None)
    return found
