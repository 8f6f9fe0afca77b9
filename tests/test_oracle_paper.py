"""Pins of the CPU oracle against values the paper prints (worked example,
printed run) and against the paper's semantic claim about Π.  CPU only."""
import numpy as np
import pytest

import oracle
from oracle import brute
from paper_1104_1824_b200 import workloads as W
from golden_util import read_kv, read_lines


def cfg_str(c):
    return "-".join(str(int(x)) for x in c)


@pytest.fixture(scope="module")
def golden():
    return read_kv("pi_worked_example.txt")


def test_matrix_eq1_matches_row_major_eq3(golden):
    # PAPER.md:123 eq. (1) vs PAPER.md:193 eq. (3)
    eq3 = [int(x) for x in golden["M_row_major"].split()]
    assert W.PI_M.flatten().tolist() == eq3
    w = W.pi_system("simulator")
    assert w.dense_M().flatten().tolist() == eq3


def test_def2_rebuilds_eq1_from_synapses_and_rules():
    # Def. 2 applied to syn and the rules'
    # (c, p) reproduces M_Π of eq. (1).
    w = W.pi_system("textbook")
    out = [[j for (s, j) in W.PI_SYN if s == i] for i in range(3)]
    rows = W.matrix_rows_from_rules(w.rules, out)
    M = np.zeros((5, 3), np.int32)
    for r, entries in enumerate(rows):
        for j, v in entries:
            M[r, j] = v
    assert (M == W.PI_M).all()


def test_rule_file_exponents(golden):
    # eq. (4)/(6): the r file holds the regex exponents (reading A2)
    exps = [int(x) for x in golden["r_file"].replace("$", " ").split()]
    for enc in ("simulator", "textbook"):
        assert W.pi_system(enc).rules[:, 2].tolist() == exps


@pytest.mark.parametrize("enc", ["simulator", "textbook"])
def test_worked_example_II1_and_psi(golden, enc):
    sys_ = oracle.System.from_workload(W.pi_system(enc))
    tmp, d = sys_.applicability(W.PI_C0)
    assert tmp.tolist() == [int(x) for x in golden["tmp_II1"].split()]
    psi = int(np.prod([x for x in d if x > 0]))
    assert psi == int(golden["psi_C0"])
    # tmp2 per neuron: one one-hot string per applicable rule
    tmp2 = []
    for s in range(3):
        rules_s = [r for r in range(5) if W.pi_system(enc).rules[r, 0] == s]
        tmp2.append(["".join("1" if q == r else "0" for q in rules_s) for r in rules_s if tmp[r] > 0])
    assert " | ".join(" ".join(x) for x in tmp2) == golden["tmp2"]


@pytest.mark.parametrize("enc", ["simulator", "textbook"])
def test_worked_example_spiking_vectors_and_C1(golden, enc):
    sys_ = oracle.System.from_workload(W.pi_system(enc))
    psi, S, C = sys_.children(W.PI_C0)
    assert psi == 2
    assert ["".join(map(str, s)) for s in S] == golden["spiking_vectors"].split()
    assert [cfg_str(c) for c in C] == golden["allGenCk_after_C0"].split()[1:]


def test_printed_run_prefixes(golden):
    # The paper processes parents in generation order and appends new C_k to
    # allGenCk: a prefix of the BFS discovery order.
    run = oracle.System.from_workload(W.pi_system("simulator")).explore(W.PI_C0, depth=3)
    order = [cfg_str(c) for c in run.configs]
    for key in ("allGenCk_after_C0", "allGenCk_after_212", "allGenCk_after_112"):
        exp = golden[key].split()
        assert order[:len(exp)] == exp


def test_printed_run_first45_entries():
    # PAPER.md:408 entries 1-45 = BFS levels 0..9 (reading A1 simulator encoding)
    exp = read_lines("pi_allgenck_first45.txt")
    run = oracle.System.from_workload(W.pi_system("simulator")).explore(W.PI_C0, depth=9)
    assert run.status == 0
    assert [cfg_str(c) for c in run.configs] == exp
    assert np.diff(run.level_offsets).tolist() == [1, 2, 4, 6, 6, 6, 5, 5, 5, 5]


def test_textbook_reading_diverges_at_entry_4():
    # reading A1: the literal Def. 1 reading cannot print '2-1-3'
    run = oracle.System.from_workload(W.pi_system("textbook")).explore(W.PI_C0, depth=12)
    order = [cfg_str(c) for c in run.configs]
    assert order[:3] == ["2-1-1", "2-1-2", "1-1-2"] and "2-1-3" not in order


def test_textbook_reachable_set_and_halting():
    run = oracle.System.from_workload(W.pi_system("textbook")).explore(W.PI_C0, depth=12)
    assert sorted(cfg_str(c) for c in run.configs) == sorted(
        ["2-1-1", "2-1-2", "1-1-2", "2-0-1", "1-1-1", "0-1-1", "1-0-1", "1-0-0"])
    assert np.diff(run.level_offsets).tolist()[:6] == [1, 2, 1, 2, 1, 1]
    assert int(run.counters.T.sum()) == 10
    assert [cfg_str(c) for c in run.configs[run.halting == 1]] == ["1-0-0"]


def test_simulator_closed_form_levels():
    # Under the ≥ reading, level d >= 6 is {(2,1,d+1),(1,1,d+1),(2,0,d),(0,1,d-1),(1,0,d-2)}
    # (derived from the rules; cross-checked by the brute-force BFS below).
    run = oracle.System.from_workload(W.pi_system("simulator")).explore(W.PI_C0, depth=30)
    for d in range(6, 31):
        got = {tuple(int(x) for x in c) for c in run.level(d)}
        assert got == {(2, 1, d + 1), (1, 1, d + 1), (2, 0, d), (0, 1, d - 1), (1, 0, d - 2)}
    assert [cfg_str(c) for c in run.configs[run.halting == 1]] == ["1-0-0"]


@pytest.mark.parametrize("enc", ["simulator", "textbook"])
def test_bfs_level_sets_match_bruteforce(enc):
    w = W.pi_system(enc)
    levels, transitions = brute.bfs_levels(w.rules.tolist(), w.dense_M().tolist(), w.C0.tolist(), 12)
    run = oracle.System.from_workload(w).explore(w.C0, depth=12)
    for d, lev in enumerate(levels):
        assert {tuple(int(x) for x in c) for c in run.level(d)} == lev
    assert int(run.counters.T.sum()) == transitions
    # totals through depth 12: simulator 60 configs / 147 transitions; textbook 8 / 10
    assert (len(run.configs), transitions) == ((60, 147) if enc == "simulator" else (8, 10))


def test_config2_depth200_totals():
    run = oracle.System.from_workload(W.pi_system("simulator")).explore(W.PI_C0, depth=200)
    assert len(run.configs) == 25 + 5 * (200 - 5) == 1000
    assert int(run.counters.T.sum()) == 2779
    assert int(run.configs.max()) == 201


@pytest.mark.parametrize("T", [6, 10, 14])
def test_pi_generates_N_minus_1_textbook(T):
    # Π generates N − {1}.  The literal (textbook) reading does;
    # numbers generated within T steps are {2, ..., T-1}.
    w = W.pi_system("textbook")
    nums = brute.generated_numbers_paths(w.rules.tolist(), w.dense_M().tolist(), w.C0.tolist(),
                                         w.meta["out_rule"], T)
    assert nums == set(range(2, T))
    w2 = W.pi_system("simulator")
    nums2 = brute.generated_numbers_paths(w2.rules.tolist(), w2.dense_M().tolist(), w2.C0.tolist(),
                                          w2.meta["out_rule"], T)
    assert nums2 == set(range(1, T))  # the ≥ reading also generates 1 (reading A1)
