"""CPU oracle for the batched SNP transition step (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_1104_1824_b200``) never imports it and shares no code with it.

Two independent implementations live here:

* ``oracle.cpp`` → ``liboracle.so``: a plain C++17 BFS over the computation tree
  (Alg. 1), exact int64 counts, ``std::set`` dedup.
* ``brute.py``: an even plainer pure-Python enumerator (all 2^n 0/1 vectors,
  validity per PAPER.md:111-113) used to pin the C++ oracle on tiny systems.

Parity pins for every function are in ``tests/test_oracle_*.py``; readings of
silent or garbled passages are listed in DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

OR_OK = 0
OR_E_ARG = -1
OR_E_INVALID_SYSTEM = -2
OR_E_OVERFLOW = -3
OR_E_CAPACITY = -4

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_U64 = ctypes.c_uint64


def build(force: bool = False) -> str:
    """Compile oracle.cpp into liboracle.so (plain g++, no GPU code)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-pthread", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        L.oracle_load.argtypes = [_I64, _I64, _P, _P, _P, _P, ctypes.POINTER(_P), ctypes.c_char_p, _I64]
        L.oracle_load.restype = ctypes.c_int
        L.oracle_load_unary.argtypes = [_I64, _I64, _P, _P, _P, _P, _P, ctypes.POINTER(_P), ctypes.c_char_p, _I64]
        L.oracle_load_unary.restype = ctypes.c_int
        L.oracle_free.argtypes = [_P]
        L.oracle_applicability.argtypes = [_P, _P, _P, _P]
        L.oracle_children.argtypes = [_P, _P, _I64, _P, _P, ctypes.POINTER(_U64)]
        L.oracle_children.restype = ctypes.c_int
        L.oracle_fingerprint.argtypes = [_P, _I64, _U64, _U64, _P]
        L.oracle_fmix64.argtypes = [_U64]
        L.oracle_fmix64.restype = _U64
        L.oracle_thinning_tau.argtypes = [_I64, _I64]
        L.oracle_thinning_tau.restype = _U64
        L.oracle_explore.argtypes = [_P, _I64, _P, _I32, _I32, _I32, _I64, _I64, _U64, _U64, ctypes.POINTER(_P)]
        L.oracle_explore.restype = ctypes.c_int
        L.oracle_explore_gen.argtypes = [_P, _I64, _P, _I32, _I32, _I32, _I64, _I64, _U64, _U64, _I32,
                                         ctypes.POINTER(_P)]
        L.oracle_explore_gen.restype = ctypes.c_int
        L.oracle_children_delay.argtypes = [_P, _P, _P, _I64, _P, _P, ctypes.POINTER(_U64)]
        L.oracle_children_delay.restype = ctypes.c_int
        L.oracle_explore_delay.argtypes = [_P, _P, _I64, _P, _I32, _I32, _I32, _I64, _I64, _U64, _U64,
                                           ctypes.POINTER(_P)]
        L.oracle_explore_delay.restype = ctypes.c_int
        L.oracle_sample.argtypes = [_P, _I64, _P, _U64, _I32, _I32, _P, _I32, _I32, _P]
        L.oracle_sample.restype = ctypes.c_int
        L.oracle_run_num_numbers.argtypes = [_P]
        L.oracle_run_num_numbers.restype = _I64
        L.oracle_run_numbers.argtypes = [_P, _P]
        L.oracle_run_status.argtypes = [_P]
        L.oracle_run_error.argtypes = [_P]
        L.oracle_run_error.restype = ctypes.c_char_p
        for f in ("oracle_run_num_configs", "oracle_run_num_levels", "oracle_run_num_expanded"):
            getattr(L, f).argtypes = [_P]
            getattr(L, f).restype = _I64
        L.oracle_run_level_offsets.argtypes = [_P, _P]
        L.oracle_run_configs.argtypes = [_P, _I64, _P]
        L.oracle_run_tree.argtypes = [_P, _P, _P, _P, _P]
        L.oracle_run_counters.argtypes = [_P, _P, _P, _P]
        L.oracle_run_free.argtypes = [_P]
        L.oracle_run_num_edges.argtypes = [_P, _I64]
        L.oracle_run_num_edges.restype = _I64
        L.oracle_run_edges.argtypes = [_P, _I64, _P]
        L.oracle_explore_par.argtypes = [_P, _I64, _P, _I32, _I32, _I32, _I64, _I64, _U64, _U64, _I32,
                                         ctypes.POINTER(_P)]
        L.oracle_explore_par.restype = ctypes.c_int
        L.oracle_prun_free.argtypes = [_P]
        L.oracle_prun_status.argtypes = [_P]
        L.oracle_prun_error.argtypes = [_P]
        L.oracle_prun_error.restype = ctypes.c_char_p
        for f in ("oracle_prun_num_configs", "oracle_prun_num_levels", "oracle_prun_num_expanded"):
            getattr(L, f).argtypes = [_P]
            getattr(L, f).restype = _I64
        L.oracle_prun_level_offsets.argtypes = [_P, _P]
        L.oracle_prun_tree.argtypes = [_P, _P, _P, _P, _P]
        L.oracle_prun_counters.argtypes = [_P, _P, _P, _P]
        L.oracle_prun_rows.argtypes = [_P, _P, _I64, _P]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"oracle status {status}: {msg}")
        self.status = status


class System:
    """An SNP system loaded into the oracle (rules n×6 int32, M as CSR)."""

    def __init__(self, m: int, rules: np.ndarray, row_ptr: np.ndarray, col: np.ndarray, val: np.ndarray,
                 re_bits: np.ndarray | None = None):
        """re_bits: n × 4 uint64 membership rows of UNARY rules (kind 2), or None."""
        self.m = int(m)
        self.rules = np.ascontiguousarray(rules, dtype=np.int32).reshape(-1, 6)
        self.n = self.rules.shape[0]
        self._keep = (np.ascontiguousarray(row_ptr, dtype=np.int64), np.ascontiguousarray(col, dtype=np.int32),
                      np.ascontiguousarray(val, dtype=np.int32))
        h = _P()
        err = ctypes.create_string_buffer(256)
        self._bits = None if re_bits is None else np.ascontiguousarray(re_bits, dtype=np.uint64).reshape(-1, 4)
        st = lib().oracle_load_unary(self.m, self.n, _ptr(self.rules),
                                     None if self._bits is None else _ptr(self._bits), _ptr(self._keep[0]),
                                     _ptr(self._keep[1]), _ptr(self._keep[2]), ctypes.byref(h), err, 256)
        if st != OR_OK:
            raise OracleError(st, err.value.decode())
        self._h = h

    @classmethod
    def from_dense(cls, rules: np.ndarray, M: np.ndarray) -> "System":
        M = np.asarray(M, dtype=np.int64)
        n, m = M.shape
        row_ptr = [0]
        col, val = [], []
        for r in range(n):
            for j in range(m):
                if M[r, j] != 0:
                    col.append(j)
                    val.append(int(M[r, j]))
            row_ptr.append(len(col))
        return cls(m, rules, np.array(row_ptr), np.array(col, dtype=np.int32), np.array(val, dtype=np.int32))

    @classmethod
    def from_workload(cls, w) -> "System":
        return cls(w.m, w.rules, w.row_ptr, w.col, w.val, getattr(w, "re_bits", None))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().oracle_free(self._h)
            self._h = None

    # Alg. 2 II-1: per-rule marks tmp and per-neuron |σ_V|
    def applicability(self, C):
        C = np.ascontiguousarray(C, dtype=np.int32)
        tmp = np.zeros(self.n, np.int32)
        d = np.zeros(self.m, np.int32)
        lib().oracle_applicability(self._h, _ptr(C), _ptr(tmp), _ptr(d))
        return tmp, d

    # Alg. 1 II+III: all (S, C') pairs of one configuration, t order
    def children(self, C, cap: int = 1 << 20):
        C = np.ascontiguousarray(C, dtype=np.int32)
        psi = _U64()
        st = lib().oracle_children(self._h, _ptr(C), 0, None, None, ctypes.byref(psi))
        if st != OR_OK:
            raise OracleError(st)
        k = min(int(psi.value), cap)
        S = np.zeros((k, self.n), np.uint8)
        Cn = np.zeros((k, self.m), np.int64)
        lib().oracle_children(self._h, _ptr(C), k, _ptr(S), _ptr(Cn), ctypes.byref(psi))
        return int(psi.value), S, Cn

    # systems with delays (reading A26).  A state is the
    # row [C | τ | π] of width 3m; `delays` gives d >= 0 per rule.
    def children_delay(self, delays, X, cap: int = 1 << 20):
        d = np.ascontiguousarray(delays, dtype=np.int32)
        X = np.ascontiguousarray(X, dtype=np.int32)
        assert d.shape == (self.n,) and X.shape == (3 * self.m,)
        psi = _U64()
        st = lib().oracle_children_delay(self._h, _ptr(d), _ptr(X), 0, None, None, ctypes.byref(psi))
        if st != OR_OK:
            raise OracleError(st)
        k = min(int(psi.value), cap)
        S = np.zeros((k, self.n), np.uint8)
        Y = np.zeros((k, 3 * self.m), np.int64)
        lib().oracle_children_delay(self._h, _ptr(d), _ptr(X), k, _ptr(S), _ptr(Y), ctypes.byref(psi))
        return int(psi.value), S, Y

    def explore_delay(self, delays, level0, depth: int, dedup: int = 0, count_bits: int = 32,
                      frontier_target: int = 0, max_transitions: int = 0, seeds=(0x5EED0, 0x5EED1)) -> "Run":
        """BFS over delayed states; level-0 rows have m columns (all neurons
        open, τ = π = 0 appended) or 3m (oracle.cpp ``oracle_explore_delay``)."""
        d = np.ascontiguousarray(delays, dtype=np.int32)
        assert d.shape == (self.n,)
        L0 = np.ascontiguousarray(np.atleast_2d(level0), dtype=np.int32)
        if L0.shape[1] == self.m:
            L0 = np.ascontiguousarray(np.hstack([L0, np.zeros((L0.shape[0], 2 * self.m), np.int32)]))
        assert L0.shape[1] == 3 * self.m
        h = _P()
        st = lib().oracle_explore_delay(self._h, _ptr(d), L0.shape[0], _ptr(L0), depth, dedup, count_bits,
                                        frontier_target, max_transitions, seeds[0], seeds[1], ctypes.byref(h))
        if st == OR_E_ARG and not h:
            raise OracleError(st, "bad argument")
        return Run(self, h, st, 3 * self.m)

    def sample(self, walkers, seed: int, steps: int, input_neuron: int = -1, train=None, count_bits: int = 32):
        """Single-path sampling (oracle.cpp ``oracle_sample``): returns (final
        configurations W × m, halted_step W)."""
        C = np.ascontiguousarray(np.atleast_2d(walkers), dtype=np.int32).copy()
        assert C.shape[1] == self.m
        tr = np.ascontiguousarray(np.zeros(0) if train is None else train, dtype=np.int32)
        hs = np.zeros(C.shape[0], np.int32)
        st = lib().oracle_sample(self._h, C.shape[0], _ptr(C), seed, steps, input_neuron,
                                 _ptr(tr) if tr.size else None, tr.size, count_bits, _ptr(hs))
        if st != OR_OK:
            raise OracleError(st, "sample")
        return C, hs

    def explore(self, level0, depth: int, dedup: int = 0, count_bits: int = 32, frontier_target: int = 0,
                max_transitions: int = 0, seeds=(0x5EED0, 0x5EED1), out_rule: int | None = None) -> "Run":
        """BFS computation tree.  ``out_rule``: index of
        the output neuron's rule whose firing is an output spike; the state is
        then augmented with A (steps since the first output spike), level-0
        rows may have m (A = 0 appended) or m + 1 columns, and ``Run.numbers``
        holds the generated numbers (oracle.cpp ``oracle_explore_gen``)."""
        L0 = np.ascontiguousarray(np.atleast_2d(level0), dtype=np.int32)
        width = self.m + (0 if out_rule is None else 1)
        if out_rule is not None and L0.shape[1] == self.m:
            L0 = np.ascontiguousarray(np.hstack([L0, np.zeros((L0.shape[0], 1), np.int32)]))
        assert L0.shape[1] == width
        h = _P()
        st = lib().oracle_explore_gen(self._h, L0.shape[0], _ptr(L0), depth, dedup, count_bits, frontier_target,
                                      max_transitions, seeds[0], seeds[1], -1 if out_rule is None else out_rule,
                                      ctypes.byref(h))
        if st == OR_E_ARG and not h:
            raise OracleError(st, "bad argument")
        return Run(self, h, st, width)

    def explore_par(self, level0, depth: int, dedup: int = 0, count_bits: int = 32, frontier_target: int = 0,
                    max_transitions: int = 0, seeds=(0x5EED0, 0x5EED1), n_threads: int | None = None) -> "ParRun":
        """oracle_explore_par: the tree of ``explore`` (no generated numbers)
        with the children of each parent computed by ``n_threads`` threads and
        every decision taken in canonical order by one thread (oracle.cpp);
        pinned against ``explore`` in tests/test_oracle_par.py."""
        L0 = np.ascontiguousarray(np.atleast_2d(level0), dtype=np.int32)
        assert L0.shape[1] == self.m
        n_threads = n_threads or os.cpu_count() or 1
        h = _P()
        st = lib().oracle_explore_par(self._h, L0.shape[0], _ptr(L0), depth, dedup, count_bits, frontier_target,
                                      max_transitions, seeds[0], seeds[1], n_threads, ctypes.byref(h))
        if st == OR_E_ARG and not h:
            raise OracleError(st, "bad argument")
        return ParRun(self, h, st)


class ParRun:
    """Result of ``System.explore_par``: the tree's edges, fingerprints and
    counters on the host; configuration rows fetched on demand (``rows``)."""

    def __init__(self, sys: System, h, status: int):
        L = lib()
        self._h, self.m, self.status = h, sys.m, status
        self.error = L.oracle_prun_error(h).decode() if h else ""
        nc = L.oracle_prun_num_configs(h)
        nl = L.oracle_prun_num_levels(h)
        ne = L.oracle_prun_num_expanded(h)
        self.level_offsets = np.zeros(nl + 1, np.int64)
        L.oracle_prun_level_offsets(h, _ptr(self.level_offsets))
        self.parent = np.zeros(nc, np.int64)
        self.t = np.zeros(nc, np.uint64)
        self.halting = np.zeros(nc, np.uint8)
        self.fp = np.zeros((nc, 2), np.uint64)
        L.oracle_prun_tree(h, _ptr(self.parent), _ptr(self.t), _ptr(self.halting), _ptr(self.fp))
        T, nn, kp = (np.zeros(ne, np.int64) for _ in range(3))
        L.oracle_prun_counters(h, _ptr(T), _ptr(nn), _ptr(kp))
        self.counters = Counters(T, nn, kp)

    def rows(self, idx) -> np.ndarray:
        idx = np.ascontiguousarray(idx, np.int64)
        out = np.zeros((idx.shape[0], self.m), np.int32)
        lib().oracle_prun_rows(self._h, _ptr(idx), idx.shape[0], _ptr(out))
        return out

    @property
    def num_levels(self) -> int:
        return len(self.level_offsets) - 1

    def close(self):
        if self._h:
            lib().oracle_prun_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class Counters:
    T: np.ndarray
    new: np.ndarray
    kept: np.ndarray


class Run:
    """Result of ``System.explore`` — the BFS computation tree."""

    def __init__(self, sys: System, h, status: int, width: int | None = None):
        L = lib()
        width = sys.m if width is None else width
        self.status = status
        self.error = L.oracle_run_error(h).decode() if h else ""
        try:
            nc = L.oracle_run_num_configs(h)
            nl = L.oracle_run_num_levels(h)
            ne = L.oracle_run_num_expanded(h)
            self.level_offsets = np.zeros(nl + 1, np.int64)
            L.oracle_run_level_offsets(h, _ptr(self.level_offsets))
            self.configs = np.zeros((nc, width), np.int64)
            L.oracle_run_configs(h, width, _ptr(self.configs))
            self.parent = np.zeros(nc, np.int64)
            self.t = np.zeros(nc, np.uint64)
            self.halting = np.zeros(nc, np.uint8)
            self.fp = np.zeros((nc, 2), np.uint64)
            if status == OR_OK:
                L.oracle_run_tree(h, _ptr(self.parent), _ptr(self.t), _ptr(self.halting), _ptr(self.fp))
            T = np.zeros(ne, np.int64)
            nn = np.zeros(ne, np.int64)
            kp = np.zeros(ne, np.int64)
            L.oracle_run_counters(h, _ptr(T), _ptr(nn), _ptr(kp))
            self.counters = Counters(T, nn, kp)
            nums = np.zeros(L.oracle_run_num_numbers(h), np.int64)
            L.oracle_run_numbers(h, _ptr(nums))
            self.numbers = set(int(x) for x in nums)
            # reading A17: every transition of expanded level L -> configuration index (-1 = not stored)
            self.edge_ref = []
            for lv in range(ne):
                e = np.zeros(L.oracle_run_num_edges(h, lv), np.int64)
                L.oracle_run_edges(h, lv, _ptr(e))
                self.edge_ref.append(e)
        finally:
            L.oracle_run_free(h)

    def level(self, L: int) -> np.ndarray:
        return self.configs[self.level_offsets[L]:self.level_offsets[L + 1]]

    @property
    def num_levels(self) -> int:
        return len(self.level_offsets) - 1


def fingerprint(C, seeds=(0x5EED0, 0x5EED1)):
    C = np.ascontiguousarray(C, dtype=np.int64)
    out = np.zeros(2, np.uint64)
    lib().oracle_fingerprint(_ptr(C), C.shape[0], seeds[0], seeds[1], _ptr(out))
    return int(out[0]), int(out[1])


def fmix64(k: int) -> int:
    return int(lib().oracle_fmix64(k))


def thinning_tau(F: int, n_new: int) -> int:
    return int(lib().oracle_thinning_tau(F, n_new))
