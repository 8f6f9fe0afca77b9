"""Thin Python binding of libsnp.so (include/snp.h): argument marshalling only.

Every step of the transition path runs in the CUDA kernels behind the C ABI.
There is no CPU fallback: if ``libsnp.so`` is missing or no CUDA device is
present, loading a system raises ``SnpError`` (status SNP_E_CUDA).

The functions keep the C names (``snp_load``, ``snp_begin``, ``snp_advance``,
``snp_explore``, ``snp_step``, ``snp_tree_*``); ``System`` / ``Tree`` are small
owning wrappers around the handles.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

SNP_OK = 0
SNP_E_ARG = -1
SNP_E_INVALID_SYSTEM = -2
SNP_E_OVERFLOW = -3
SNP_E_CAPACITY = -4
SNP_E_OOM = -5
SNP_E_CUDA = -6
SNP_E_NCCL = -7
SNP_E_COLLISION = -8
SNP_E_STATE = -9

SNP_LAYOUT_ROW_MAJOR = 0
SNP_LAYOUT_NEURON_MAJOR = 1

EXPORTED = [
    "snp_abi_version", "snp_last_error", "snp_load", "snp_load_unary", "snp_load_delay", "snp_system_free", "snp_set_stream", "snp_begin",
    "snp_advance", "snp_frontier_size", "snp_state_width", "snp_generated_numbers", "snp_depth", "snp_summary",
    "snp_explore", "snp_step", "snp_sample",
    "snp_tree_num_levels", "snp_tree_num_configs", "snp_tree_level_offsets", "snp_tree_configs",
    "snp_tree_edges", "snp_tree_counters", "snp_tree_spiking_vectors", "snp_tree_free",
    "snp_level_size", "snp_level_edges", "snp_level_columns", "snp_set_profiling", "snp_profile",
    "snp_kernel_launches", "snp_kernel_paths", "snp_host_alloc", "snp_host_free", "snp_dist_begin", "snp_dist_expand", "snp_dist_pack", "snp_dist_owner_dedup",
    "snp_dist_owner_keep", "snp_dist_finalize", "snp_dist_commit",
    "snp_spiking_vector", "snp_level_spiking_vectors", "snp_frontier_copy", "snp_level_all_edges",
    "snp_dist_unique_id", "snp_dist_init", "snp_local_group_create", "snp_local_group_free", "snp_dist_init_local",
    "snp_dist_set_rebalance", "snp_dist_start", "snp_dist_advance", "snp_dist_summary", "snp_dist_local",
    "snp_set_device",
]
SNP_DIST_ID_BYTES = 128
SNP_NUM_PHASES = 5
SNP_PATH_TC_EXPAND = 1
PHASES = ["expand", "keys", "dedup", "materialize", "verify"]


class snp_rule(ctypes.Structure):
    _fields_ = [("neuron", ctypes.c_int32), ("kind", ctypes.c_int32), ("a", ctypes.c_int32),
                ("b", ctypes.c_int32), ("consumed", ctypes.c_int32), ("produced", ctypes.c_int32)]


class snp_matrix(ctypes.Structure):
    _fields_ = [("n_rules", ctypes.c_int64), ("n_neurons", ctypes.c_int64), ("dense", ctypes.c_void_p),
                ("row_ptr", ctypes.c_void_p), ("col", ctypes.c_void_p), ("val", ctypes.c_void_p)]


class snp_options(ctypes.Structure):
    _fields_ = [("count_bits", ctypes.c_int32), ("dedup", ctypes.c_int32), ("frontier_target", ctypes.c_int64),
                ("max_transitions", ctypes.c_int64), ("fp_seed", ctypes.c_uint64 * 2),
                ("keep_tree", ctypes.c_int32), ("out_rule1", ctypes.c_int32), ("keep_all_edges", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class snp_configs(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("n_configs", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("elem_bytes", ctypes.c_int32), ("layout", ctypes.c_int32), ("on_device", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class snp_level_counters(ctypes.Structure):
    _fields_ = [("parents", ctypes.c_int64), ("halting", ctypes.c_int64), ("T", ctypes.c_int64),
                ("n_new", ctypes.c_int64), ("kept", ctypes.c_int64), ("tau", ctypes.c_uint64),
                ("ms", ctypes.c_double), ("overflow_fixes", ctypes.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_P = ctypes.c_void_p
_lib = None


class SnpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"snp status {status}: {msg}")
        self.status = status


def lib() -> ctypes.CDLL:
    """Load libsnp.so (building it in-tree if it is missing or stale)."""
    global _lib
    if _lib is None:
        path = os.environ.get("SNP_LIB")  # tuning aid: an in-tree variant build (tools/gpu_ab.sh)
        if not path:
            if not os.path.exists(_build.LIB_SNP) or os.environ.get("SNP_REBUILD"):
                _build.build()
            path = _build.LIB_SNP
        L = ctypes.CDLL(path)
        L.snp_abi_version.restype = ctypes.c_int
        L.snp_last_error.restype = ctypes.c_char_p
        L.snp_load.argtypes = [ctypes.POINTER(snp_matrix), _P, ctypes.c_int64, _P, ctypes.c_int64,
                               ctypes.POINTER(snp_options), ctypes.POINTER(_P)]
        L.snp_system_free.argtypes = [_P]
        L.snp_set_stream.argtypes = [_P, _P]
        L.snp_begin.argtypes = [_P, ctypes.POINTER(snp_configs)]
        L.snp_advance.argtypes = [_P, ctypes.POINTER(snp_level_counters)]
        L.snp_frontier_size.argtypes = [_P]
        L.snp_frontier_size.restype = ctypes.c_int64
        L.snp_load_unary.argtypes = [ctypes.POINTER(snp_matrix), _P, ctypes.c_int64, _P, _P, ctypes.c_int64,
                                     ctypes.POINTER(snp_options), ctypes.POINTER(_P)]
        L.snp_load_delay.argtypes = [ctypes.POINTER(snp_matrix), _P, ctypes.c_int64, _P, _P, ctypes.c_int64,
                                     ctypes.POINTER(snp_options), ctypes.POINTER(_P)]
        L.snp_state_width.argtypes = [_P]
        L.snp_state_width.restype = ctypes.c_int64
        L.snp_generated_numbers.argtypes = [_P, _P, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
        L.snp_depth.argtypes = [_P]
        L.snp_depth.restype = ctypes.c_int32
        L.snp_summary.argtypes = [_P, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                  ctypes.POINTER(ctypes.c_uint64)]
        L.snp_explore.argtypes = [_P, ctypes.POINTER(snp_configs), ctypes.c_int32, ctypes.POINTER(_P)]
        L.snp_step.argtypes = [_P, ctypes.POINTER(snp_configs), ctypes.POINTER(_P)]
        L.snp_tree_num_levels.argtypes = [_P]
        L.snp_tree_num_levels.restype = ctypes.c_int32
        L.snp_tree_num_configs.argtypes = [_P]
        L.snp_tree_num_configs.restype = ctypes.c_int64
        L.snp_tree_level_offsets.argtypes = [_P, _P]
        L.snp_tree_configs.argtypes = [_P, _P]
        L.snp_tree_edges.argtypes = [_P, _P, _P, _P, _P]
        L.snp_tree_counters.argtypes = [_P, _P]
        L.snp_tree_spiking_vectors.argtypes = [_P, ctypes.c_int32, _P]
        L.snp_tree_free.argtypes = [_P]
        L.snp_level_size.argtypes = [_P, ctypes.c_int32]
        L.snp_level_size.restype = ctypes.c_int64
        L.snp_level_edges.argtypes = [_P, ctypes.c_int32, _P, _P, _P, _P]
        L.snp_host_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]
        L.snp_host_free.argtypes = [_P]
        L.snp_level_columns.argtypes = [_P, ctypes.c_int32, _P, ctypes.c_int64, _P]
        L.snp_set_profiling.argtypes = [_P, ctypes.c_int32]
        L.snp_profile.argtypes = [_P, _P]
        L.snp_kernel_launches.restype = ctypes.c_int64
        L.snp_set_device.argtypes = [ctypes.c_int32]
        L.snp_sample.argtypes = [_P, ctypes.c_int64, _P, ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32, _P,
                                 ctypes.c_int32, _P]
        L.snp_kernel_paths.argtypes = [_P]
        L.snp_kernel_paths.restype = ctypes.c_int32
        _I64P = ctypes.POINTER(ctypes.c_int64)
        L.snp_dist_begin.argtypes = [_P, ctypes.POINTER(snp_configs), ctypes.c_int32, _I64P]
        L.snp_dist_expand.argtypes = [_P, _I64P]
        L.snp_dist_pack.argtypes = [_P, ctypes.c_uint64, _P, _P]
        L.snp_dist_owner_dedup.argtypes = [_P, _P, ctypes.c_int64, _I64P]
        L.snp_dist_owner_keep.argtypes = [_P, ctypes.c_int64, _P]
        L.snp_dist_finalize.argtypes = [_P, _P, _I64P]
        L.snp_dist_commit.argtypes = [_P, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(snp_level_counters)]
        L.snp_spiking_vector.argtypes = [_P, _P, ctypes.c_uint64, _P]
        L.snp_level_spiking_vectors.argtypes = [_P, ctypes.c_int32, _P, ctypes.c_int64, _P]
        L.snp_frontier_copy.argtypes = [_P, _P, _P, _P, ctypes.c_int64, _I64P]
        L.snp_level_all_edges.argtypes = [_P, ctypes.c_int32, _P, _P, _P, ctypes.c_int64, _I64P]
        L.snp_dist_unique_id.argtypes = [_P]
        L.snp_dist_init.argtypes = [_P, _P, ctypes.c_int32, ctypes.c_int32]
        L.snp_local_group_create.argtypes = [ctypes.c_int32, ctypes.POINTER(_P)]
        L.snp_local_group_free.argtypes = [_P]
        L.snp_dist_init_local.argtypes = [_P, _P, ctypes.c_int32]
        L.snp_dist_set_rebalance.argtypes = [_P, ctypes.c_double]
        L.snp_dist_start.argtypes = [_P, ctypes.POINTER(snp_configs), _I64P]
        L.snp_dist_advance.argtypes = [_P, ctypes.POINTER(snp_level_counters), ctypes.POINTER(snp_level_counters)]
        L.snp_dist_summary.argtypes = [_P, _I64P, _I64P, ctypes.POINTER(ctypes.c_uint64)]
        L.snp_dist_local.argtypes = [_P, _I64P, _I64P, _I64P]
        for f in EXPORTED:
            if f not in ("snp_kernel_launches", "snp_kernel_paths", "snp_system_free", "snp_tree_free", "snp_frontier_size", "snp_depth", "snp_level_size", "snp_local_group_free",
                         "snp_tree_num_levels", "snp_tree_num_configs", "snp_abi_version", "snp_last_error"):
                getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(st: int):
    if st != SNP_OK:
        raise SnpError(st, lib().snp_last_error().decode(errors="replace"))


def _check_allow(st: int, *ok):
    if st != SNP_OK and st not in ok:
        _check(st)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class PinnedHost:
    """Pinned host bytes from snp_host_alloc, freed by snp_host_free."""

    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        _check(lib().snp_host_alloc(ctypes.c_size_t(nbytes), ctypes.byref(p)))
        self.p, self.nbytes = p, nbytes

    def array(self, offset: int, shape, dtype) -> np.ndarray:
        """A numpy view of bytes [offset, offset + size); the view keeps this
        PinnedHost alive (its base chain holds it), so the pinned block is
        freed only after the last view is gone."""
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        assert offset + n <= self.nbytes
        buf = (ctypes.c_uint8 * n).from_address(self.p.value + offset)
        buf._owner = self
        return np.frombuffer(buf, dtype=dtype).reshape(shape)

    def __del__(self):
        try:
            if self.p:
                lib().snp_host_free(self.p)
                self.p = None
        except Exception:
            pass


class PinnedEdges:
    """Pinned parent / t / halting / fp buffers for up to cap configurations."""

    def __init__(self, cap: int):
        self.cap = cap
        self.mem = PinnedHost(cap * (8 + 8 + 16) + cap)

    def views(self, F: int):
        c = self.cap
        return (self.mem.array(0, (F,), np.int64), self.mem.array(8 * c, (F,), np.uint64),
                self.mem.array(32 * c, (F,), np.uint8), self.mem.array(16 * c, (F, 2), np.uint64))


# ---- C-named entry points (marshalling only) --------------------------------
def snp_load(rules: np.ndarray, row_ptr: np.ndarray, col: np.ndarray, val: np.ndarray, C0: np.ndarray,
             count_bits=32, dedup=0, frontier_target=0, max_transitions=0, fp_seed=(0x5EED0, 0x5EED1),
             keep_tree=1, out_rule=None, re_bits=None, delays=None, keep_all_edges=0):
    rules = np.ascontiguousarray(rules, np.int32).reshape(-1, 6)
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    val = np.ascontiguousarray(val, np.int32)
    C0 = np.ascontiguousarray(C0, np.int32)
    M = snp_matrix(rules.shape[0], C0.shape[0], None, _ptr(row_ptr).value, _ptr(col).value, _ptr(val).value)
    o = snp_options(count_bits, dedup, frontier_target, max_transitions, (ctypes.c_uint64 * 2)(*fp_seed),
                    keep_tree, 0 if out_rule is None else int(out_rule) + 1, int(keep_all_edges), 0)
    h = _P()
    if delays is not None:
        d = np.ascontiguousarray(delays, np.int32)
        if d.shape != (rules.shape[0],):
            raise ValueError("delays: one int32 per rule")
        _check(lib().snp_load_delay(ctypes.byref(M), _ptr(rules), rules.shape[0], _ptr(d), _ptr(C0), C0.shape[0],
                                    ctypes.byref(o), ctypes.byref(h)))
    elif re_bits is None:
        _check(lib().snp_load(ctypes.byref(M), _ptr(rules), rules.shape[0], _ptr(C0), C0.shape[0], ctypes.byref(o),
                              ctypes.byref(h)))
    else:
        bits = np.ascontiguousarray(re_bits, np.uint64).reshape(-1, 4)
        _check(lib().snp_load_unary(ctypes.byref(M), _ptr(rules), rules.shape[0], _ptr(bits), _ptr(C0), C0.shape[0],
                                    ctypes.byref(o), ctypes.byref(h)))
    return h


def configs_from_host(a: np.ndarray, layout=SNP_LAYOUT_ROW_MAJOR) -> tuple:
    a = np.ascontiguousarray(np.atleast_2d(a))
    if a.dtype not in (np.uint8, np.uint16, np.int32):
        a = a.astype(np.int32)
    n = a.shape[0] if layout == SNP_LAYOUT_ROW_MAJOR else a.shape[1]
    c = snp_configs(_ptr(a).value, n, a.shape[1], a.dtype.itemsize, layout, 0, 0)
    return c, a  # keep `a` alive


def configs_from_device(ptr: int, n_configs: int, ld: int, elem_bytes: int, layout=SNP_LAYOUT_NEURON_MAJOR):
    return snp_configs(ptr, n_configs, ld, elem_bytes, layout, 1, 0)


class System:
    """Owning wrapper of an ``snp_system*``."""

    def __init__(self, workload, count_bits=32, dedup=0, frontier_target=0, max_transitions=0,
                 fp_seed=(0x5EED0, 0x5EED1), keep_tree=1, out_rule=None, delays=None, keep_all_edges=0):
        """out_rule: generated numbers (include/snp.h) with that output rule;
        configurations then have ``width = m + 1`` entries (last = A).
        delays: one d >= 0 per rule (snp_load_delay);
        configurations then have ``width = 3m`` entries [C | τ | π]."""
        self.m = int(workload.m)
        self.n = int(workload.rules.shape[0])
        self.count_bits = count_bits
        self._h = None
        self._h = snp_load(workload.rules, workload.row_ptr, workload.col, workload.val, workload.C0,
                           count_bits, dedup, frontier_target, max_transitions, fp_seed, keep_tree, out_rule,
                           getattr(workload, "re_bits", None), delays, keep_all_edges)
        self.width = int(lib().snp_state_width(self._h))

    def generated_numbers(self) -> set:
        """snp_generated_numbers: the numbers generated since the last begin."""
        mx = ctypes.c_int64(-1)
        _check(lib().snp_generated_numbers(self._h, None, 0, ctypes.byref(mx)))
        if mx.value < 0:
            return set()
        words = np.zeros(mx.value // 64 + 1, np.uint64)
        _check(lib().snp_generated_numbers(self._h, _ptr(words), words.shape[0], None))
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")
        return set(int(i) for i in np.nonzero(bits)[0])

    def sample(self, walkers, seed: int, steps: int, input_neuron: int = -1, train=None):
        """snp_sample: single-path sampling of W walkers;
        returns (final configurations W × m int32, halted_step W int32)."""
        C = np.ascontiguousarray(np.atleast_2d(walkers), dtype=np.int32).copy()
        if C.shape[1] != self.m:
            raise ValueError(f"walkers have {C.shape[1]} columns, the system has {self.m} neurons")
        tr = np.ascontiguousarray(np.zeros(0) if train is None else train, dtype=np.int32)
        hs = np.zeros(C.shape[0], np.int32)
        _check(lib().snp_sample(self._h, C.shape[0], _ptr(C), seed, steps, input_neuron,
                                _ptr(tr) if tr.size else None, tr.size, _ptr(hs)))
        return C, hs

    @property
    def kernel_paths(self) -> int:
        """snp_kernel_paths: SNP_PATH_* bits of the kernels this system runs."""
        return int(lib().snp_kernel_paths(self._h))

    def close(self):
        if self._h:
            lib().snp_system_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int):
        _check(lib().snp_set_stream(self._h, stream_handle))

    def begin(self, level0=None):
        if level0 is None:
            _check(lib().snp_begin(self._h, None))
        elif isinstance(level0, snp_configs):
            _check(lib().snp_begin(self._h, ctypes.byref(level0)))
        else:
            c, keep = configs_from_host(self._widen(level0))
            _check(lib().snp_begin(self._h, ctypes.byref(c)))

    def _widen(self, rows):
        """Generated-numbers mode: rows of m counts get A = 0 appended; delays
        mode: rows of m counts get τ = π = 0 (2m zero columns) appended."""
        rows = np.atleast_2d(rows)
        if self.width != self.m and rows.shape[1] == self.m:
            rows = np.hstack([rows, np.zeros((rows.shape[0], self.width - self.m), rows.dtype)])
        return rows

    def advance(self) -> dict:
        lc = snp_level_counters()
        _check(lib().snp_advance(self._h, ctypes.byref(lc)))
        return lc.as_dict()

    @property
    def frontier_size(self) -> int:
        return int(lib().snp_frontier_size(self._h))

    def summary(self):
        n = ctypes.c_int64()
        T = ctypes.c_int64()
        d = ctypes.c_uint64()
        _check(lib().snp_summary(self._h, ctypes.byref(n), ctypes.byref(T), ctypes.byref(d)))
        return int(n.value), int(T.value), int(d.value)

    def set_profiling(self, on: bool = True):
        _check(lib().snp_set_profiling(self._h, 1 if on else 0))

    def profile(self) -> dict:
        ms = np.zeros(SNP_NUM_PHASES, np.float64)
        _check(lib().snp_profile(self._h, _ptr(ms)))
        return dict(zip(PHASES, ms.tolist()))

    @property
    def depth(self) -> int:
        return int(lib().snp_depth(self._h))

    def level_size(self, L: int) -> int:
        return int(lib().snp_level_size(self._h, L))

    def reserve_edges(self, cap: int) -> None:
        """Allocate the pinned buffers level_edges(pinned=True) uses for up to
        cap configurations now (cudaHostAlloc is slow: keep it out of a loop)."""
        pb = getattr(self, "_pinned_edges", None)
        if pb is None or pb.cap < cap:
            self._pinned_edges = PinnedEdges(max(cap, 1))

    def level_edges(self, L: int, pinned: bool = False, halting: bool = True):
        """snp_level_edges into new numpy arrays, or (pinned=True) into pinned
        host buffers owned by this System and reused by the next pinned call
        (full PCIe rate; the returned arrays are views of them, valid until the
        next pinned call).  halting=False skips the flags (the newest level's
        are known only once it is expanded or classified); None is returned."""
        F = self.level_size(L)
        if pinned:
            pb = getattr(self, "_pinned_edges", None)
            if pb is None or pb.cap < F:
                pb = self._pinned_edges = PinnedEdges(max(F + F // 8, 1))  # headroom: thinned levels hover around F
            parent, t, hb, fp = pb.views(F)
        else:
            parent = np.empty(F, np.int64)
            t = np.empty(F, np.uint64)
            hb = np.empty(F, np.uint8)
            fp = np.empty((F, 2), np.uint64)
        _check(lib().snp_level_edges(self._h, L, _ptr(parent), _ptr(t), _ptr(hb) if halting else None, _ptr(fp)))
        return parent, t, (hb if halting else None), fp

    def spiking_vector(self, C, t: int) -> np.ndarray:
        """snp_spiking_vector: the t-th valid spiking vector of configuration C."""
        C = np.ascontiguousarray(C, np.int32).reshape(-1)
        S = np.zeros(self.n, np.uint8)
        _check(lib().snp_spiking_vector(self._h, _ptr(C), int(t), _ptr(S)))
        return S

    def level_spiking_vectors(self, L: int, idx) -> np.ndarray:
        """snp_level_spiking_vectors: S that produced configurations idx of level L."""
        idx = np.ascontiguousarray(idx, np.int64)
        out = np.zeros((idx.shape[0], self.n), np.uint8)
        _check(lib().snp_level_spiking_vectors(self._h, L, _ptr(idx), idx.shape[0], _ptr(out)))
        return out

    def frontier_copy(self):
        """snp_frontier_copy: (configs F × width int32, parent, t) of the newest level."""
        n = ctypes.c_int64()
        _check_allow(lib().snp_frontier_copy(self._h, None, None, None, 0, ctypes.byref(n)), SNP_E_CAPACITY)
        F = int(n.value)
        C = np.zeros((F, self.width), np.int32)
        parent = np.zeros(F, np.int64)
        t = np.zeros(F, np.uint64)
        _check(lib().snp_frontier_copy(self._h, _ptr(C), _ptr(parent), _ptr(t), F, ctypes.byref(n)))
        return C, parent, t

    def level_all_edges(self, L: int):
        """snp_level_all_edges: (parent, t, ref) of every transition that produced level L."""
        n = ctypes.c_int64()
        _check_allow(lib().snp_level_all_edges(self._h, L, None, None, None, 0, ctypes.byref(n)), SNP_E_CAPACITY)
        T = int(n.value)
        parent = np.zeros(T, np.int64)
        t = np.zeros(T, np.uint64)
        ref = np.zeros(T, np.int64)
        _check(lib().snp_level_all_edges(self._h, L, _ptr(parent), _ptr(t), _ptr(ref), T, ctypes.byref(n)))
        return parent, t, ref

    def level_columns(self, L: int, idx) -> np.ndarray:
        idx = np.ascontiguousarray(idx, np.int64)
        out = np.zeros((idx.shape[0], self.width), np.int32)
        _check(lib().snp_level_columns(self._h, L, _ptr(idx), idx.shape[0], _ptr(out)))
        return out

    def explore(self, level0=None, depth: int = 1) -> "Tree":
        h = _P()
        if level0 is None:
            _check(lib().snp_explore(self._h, None, depth, ctypes.byref(h)))
        elif isinstance(level0, snp_configs):
            _check(lib().snp_explore(self._h, ctypes.byref(level0), depth, ctypes.byref(h)))
        else:
            c, keep = configs_from_host(self._widen(level0))
            _check(lib().snp_explore(self._h, ctypes.byref(c), depth, ctypes.byref(h)))
        return Tree(self, h)

    def step(self, frontier) -> "Tree":
        h = _P()
        c, keep = configs_from_host(self._widen(frontier))
        _check(lib().snp_step(self._h, ctypes.byref(c), ctypes.byref(h)))
        return Tree(self, h)


@dataclass
class Counters:
    T: np.ndarray
    new: np.ndarray
    kept: np.ndarray
    halting: np.ndarray
    tau: np.ndarray
    ms: np.ndarray
    overflow_fixes: np.ndarray


class Tree:
    """Owning wrapper of an ``snp_tree*`` with host copies of its arrays."""

    def __init__(self, sys_: System, h):
        self.sys = sys_
        self._h = h
        L = lib()
        self.num_levels = int(L.snp_tree_num_levels(h))
        n = int(L.snp_tree_num_configs(h))
        self.level_offsets = np.zeros(self.num_levels + 1, np.int64)
        _check(L.snp_tree_level_offsets(h, _ptr(self.level_offsets)))
        self.parent = np.zeros(n, np.int64)
        self.t = np.zeros(n, np.uint64)
        self.halting = np.zeros(n, np.uint8)
        self.fp = np.zeros((n, 2), np.uint64)
        _check(L.snp_tree_edges(h, _ptr(self.parent), _ptr(self.t), _ptr(self.halting), _ptr(self.fp)))
        nl = max(self.num_levels - 1, 0)
        arr = (snp_level_counters * max(nl, 1))()
        _check(L.snp_tree_counters(h, ctypes.cast(arr, ctypes.c_void_p)))
        rows = [arr[i].as_dict() for i in range(nl)]
        self.counters = Counters(*(np.array([r[k] for r in rows]) for k in ("T", "n_new", "kept", "halting", "tau",
                                                                          "ms", "overflow_fixes")))
        self._configs = None

    @property
    def num_configs(self) -> int:
        return int(self.level_offsets[-1])

    @property
    def configs(self) -> np.ndarray:
        if self._configs is None:
            out = np.zeros((self.num_configs, self.sys.width), np.int32)
            _check(lib().snp_tree_configs(self._h, _ptr(out)))
            self._configs = out
        return self._configs

    def level(self, L: int) -> np.ndarray:
        return self.configs[self.level_offsets[L]:self.level_offsets[L + 1]]

    def spiking_vectors(self, L: int) -> np.ndarray:
        k = int(self.level_offsets[L + 1] - self.level_offsets[L])
        out = np.zeros((k, self.sys.n), np.uint8)
        _check(lib().snp_tree_spiking_vectors(self._h, L, _ptr(out)))
        return out

    def close(self):
        if self._h:
            lib().snp_tree_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def set_device(device: int) -> None:
    """snp_set_device: CUDA device `device` current inside libsnp.so (one
    process per GPU: its local rank, before the first System)."""
    _check(lib().snp_set_device(int(device)))


def snp_kernel_launches() -> int:
    return int(lib().snp_kernel_launches())


# ---- device level-0 generator (libsnpgen.so; inputs only) -------------------
_gen = None


def generate_level0_device(w, F: int, seed: int, dst_ptr: int, elem_bytes: int, layout: int, ld: int,
                           stream: int = 0, row_begin: int = 0):
    """Fill device memory with workloads.level0_counts(w, F, seed) (same values)."""
    global _gen
    from . import workloads as W
    if _gen is None:
        if not os.path.exists(_build.LIB_GEN):
            _build.build()
        _gen = ctypes.CDLL(_build.LIB_GEN)
        _gen.snpgen_level0.argtypes = [_P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                       ctypes.c_int64, ctypes.c_uint64, _P, ctypes.c_int64, _P]
        _gen.snpgen_level0.restype = ctypes.c_int
    rng = np.ascontiguousarray(w.level0_range, np.int32)
    st = _gen.snpgen_level0(dst_ptr, elem_bytes, layout, ld, w.m, F, W.level0_seed_key(seed), _ptr(rng), row_begin,
                            stream)
    if st != 0:
        raise SnpError(st, "snpgen_level0 failed")
