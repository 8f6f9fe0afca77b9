"""Multi-GPU exploration driver (one process per GPU).

The library runs every level itself (include/snp.h, ``snp_dist_advance``):
local K-a/K-b, the key all-to-all to owner = fmix64(fp1) mod P, owner-side
dedup and thinning, the verdict all-to-all back, local K-c and, when the
frontier drifts out of balance, the row redistribution — all exchanges issued
by libsnp.so on the engine's stream (NCCL over NVLink between processes, or
device-to-device copies between the logical ranks of one process).  This
module only sets the transport up: torch.distributed broadcasts the NCCL
unique id once (setup, outside every level), or a ``LocalGroup`` joins P
engine handles of one process.

The frontier stays range-partitioned by rank, so the global order and every
result equal a 1-GPU run (the digest is additive over ranks).
"""
from __future__ import annotations

import ctypes

from . import snp


def level0_slice(F0: int, rank: int, P: int):
    """contiguous range of the global level 0 held by `rank`."""
    lo = F0 * rank // P
    hi = F0 * (rank + 1) // P
    return lo, hi


def unique_id_bytes() -> bytes:
    """snp_dist_unique_id: the NCCL unique id (rank 0 creates it)."""
    buf = ctypes.create_string_buffer(snp.SNP_DIST_ID_BYTES)
    snp._check(snp.lib().snp_dist_unique_id(buf))
    return buf.raw


def broadcast_unique_id(group=None) -> bytes:
    """rank 0's NCCL unique id on every rank (torch.distributed, host objects;
    called once before the first level)."""
    import torch.distributed as dist
    obj = [unique_id_bytes() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class LocalGroup:
    """snp_local_group: P logical ranks (engine handles) of ONE process."""

    def __init__(self, P: int):
        self.P = P
        self._h = ctypes.c_void_p()
        snp._check(snp.lib().snp_local_group_create(P, ctypes.byref(self._h)))

    def close(self):
        if self._h:
            snp.lib().snp_local_group_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistExplorer:
    """Explore one SNP system over P ranks.  transport: None → NCCL with the
    torch.distributed rank / world size (unique id broadcast once); or a
    ``(LocalGroup, rank)`` pair for logical ranks inside one process."""

    def __init__(self, system: snp.System, transport=None, rebalance: float = 1.1, group=None):
        self.sys = system
        self.L = snp.lib()
        if transport is None:
            import torch.distributed as dist
            self.rank, self.P = dist.get_rank(group), dist.get_world_size(group)
            uid = broadcast_unique_id(group)
            snp._check(self.L.snp_dist_init(system._h, uid, self.rank, self.P))
        else:
            grp, self.rank = transport
            self.P = grp.P
            self._group = grp  # the handles keep their own reference; this keeps the wrapper alive
            snp._check(self.L.snp_dist_init_local(system._h, grp._h, self.rank))
        snp._check(self.L.snp_dist_set_rebalance(system._h, float(rebalance)))
        self.depth = -1

    def begin(self, level0_local: "snp.snp_configs") -> int:
        """level0_local: this rank's contiguous slice of the global level 0;
        returns the global level-0 size."""
        F = ctypes.c_int64()
        snp._check(self.L.snp_dist_start(self.sys._h, ctypes.byref(level0_local), ctypes.byref(F)))
        self.depth = 0
        return int(F.value)

    def advance(self) -> dict:
        lc, lo = snp.snp_level_counters(), snp.snp_level_counters()
        snp._check(self.L.snp_dist_advance(self.sys._h, ctypes.byref(lc), ctypes.byref(lo)))
        self.depth += 1
        d = lc.as_dict()
        F, off, moved = self.local()
        d.update(parents_local=lo.parents, T_local=lo.T, kept_local=lo.kept, frontier_local=F, global_offset=off,
                 rebalanced_rows=moved)
        return d

    def local(self):
        """(local frontier size, its global offset, rows sent in the last rebalancing)."""
        F, off, moved = (ctypes.c_int64() for _ in range(3))
        snp._check(self.L.snp_dist_local(self.sys._h, ctypes.byref(F), ctypes.byref(off), ctypes.byref(moved)))
        return int(F.value), int(off.value), int(moved.value)

    def summary(self):
        """global (configurations, transitions, digest) — a collective call."""
        n, T, d = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_uint64()
        snp._check(self.L.snp_dist_summary(self.sys._h, ctypes.byref(n), ctypes.byref(T), ctypes.byref(d)))
        return int(n.value), int(T.value), int(d.value)
