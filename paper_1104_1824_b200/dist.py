"""Multi-GPU exploration driver: one process per GPU, torch.distributed (NCCL)
for the collectives only — plumbing between the snp_dist_* calls of libsnp.so
(include/snp.h).  Every step of the method (applicability, Ψ, decode, keys,
owner-side dedup, thinning, C + S·M) runs in the library's CUDA kernels.

Per level:
  1. snp_dist_expand                 local children keys, local T
  2. all_gather(T) → global tag base of this rank
  3. snp_dist_pack                   keys grouped by owner = fmix64(fp1) mod P
  4. all_to_all(counts), all_to_all(keys)        (keys only: 24 B per child)
  5. snp_dist_owner_dedup            owner's visited shard + level table
  6. all_reduce(N_new)               → global thinning threshold τ
  7. snp_dist_owner_keep             verdicts (1 B per key) for the producers
  8. all_to_all(verdicts back)
  9. snp_dist_finalize               local kept count K
 10. all_gather(K, F) → global offsets; snp_dist_commit (K-c materialization)

The frontier stays range-partitioned by rank, so the global order and every
result equal a 1-GPU run (the digest is additive over ranks).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import snp

M64 = (1 << 64) - 1


# ---- collective helpers (pure plumbing; also exercised with gloo in tests) ----
def all_gather_ints(values, device, group=None):
    """all_gather of a small vector of python ints → list of lists (rank order)."""
    t = torch.tensor(list(values), dtype=torch.int64, device=device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return [o.tolist() for o in out]


def all_reduce_int(v: int, device, group=None) -> int:
    t = torch.tensor([v], dtype=torch.int64, device=device)
    dist.all_reduce(t, group=group)
    return int(t.item())


def exchange(send: torch.Tensor, send_counts, group=None):
    """all-to-all-v along dim 0: rows [Σ_{r'<r} send_counts[r'], +send_counts[r]) go to rank r.
    Returns (recv, recv_counts)."""
    P = dist.get_world_size(group)
    sc = torch.tensor(list(send_counts), dtype=torch.int64, device=send.device)
    rc = torch.empty(P, dtype=torch.int64, device=send.device)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = rc.tolist()
    recv = torch.empty((sum(recv_counts),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send, output_split_sizes=recv_counts, input_split_sizes=list(send_counts),
                           group=group)
    return recv, recv_counts


def exchange_back(verdict: torch.Tensor, recv_counts, send_counts, group=None) -> torch.Tensor:
    """the reverse all-to-all-v: what rank r received comes back to it in send order."""
    back = torch.empty((sum(send_counts),) + tuple(verdict.shape[1:]), dtype=verdict.dtype, device=verdict.device)
    dist.all_to_all_single(back, verdict, output_split_sizes=list(send_counts), input_split_sizes=list(recv_counts),
                           group=group)
    return back


def level0_slice(F0: int, rank: int, P: int):
    """contiguous range of the global level 0 held by `rank`."""
    lo = F0 * rank // P
    hi = F0 * (rank + 1) // P
    return lo, hi


class TorchComm:
    """The collectives DistExplorer needs, over a torch.distributed group."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.P = dist.get_world_size(group)

    def all_gather_ints(self, values, device):
        return all_gather_ints(values, device, self.group)

    def all_reduce_int(self, v, device):
        return all_reduce_int(v, device, self.group)

    def exchange(self, send, counts):
        return exchange(send, counts, self.group)

    def exchange_back(self, verdict, recv_counts, send_counts):
        return exchange_back(verdict, recv_counts, send_counts, self.group)

    def all_reduce_u64(self, v: int, device) -> int:
        t = torch.tensor([v - (1 << 64) if v >= (1 << 63) else v], dtype=torch.int64, device=device)
        dist.all_reduce(t, group=self.group)
        return int(t.item()) & M64


class DistExplorer:
    """Explore one SNP system over the ranks of a communicator (one GPU each)."""

    def __init__(self, system: snp.System, comm=None):
        self.sys = system
        self.comm = comm if comm is not None else TorchComm()
        self.rank = self.comm.rank
        self.P = self.comm.P
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.L = snp.lib()
        self.F_local = 0
        self.depth = -1
        self.T_total = 0
        self.n_configs = 0

    def _check(self, st):
        snp._check(st)

    def _keys_round(self, T_local: int):
        """steps 2-9 of the module docstring; returns (n_new_global, K_local, T_global)."""
        T_all = [r[0] for r in self.comm.all_gather_ints([T_local], self.device)]
        tag_base = sum(T_all[: self.rank])
        send = torch.empty((T_local, 3), dtype=torch.int64, device=self.device)
        counts = np.zeros(self.P, np.int64)
        torch.cuda.synchronize()
        self._check(self.L.snp_dist_pack(self.sys._h, tag_base, send.data_ptr() if T_local else None,
                                         counts.ctypes.data_as(ctypes.c_void_p)))
        recv, recv_counts = self.comm.exchange(send, counts.tolist())
        torch.cuda.synchronize()
        R = int(sum(recv_counts))
        n_new_local = ctypes.c_int64()
        self._check(self.L.snp_dist_owner_dedup(self.sys._h, recv.data_ptr() if R else None, R,
                                                ctypes.byref(n_new_local)))
        n_new = self.comm.all_reduce_int(n_new_local.value, self.device)
        verdict = torch.empty(R, dtype=torch.uint8, device=self.device)
        torch.cuda.synchronize()
        self._check(self.L.snp_dist_owner_keep(self.sys._h, n_new, verdict.data_ptr() if R else None))
        back = self.comm.exchange_back(verdict, recv_counts, counts.tolist())
        torch.cuda.synchronize()
        K = ctypes.c_int64()
        self._check(self.L.snp_dist_finalize(self.sys._h, back.data_ptr() if T_local else None, ctypes.byref(K)))
        del recv, send, verdict, back
        return n_new, int(K.value), sum(T_all)

    def _commit(self, K_local: int):
        KF = self.comm.all_gather_ints([K_local, self.F_local], self.device)
        q_off = sum(k for k, _ in KF[: self.rank])
        p_off = sum(f for _, f in KF[: self.rank])
        lc = snp.snp_level_counters()
        self._check(self.L.snp_dist_commit(self.sys._h, p_off, q_off, ctypes.byref(lc)))
        self.F_local = K_local
        return lc, sum(k for k, _ in KF)

    def begin(self, level0_local: "snp.snp_configs") -> int:
        """level0_local: this rank's contiguous slice of the global level 0."""
        n = ctypes.c_int64()
        self._check(self.L.snp_dist_begin(self.sys._h, ctypes.byref(level0_local), self.P, ctypes.byref(n)))
        _n_new, K, _ = self._keys_round(int(n.value))
        self.F_local = 0
        _, K_total = self._commit(K)
        self.depth = 0
        self.n_configs = K_total
        self.T_total = 0
        return K_total

    def advance(self) -> dict:
        T_local = ctypes.c_int64()
        self._check(self.L.snp_dist_expand(self.sys._h, ctypes.byref(T_local)))
        n_new, K, T_total = self._keys_round(int(T_local.value))
        lc, K_total = self._commit(K)
        halting = self.comm.all_reduce_int(int(lc.halting), self.device)
        parents = self.comm.all_reduce_int(int(lc.parents), self.device)
        self.depth += 1
        self.T_total += T_total
        self.n_configs += K_total
        return {"parents": parents, "halting": halting, "T": T_total, "n_new": n_new, "kept": K_total,
                "tau": int(lc.tau), "ms": lc.ms, "parents_local": int(lc.parents), "kept_local": K,
                "T_local": int(lc.T)}

    @property
    def frontier_size_local(self) -> int:
        return self.F_local

    def summary(self):
        """global (configurations, transitions, digest); the digest is the sum of
        the ranks' digests mod 2^64 and equals the 1-GPU digest."""
        _n, _T, d = self.sys.summary()
        return self.n_configs, self.T_total, self.comm.all_reduce_u64(d, self.device)
