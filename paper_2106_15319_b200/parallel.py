"""Realization sharding across GPUs.

EEMD realizations are independent units: rank r of W owns the contiguous
range shard_range(nr, r, W) and runs them on its own GPU (seeds derive from
the GLOBAL realization index, emd.cpp:238, so the work of realization m is
identical on any rank). The only exchange is the ensemble mean: an
all-reduce(max) of the IMF count and one all-reduce(sum) of the K x L partial
sums (NCCL over NVLink on GPUs; gloo in the CPU tests), followed by the same
finish on every rank (emd.cpp:252-260). No collective inside the sift loop.
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def shard_range(nr: int, rank: int, world: int) -> tuple[int, int]:
    per = -(-nr // world)
    b = min(nr, rank * per)
    return b, min(nr, b + per)


def sharded_ensemble(nr: int, rank: int, world: int,
                     partial: Callable[[int, int], tuple[object, int]],
                     allreduce_max: Callable[[int], int],
                     allreduce_sum: Callable[[object, int], object],
                     finish: Callable[[object, int], object]):
    """Generic driver: partial(m_begin, m_end) -> (sums, K_local);
    allreduce_sum(sums, K) returns the K-row global sums; finish(sums, K)."""
    mb, me = shard_range(nr, rank, world)
    sums, k_local = partial(mb, me)
    K = allreduce_max(k_local)
    total = allreduce_sum(sums, K)
    return finish(total, K)


# ------------------------------------------------------------- torch / GPU driver

def eemd_distributed(x_dev, n: int, cfg: dict, ens: dict, rank: int, world: int, ctx=None, k_cap: int = 64,
                     group=None):
    """EEMD on this rank's GPU shard + NCCL all-reduce; returns (imfs (K, n), residue) torch tensors.

    x_dev: torch.float64 CUDA tensor of the serialized signal (resident in HBM).
    """
    import ctypes as C

    import torch
    import torch.distributed as dist

    from . import _native as N
    from .api import context

    c = ctx or context(x_dev.device.index or 0)
    scfg = N.SiftCfg(cfg.get("sd_threshold", 0.2), cfg.get("max_sift_iters", 300), cfg.get("max_imfs", 0))
    ecfg = N.EnsCfg(ens.get("nstd", 0.2), ens.get("nr", 100), 0, ens.get("base_seed", 0))
    nr = ecfg.nr
    state = {}

    def partial(mb, me):
        sums = torch.zeros((k_cap, n), dtype=torch.float64, device=x_dev.device)
        kout = C.c_size_t()
        c.check(c.lib.semd_eemd_partial_device(c.ptr, C.c_void_p(x_dev.data_ptr()), n, C.byref(scfg), C.byref(ecfg),
                                               mb, me, C.c_void_p(sums.data_ptr()), k_cap, C.byref(kout)))
        state["stats"] = c.stats()
        return sums, int(kout.value)

    def amax(k):
        if world == 1:
            return k
        t = torch.tensor([k], dtype=torch.int64, device=x_dev.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return int(t.item())

    def asum(sums, K):
        s = sums[:K].contiguous()
        if world > 1 and K:
            dist.all_reduce(s, op=dist.ReduceOp.SUM, group=group)
        return s

    def finish(total, K):
        residue = torch.empty(n, dtype=torch.float64, device=x_dev.device)
        c.check(c.lib.semd_ensemble_finish_device(c.ptr, C.c_void_p(x_dev.data_ptr()), n,
                                                  C.c_void_p(total.data_ptr()), K, nr, C.c_void_p(residue.data_ptr())))
        return total, residue

    imfs, residue = sharded_ensemble(nr, rank, world, partial, amax, asum, finish)
    return imfs, residue, state.get("stats", {})


# ------------------------------------------------------------- numpy reference driver (tests)

def finish_numpy(x: np.ndarray, sums: np.ndarray, K: int, nr: int):
    """emd.cpp:252-260 restated for the host-logic tests."""
    inv = 1.0 / float(nr)
    imfs = sums[:K] * inv
    residue = x.copy()
    for k in range(K):
        residue = residue - imfs[k]
    return imfs, residue
