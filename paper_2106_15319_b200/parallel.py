"""Realization sharding across GPUs.

CEEMDAN (emd.cpp:264-344) shards the same way but exchanges once per stage:
each rank sums the first modes of its realizations, one all-reduce(sum) of L
doubles forms the global stage sum, and every rank applies the identical
mode / residue update and stop tests (sharded_ceemdan).

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


def sharded_ceemdan(nr: int, rank: int, world: int, engine, allreduce_sum: Callable[[object], object],
                    max_imfs: int = 0):
    """Generic CEEMDAN stage driver (emd.cpp:290-341) over an engine exposing
    begin(m_begin, m_end), stage() -> unscaled shard sum, finish(total, check_zero) -> accepted,
    residue_extrema() -> int and result() -> (modes, residue)."""
    mb, me = shard_range(nr, rank, world)
    engine.begin(mb, me)
    engine.finish(allreduce_sum(engine.stage()), False)  # mode 1
    k = 1
    while max_imfs == 0 or k < max_imfs:
        if engine.residue_extrema() < 3:  # emd.cpp:311
            break
        if not engine.finish(allreduce_sum(engine.stage()), True):  # all-zero mode, emd.cpp:332-337
            break
        k += 1
    return engine.result()


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


class GpuCeemdanShard:
    """sharded_ceemdan engine over the C ABI (semd_ceemdan_shard_*) on one GPU."""

    def __init__(self, ctx, x_dev, n: int, cfg: dict, ens: dict):
        import ctypes as C

        from . import _native as N
        self.C, self.c, self.x, self.n = C, ctx, x_dev, n
        self.scfg = N.SiftCfg(cfg.get("sd_threshold", 0.2), cfg.get("max_sift_iters", 300), cfg.get("max_imfs", 0))
        self.ecfg = N.EnsCfg(ens.get("nstd", 0.2), ens.get("nr", 100), 0, ens.get("base_seed", 0))
        self.modes = []

    def begin(self, mb, me):
        C, c = self.C, self.c
        c.check(c.lib.semd_ceemdan_shard_begin(c.ptr, C.c_void_p(self.x.data_ptr()), self.n, C.byref(self.scfg),
                                               C.byref(self.ecfg), mb, me))

    def stage(self):
        import torch
        part = torch.empty(self.n, dtype=torch.float64, device=self.x.device)
        self.c.check(self.c.lib.semd_ceemdan_shard_stage(self.c.ptr, self.C.c_void_p(part.data_ptr())))
        return part

    def finish(self, total, check_zero):
        import torch
        C, c = self.C, self.c
        mode = torch.empty(self.n, dtype=torch.float64, device=self.x.device)
        ok = C.c_int32()
        c.check(c.lib.semd_ceemdan_shard_finish_stage(c.ptr, C.c_void_p(total.data_ptr()), self.ecfg.nr,
                                                      int(check_zero), C.c_void_p(mode.data_ptr()), C.byref(ok)))
        if ok.value:
            self.modes.append(mode)
        return bool(ok.value)

    def residue_extrema(self):
        t = self.C.c_size_t()
        self.c.check(self.c.lib.semd_ceemdan_shard_residue_extrema(self.c.ptr, self.C.byref(t)))
        return int(t.value)

    def result(self):
        import torch
        res = torch.empty(self.n, dtype=torch.float64, device=self.x.device)
        self.c.check(self.c.lib.semd_ceemdan_shard_residue(self.c.ptr, self.C.c_void_p(res.data_ptr())))
        imfs = torch.stack(self.modes) if self.modes else torch.empty((0, self.n), dtype=torch.float64,
                                                                        device=self.x.device)
        return imfs, res


def ceemdan_distributed(x_dev, n: int, cfg: dict, ens: dict, rank: int, world: int, ctx=None, group=None):
    """CEEMDAN with realizations sharded over the ranks' GPUs and one NCCL all-reduce per stage;
    returns (imfs (K, n), residue) torch tensors (identical on every rank)."""
    import torch.distributed as dist

    from .api import context
    c = ctx or context(x_dev.device.index or 0)
    if float(ens.get("nstd", 0.2)) == 0.0:  # degenerate ensemble is plain EMD (emd.cpp:267), same on every rank
        import ctypes as C

        import torch

        from . import _native as N
        k_cap = 64
        imfs = torch.empty((k_cap, n), dtype=torch.float64, device=x_dev.device)
        res = torch.empty(n, dtype=torch.float64, device=x_dev.device)
        k = C.c_size_t()
        c.check(c.lib.semd_decompose_device(c.ptr, 0, C.c_void_p(x_dev.data_ptr()), n,
                                            C.byref(N.SiftCfg(cfg.get("sd_threshold", 0.2),
                                                              cfg.get("max_sift_iters", 300), cfg.get("max_imfs", 0))),
                                            None, C.c_void_p(imfs.data_ptr()), k_cap, C.byref(k),
                                            C.c_void_p(res.data_ptr())))
        return imfs[:k.value], res
    eng = GpuCeemdanShard(c, x_dev, n, cfg, ens)

    def asum(part):
        if world > 1:
            dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
        return part

    return sharded_ceemdan(int(ens.get("nr", 100)), rank, world, eng, asum, int(cfg.get("max_imfs", 0)))


# ------------------------------------------------------------- numpy reference driver (tests)

def finish_numpy(x: np.ndarray, sums: np.ndarray, K: int, nr: int):
    """emd.cpp:252-260 restated for the host-logic tests."""
    inv = 1.0 / float(nr)
    imfs = sums[:K] * inv
    residue = x.copy()
    for k in range(K):
        residue = residue - imfs[k]
    return imfs, residue
