"""Realization sharding across GPUs.

CEEMDAN (emd.cpp:264-344) shards the same way but exchanges once per stage:
each rank sums the first modes of its realizations, one all-reduce(sum) of L
doubles forms the global stage sum, and every rank applies the identical
mode / residue update and stop tests (sharded_ceemdan).

EEMD realizations are independent units: rank r of W owns the contiguous
range shard_range(nr, r, W) and runs them on its own GPU (seeds derive from
the GLOBAL realization index, emd.cpp:238, so the work of realization m is
identical on any rank). The only exchange is the ensemble mean: an
all-reduce(max) of the IMF count and one reduce/all-reduce(sum) of the K x L
partial sums, followed by the finish (emd.cpp:252-260). No collective inside
the sift loop.

sharded_ensemble / sharded_ceemdan below are the host logic, written against
abstract collectives so the CPU tests can drive them with gloo (world size 2)
and the oracle. The GPU product runs the same logic inside the C engine
(semd_capi.cu, semd_comm_* in include/semd_b200.h) with NCCL on the engine
stream; init_comm joins a context to its communicator.
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


# ------------------------------------------------------------- GPU: NCCL inside the C ABI
#
# On GPUs the drivers above run inside the engine (semd_capi.cu decompose_device /
# ceemdan_device) once a context is joined to an NCCL communicator: the collectives are
# enqueued on the engine's own stream, so they are ordered with the kernels that produce and
# consume the sums. Python only ships the 128-byte NCCL unique id from rank 0 to the others.

def _rdzv_path() -> str:
    import os
    d = os.environ.get("SEMD_RDZV_DIR", "/tmp")
    # the launcher's ranks share a parent process (torchrun's agent): its pid keeps launches apart
    tag = os.environ.get("SEMD_RDZV_TAG") or f"{os.environ.get('TORCHELASTIC_RUN_ID', 'semd')}.{os.getppid()}"
    return os.path.join(d, f"semd_nccl_id.{tag}.{os.environ.get('MASTER_PORT', '0')}")


def init_comm(ctx, rank: int, world: int, root: int = -1, timeout: float = 300.0) -> None:
    """Join this rank's context to an NCCL communicator of `world` ranks (one process per GPU,
    one node). Rank 0 makes the unique id and publishes it through a file named after the
    launcher (run id, agent pid, master port); the others read it. No-op for world == 1."""
    import os
    import time
    if world <= 1:
        return
    path = _rdzv_path()
    if rank == 0:
        uid = ctx.comm_unique_id()
        tmp = f"{path}.{os.getpid()}.tmp"
        with open(tmp, "wb") as f:
            f.write(uid)
        os.replace(tmp, path)
    else:
        t0 = time.time()
        while True:
            try:
                with open(path, "rb") as f:
                    uid = f.read()
                if len(uid) == 128:
                    break
            except FileNotFoundError:
                pass
            if time.time() - t0 > timeout:
                raise TimeoutError(f"no NCCL unique id at {path}")
            time.sleep(0.02)
    ctx.comm_init(uid, rank, world, root)
    ctx.comm_allreduce([0.0])  # every rank has read the id
    if rank == 0:
        try:
            os.remove(path)
        except OSError:
            pass


# ------------------------------------------------------------- numpy reference driver (tests)

def finish_numpy(x: np.ndarray, sums: np.ndarray, K: int, nr: int):
    """emd.cpp:252-260 restated for the host-logic tests."""
    inv = 1.0 / float(nr)
    imfs = sums[:K] * inv
    residue = x.copy()
    for k in range(K):
        residue = residue - imfs[k]
    return imfs, residue
