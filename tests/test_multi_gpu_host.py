"""World-size-2 gloo tests of the multi-GPU host logic (realization sharding
+ ensemble all-reduce), with the oracle standing in for each rank's GPU
partial sums (the GPU partial is the same function on device memory)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2106_15319_b200.parallel import finish_numpy, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, x, nr, out_q):
    import torch
    import torch.distributed as dist

    from oracle.ffi import Oracle
    from paper_2106_15319_b200.parallel import sharded_ensemble

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()

    def partial(mb, me):
        sums, _ = o.eemd_partial(x, mb, me, nr=nr, imfs=0)
        return sums, sums.shape[0]

    def amax(k):
        t = torch.tensor([k], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return int(t.item())

    def asum(sums, K):
        pad = np.zeros((K, x.size))
        pad[:sums.shape[0]] = sums
        t = torch.from_numpy(pad)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.numpy()

    imfs, res = sharded_ensemble(nr, rank, world, partial, amax, asum, lambda s, K: finish_numpy(x, s, K, nr))
    out_q.put((rank, imfs, res))
    dist.destroy_process_group()


def test_shard_range_covers():
    for nr in (1, 7, 100, 1000):
        for w in (1, 2, 3, 4, 8):
            got = [shard_range(nr, r, w) for r in range(w)]
            cover = [m for b, e in got for m in range(b, e)]
            assert cover == list(range(nr))


@pytest.mark.parametrize("nr", [6, 9])
def test_sharded_eemd_world2(oracle, nr):
    from tests.golden.inputs import rng_signal
    x = rng_signal(77, 400)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, x, nr, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_imfs, ref_res, _, _ = oracle.decompose(x, 1, nr=nr)
    for _, imfs, r in res:
        assert imfs.shape == ref_imfs.shape  # same K on every rank
        rel = np.linalg.norm(imfs - ref_imfs) / np.linalg.norm(ref_imfs)
        assert rel <= 1e-12  # shard-order sums differ from the sequential order only by rounding
        assert np.max(np.abs(x - imfs.sum(0) - r)) <= 1e-12
    assert np.array_equal(res[0][1], res[1][1])  # every rank holds the identical result
