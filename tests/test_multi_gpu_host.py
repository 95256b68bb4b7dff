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


# ------------------------------------------------------------------ CEEMDAN stage sharding

class OracleCeemdanShard:
    """sharded_ceemdan engine restated with the oracle's primitives (emd.cpp:264-344): the CPU
    stand-in for GpuCeemdanShard (same begin/stage/finish/residue_extrema/result contract)."""

    def __init__(self, o, x, nr, nstd=0.2, seed=0, sd=0.2, iters=300):
        self.o, self.x, self.nr, self.nstd, self.seed, self.sd, self.iters = o, x, nr, nstd, seed, sd, iters

    def _first_mode(self, s):
        from oracle.ffi import OracleError
        try:
            return self.o.extract_imf(s, sd=self.sd, iters=self.iters)[0]
        except OracleError:  # InsufficientExtrema -> zeros (emd.cpp:280-286)
            return np.zeros(self.x.size)

    def begin(self, mb, me):
        o, n = self.o, self.x.size
        self.ms = list(range(mb, me))
        self.noise = {m: o.white_noise(n, o.derive_seed(self.seed, m)) for m in self.ms}
        self.alive = {m: True for m in self.ms}
        self.residue = self.x.copy()
        self.modes = []
        self.beta0 = self.nstd * o.signal_std(self.x)

    def stage(self):
        from oracle.ffi import OracleError
        part = np.zeros(self.x.size)
        if not self.modes:
            for m in self.ms:
                part = part + self._first_mode(self.x + self.beta0 * self.noise[m])
            return part
        beta = self.nstd * self.o.signal_std(self.residue)
        for m in self.ms:
            ei = np.zeros(self.x.size)
            if self.alive[m]:
                try:
                    ei = self.o.extract_imf(self.noise[m], sd=self.sd, iters=self.iters)[0]
                    self.noise[m] = self.noise[m] - ei
                except OracleError:
                    self.alive[m] = False
            part = part + self._first_mode(self.residue + beta * ei)
        return part

    def finish(self, total, check_zero):
        mode = total * (1.0 / float(self.nr))
        if check_zero and not np.any(mode != 0.0):
            return False
        self.residue = self.residue - mode
        self.modes.append(mode)
        return True

    def residue_extrema(self):
        mi, _, ni, _ = self.o.find_extrema(self.residue)
        return len(mi) + len(ni)

    def result(self):
        return np.array(self.modes), self.residue


def _ceemdan_signal():
    t = np.arange(700) / 700.0
    return np.sin(2 * np.pi * 23 * t) + 0.6 * np.sin(2 * np.pi * 5 * t) + 0.3 * np.cos(2 * np.pi * 61 * t)


def test_sharded_ceemdan_world1_equals_oracle(oracle):
    from paper_2106_15319_b200.parallel import sharded_ceemdan
    x, nr = _ceemdan_signal(), 6
    imfs, res = sharded_ceemdan(nr, 0, 1, OracleCeemdanShard(oracle, x, nr), lambda p: p)
    o = oracle.decompose(x, 2, nr=nr)
    assert imfs.shape == o[0].shape
    assert np.array_equal(imfs, o[0]) and np.array_equal(res, o[1])


def _ceemdan_worker(rank, world, port, x, nr, out_q):
    import torch
    import torch.distributed as dist

    from oracle.ffi import Oracle
    from paper_2106_15319_b200.parallel import sharded_ceemdan

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def asum(part):
        t = torch.from_numpy(np.ascontiguousarray(part))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.numpy()

    imfs, res = sharded_ceemdan(nr, rank, world, OracleCeemdanShard(Oracle(), x, nr), asum)
    out_q.put((rank, imfs, res))
    dist.destroy_process_group()


def test_sharded_ceemdan_gloo_world2(oracle):
    x, nr, world = _ceemdan_signal(), 6, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ceemdan_worker, args=(r, world, port, x, nr, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict((r, (i, s)) for r, i, s in (q.get(timeout=300) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
    o = oracle.decompose(x, 2, nr=nr)
    for r in range(world):
        imfs, res = got[r]
        assert np.array_equal(imfs, got[0][0]) and np.array_equal(res, got[0][1])  # every rank identical
        assert imfs.shape == o[0].shape
        assert np.max(np.abs(imfs - o[0])) <= 1e-11 * np.max(np.abs(x))  # stage sums in a different tree


# ------------------------------------------------------------------ NCCL id rendezvous (bench / drivers)

def test_init_comm_rendezvous_world2(tmp_path, monkeypatch):
    """parallel.init_comm: rank 0 publishes the 128-byte NCCL id, the other ranks read the same
    bytes and every rank joins with its own rank (the C ABI is stood in for by a recorder)."""
    import threading

    from paper_2106_15319_b200.parallel import init_comm
    monkeypatch.setenv("SEMD_RDZV_DIR", str(tmp_path))
    monkeypatch.setenv("SEMD_RDZV_TAG", "t")
    monkeypatch.setenv("MASTER_PORT", "29555")
    uid = bytes(range(128))
    got = {}
    barrier = threading.Barrier(3)

    class FakeCtx:
        def __init__(self, rank):
            self.rank = rank

        @staticmethod
        def comm_unique_id():
            return uid

        def comm_init(self, u, rank, world, root):
            got[self.rank] = (u, rank, world, root)

        def comm_allreduce(self, vals, op="sum"):
            barrier.wait(timeout=30)

    ts = [threading.Thread(target=init_comm, args=(FakeCtx(r), r, 3, 0)) for r in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=60)
    assert got == {r: (uid, r, 3, 0) for r in range(3)}
    assert not list(tmp_path.iterdir())  # rank 0 removed the id file after everyone joined
