"""Multi-GPU API inside the C ABI (semd_comm_*, NCCL on the engine stream).

One GPU is available on the test box, so the N > 1 exchange is covered two ways:
a 1-rank NCCL communicator must be bit-identical to the plain engine (the collectives
and the shard bookkeeping run, the reductions are identities), and the world-2 sharding
arithmetic is replayed on one GPU through the shard entry points (the same partial sums
the ranks would reduce). The host logic at world size 2 is in test_multi_gpu_host.py (gloo).
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sig(n=1500, seed=3):
    rng = np.random.default_rng(seed)
    t = np.arange(n)
    return np.sin(0.13 * t) + 0.5 * np.cos(0.021 * t) + 0.05 * rng.standard_normal(n)


def _decompose(ctx, algo, x, nr, max_imfs=0, k_cap=40):
    from paper_2106_15319_b200 import _native as N
    x = np.ascontiguousarray(x, dtype=np.float64)
    imfs = np.zeros((k_cap, x.size))
    res = np.zeros(x.size)
    k = C.c_size_t()
    ctx.run("semd_decompose", algo, x.ctypes.data_as(N._dp), x.size, C.byref(N.SiftCfg(0.2, 300, max_imfs)),
            C.byref(N.EnsCfg(0.2, nr, 0, 0)), imfs.ctypes.data_as(N._dp), k_cap, C.byref(k),
            res.ctypes.data_as(N._dp), None, None)
    return imfs[:k.value], res


def test_one_rank_comm_bit_identical(se):
    x = _sig()
    base = se.Context(0)
    ref = {a: _decompose(base, a, x, nr) for a, nr in ((1, 9), (2, 6))}
    c = se.Context(0)
    c.comm_init(se.Context.comm_unique_id(), 0, 1)
    assert c.comm_info() == (0, 1)
    for a, nr in ((1, 9), (2, 6)):
        imfs, res = _decompose(c, a, x, nr)
        assert np.array_equal(imfs, ref[a][0]) and np.array_equal(res, ref[a][1]), a
    c.run("semd_comm_set_root", 0)  # root-only reduction: rank 0 still holds the result
    imfs, res = _decompose(c, 1, x, 9)
    assert np.array_equal(imfs, ref[1][0]) and np.array_equal(res, ref[1][1])
    assert c.comm_allreduce([1.5, 2.0], "max").tolist() == [1.5, 2.0]
    c.comm_destroy()
    assert c.comm_info() == (0, 1)
    c.close()
    base.close()


def test_world2_shards_replayed_on_one_gpu(se):
    """What two ranks compute: shard_range(nr, r, 2) partial sums; their sum x 1/nr is the ensemble
    (equal to the single-GPU EEMD to rounding: the sum is formed in a different order)."""
    from paper_2106_15319_b200 import _native as N
    from paper_2106_15319_b200.parallel import shard_range
    x = _sig(1200, 5)
    nr, kc = 9, 32
    c = se.context(0)
    d_x = C.c_void_p()
    d_s = C.c_void_p()
    c.run("semd_device_alloc", x.nbytes, C.byref(d_x))
    c.run("semd_device_alloc", kc * x.nbytes, C.byref(d_s))
    c.run("semd_memcpy", d_x, x.ctypes.data_as(C.c_void_p), x.nbytes)
    parts, ks = [], []
    for r in range(2):
        mb, me = shard_range(nr, r, 2)
        k = C.c_size_t()
        c.run("semd_eemd_partial_device", d_x, x.size, C.byref(N.SiftCfg(0.2, 300, 0)), C.byref(N.EnsCfg(0.2, nr, 0, 0)),
              mb, me, d_s, kc, C.byref(k))
        h = np.zeros((kc, x.size))
        c.run("semd_memcpy", h.ctypes.data_as(C.c_void_p), d_s, h.nbytes)
        parts.append(h)
        ks.append(k.value)
    K = max(ks)
    imfs = (parts[0] + parts[1])[:K] * (1.0 / nr)
    ref = se.decompose(x, "eemd", nr=nr)
    assert imfs.shape == ref["imfs"].shape
    assert np.linalg.norm(imfs - ref["imfs"]) <= 1e-12 * np.linalg.norm(ref["imfs"])
    # zero-noise shards are rejected (emd.cpp:230: nstd == 0 is plain EMD)
    k = C.c_size_t()
    rc = c.call("semd_eemd_partial_device", d_x, x.size, None, C.byref(N.EnsCfg(0.0, nr, 0, 0)), 0, 2, d_s, kc,
                C.byref(k))
    assert rc == N.SEMD_INVALID_INPUT
    c.run("semd_device_free", d_x)
    c.run("semd_device_free", d_s)


def test_timer_and_device_memory(se):
    c = se.context(0)
    c.run("semd_timer_start")
    se.decompose(_sig(800), "eemd", nr=4)
    ms = C.c_double()
    c.run("semd_timer_stop", C.byref(ms))
    assert ms.value > 0.0
