"""signal_std (emd.cpp:209-217) of long signals: the parallel evaluation of the reference's two
SEQUENTIAL sums (csrc/semd_aux.cu, "binade-locked" integer accumulation).

The reference adds left to right; beta = nstd * std(x) seeds every realization, so the last bit
matters. The kernels replace the additions of a segment by one exact integer addition whenever
the running sum provably stays inside one binade, and add term by term otherwise. Every input
must give the reference's bits -- equal to the oracle and to the single-thread kernel (debug bit
32) -- whatever share of the segments takes which path: smooth sums (fast path), sums that
cross zero and powers of two all the time, inputs full of rounding ties (values on a coarse
grid), huge dynamic range, constant and tiny inputs.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def std_stats(c):
    buf = (C.c_uint64 * 3)()
    c.run("semd_std_stats", buf)
    return list(buf)  # slow segments of the mean pass, of the variance pass, segments per pass


def cases():
    r = np.random.default_rng(20260)
    n = 300_007
    t = np.arange(n) / 4096.0
    yield "normal+1", r.standard_normal(n) * 3 + 1
    yield "zero-mean", r.standard_normal(n)
    yield "sines", np.sin(2 * np.pi * 3.1 * t) + 0.4 * np.sin(2 * np.pi * 177.0 * t + 1) + r.normal(0, 0.05, n)
    yield "ties/256", np.round(r.standard_normal(n) * 256) / 256
    yield "ties/4+3", np.round(r.normal(3, 1, n) * 4) / 4
    yield "integers", r.integers(0, 256, n).astype(np.float64)
    yield "negative", -np.abs(r.standard_normal(n)) - 0.5
    yield "dynamic-range", r.standard_normal(n) * np.exp(r.normal(0, 12, n))
    yield "constant", np.full(n, 0.1)
    yield "tiny", r.standard_normal(n) * 1e-300
    yield "huge", r.standard_normal(n) * 1e300
    yield "zeros", np.zeros(n)
    yield "ramp", np.arange(n, dtype=np.float64) - n / 3
    yield "len=65536", r.standard_normal(65536) + 0.25
    yield "len=65537", r.standard_normal(65537) - 7
    yield "len=1000003", r.standard_normal(1_000_003) * 2 + 0.01


@pytest.mark.parametrize("name,x", list(cases()), ids=[n for n, _ in cases()])
def test_parallel_std_bit_exact(se, oracle, name, x):
    c = se.context()
    want = oracle.signal_std(x)
    c.run("semd_set_debug", 32)
    try:
        single = se.signal_std(x)
        assert std_stats(c)[2] == 0  # the single-thread kernel ran
    finally:
        c.run("semd_set_debug", 0)
    got = se.signal_std(x)
    st = std_stats(c)
    assert st[2] == (x.size + 511) // 512, st  # the parallel path ran
    assert single == want or (np.isnan(single) and np.isnan(want)), (single.hex(), want.hex())
    assert got == want or (np.isnan(got) and np.isnan(want)), (name, got.hex(), want.hex(), st)


def test_parallel_std_takes_the_fast_path(se, oracle):
    """On a C5-like signal (zero-mean sines + noise, serialized) few segments need the slow path."""
    from paper_2106_15319_b200 import workloads as W
    x = W.sine_variates(256, 4096)
    s = se.concatenate(x, 64)
    c = se.context()
    assert se.signal_std(s) == oracle.signal_std(s)
    slow0, slow1, nseg = std_stats(c)
    assert nseg == (s.size + 511) // 512
    assert slow0 <= 0.15 * nseg and slow1 <= 64, (slow0, slow1, nseg)


def test_parallel_std_inside_eemd(se, oracle):
    """beta through the parallel std gives the same ensemble as through the single-thread kernel."""
    r = np.random.default_rng(5)
    n = 70_001
    x = np.sin(np.arange(n) * 0.01) + 0.3 * r.standard_normal(n)
    c = se.context()
    a = se.decompose_full(x, "eemd", nr=3, max_imfs=4)
    c.run("semd_set_debug", 32)
    try:
        b = se.decompose_full(x, "eemd", nr=3, max_imfs=4)
    finally:
        c.run("semd_set_debug", 0)
    assert np.array_equal(a["imfs"], b["imfs"]) and np.array_equal(a["residue"], b["residue"])
