"""Speculative last sifts of the lockstep engine (semd_types.cuh ST_PRIMED / ST_REDETECT).

A sift that is likely its IMF's last also writes the residue R' = X - new (emd.cpp:167) and
detects R''s extrema instead of new's; when the SD test stops there, the next IMF starts from R'
without a DETECT pass and k_final only accumulates; when it does not, the candidate is detected
in an extra step. This only changes which detection runs when, so every result -- IMFs, residue,
sift counts, the parity trace -- must be bit-identical with speculation off (debug bit 8), on the
learned policy (default) and on every sift (debug bit 16), and equal to the oracle.
"""
import ctypes as C

import numpy as np
import pytest

from tests.conftest import sort_trace
from tests.golden.inputs import rng_signal

pytestmark = pytest.mark.gpu

MODES = {"off": 8, "default": 0, "every": 16}


def spec_stats(c):
    buf = (C.c_uint64 * 4)()
    c.run("semd_spec_stats", buf)
    return list(buf)  # run, stopped, continued, lockstep steps


def run_modes(se, x, algo, **kw):
    c = se.context()
    c.set_engine("lockstep")
    out = {}
    try:
        for name, bits in MODES.items():
            c.run("semd_set_debug", bits)
            spec_stats(c)
            d = se.decompose_full(x, algo, trace_cap=400000, **kw)
            d["spec"] = spec_stats(c)
            out[name] = d
    finally:
        c.run("semd_set_debug", 0)
        c.set_engine("auto")
    return out


def same(a, b):
    assert a["imfs"].shape == b["imfs"].shape
    assert np.array_equal(a["imfs"], b["imfs"]) and np.array_equal(a["residue"], b["residue"])
    assert np.array_equal(a["sift_counts"], b["sift_counts"])
    assert np.array_equal(sort_trace(a["trace"]), sort_trace(b["trace"]))


@pytest.mark.parametrize("n,max_imfs,iters", [(9001, 0, 300), (40961, 0, 300), (40961, 3, 300), (120_000, 0, 300),
                                              (20011, 0, 1), (20011, 0, 2), (20011, 2, 2)])
def test_emd_speculation_bit_exact(se, oracle, n, max_imfs, iters):
    x = rng_signal(500 + n, n) + 0.001 * np.arange(n)
    r = run_modes(se, x, "emd", max_imfs=max_imfs, max_sift_iters=iters)
    o = oracle.emd(x, imfs=max_imfs, iters=iters, trace_cap=400000)
    for name, d in r.items():
        assert np.array_equal(d["imfs"], o[0]) and np.array_equal(d["residue"], o[1]), name
        assert d["sift_counts"].tolist() == o[2].tolist(), name
        assert np.array_equal(sort_trace(d["trace"]), sort_trace(o[3])), name
    assert r["off"]["spec"][0] == 0
    if r["default"]["imfs"].shape[0] > 1:
        assert r["every"]["spec"][0] > 0 and r["every"]["spec"][1] > 0  # speculation ran and hit
    if iters == 1 and (max_imfs == 0 or max_imfs > 1):
        assert r["default"]["spec"][2] == 0  # the iteration cap stops every sift: never a miss


def test_eemd_speculation_bit_exact(se, oracle):
    x = rng_signal(4242, 30000)
    r = run_modes(se, x, "eemd", nr=12)
    same(r["off"], r["default"])
    same(r["off"], r["every"])
    o = oracle.decompose(x, 1, nr=12, trace_cap=400000)
    assert np.array_equal(sort_trace(r["default"]["trace"]), sort_trace(o[3]))
    for k in range(o[0].shape[0]):
        assert np.linalg.norm(r["default"]["imfs"][k] - o[0][k]) <= 1e-9 * np.linalg.norm(o[0][k])
    run, hit, miss, _ = r["every"]["spec"]
    assert run == hit + miss and hit > 0 and miss > 0  # both outcomes exercised
    run, hit, miss, _ = r["default"]["spec"]
    assert run == hit + miss and hit > 0


def test_ceemdan_and_plateaus_speculation(se):
    """CEEMDAN tasks are single-IMF jobs (no speculation); a quantised signal (many equal
    neighbours) runs the plateau path of the detections."""
    x = rng_signal(77, 12000)
    r = run_modes(se, x, "ceemdan", nr=4)
    same(r["off"], r["default"])
    same(r["off"], r["every"])
    y = np.round(rng_signal(78, 25000) * 4.0) / 4.0  # many exactly equal neighbours
    r = run_modes(se, y, "emd")
    same(r["off"], r["default"])
    same(r["off"], r["every"])


def test_speculation_statistics_persist_across_calls(se):
    """The policy's stop statistics live in the context (across waves and calls, halved per
    decomposition): a repeated decomposition mispredicts no more often than the first one, and its
    results do not depend on what the context has seen before."""
    x = rng_signal(9090, 60000)
    y = rng_signal(9191, 45000) * 3.0 + np.sin(np.arange(45000) * 0.002)
    c = se.context()
    c.set_engine("lockstep")
    try:
        spec_stats(c)
        a = se.decompose_full(x, "eemd", nr=6, trace_cap=400000)
        first = spec_stats(c)
        se.decompose_full(y, "eemd", nr=6)  # another input in between
        spec_stats(c)
        b = se.decompose_full(x, "eemd", nr=6, trace_cap=400000)
        again = spec_stats(c)
    finally:
        c.set_engine("auto")
    same(a, b)
    assert first[0] > 0 and again[0] > 0
    assert again[2] * first[0] <= first[2] * again[0] + again[0]  # miss rate did not grow (one miss of slack)
