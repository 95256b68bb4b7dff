"""The exactness argument behind the parallel signal_std kernels (csrc/semd_aux.cu, k_seq_*), as a
pure-Python model checked on the CPU.

The reference adds left to right in fp64 (emd.cpp:209-217). While the running sum stays inside one
binade (same sign) every partial sum is S * u with u = 2^(e-52) and RN(s + v) = (S + rint(v/u)) * u,
a tie going to the even S -- so a segment is a function of the entry parity p -> (sum of k,
min prefix, max prefix), segments compose, and a segment may be applied as ONE integer addition when
the guessed binade equals the running sum's and entry + min/max stay inside [2^52+1, 2^53-1];
otherwise its terms are added one by one. This model mirrors the kernels' arithmetic (record(),
stitch) and must reproduce numpy's sequential cumsum bit for bit whatever the guesses are.
"""
import math
import struct

import numpy as np
import pytest

BIG = 1 << 61


def dec(s):
    b = struct.unpack("<q", struct.pack("<d", s))[0]
    return (b >> 63) & 1, (b >> 52) & 0x7FF, (b & ((1 << 52) - 1)) | (1 << 52)


def enc(sign, eb, S):
    return struct.unpack("<d", struct.pack("<Q", ((sign << 63) | (eb << 52) | (S - (1 << 52))) & ((1 << 64) - 1)))[0]


def record(v, sign, eb):
    """k_seq_records: the segment for the guessed (sign, exponent), per entry parity."""
    if eb < 60 or eb > 2040:
        return None
    scale = math.ldexp(1.0, 52 - (eb - 1023)) * (-1.0 if sign else 1.0)
    K, mn, mx = [0, 0], [BIG, BIG], [-BIG, -BIG]
    for x in v:
        t = float(x) * scale
        if not abs(t) < 2.0 ** 53:
            return None
        fl = math.floor(t)
        fr = t - fl
        for p in (0, 1):
            k = int(fl)
            if fr > 0.5:
                k += 1
            elif fr == 0.5:
                k += (p + K[p] + int(fl)) & 1
            K[p] += k
            mn[p] = min(mn[p], K[p])
            mx[p] = max(mx[p], K[p])
    return K, mn, mx


def seq_sum(v, seg, guess_bias=0.0):
    """k_seq_stitch over records built for guesses taken from approximate prefix sums."""
    n = len(v)
    segs = [v[i:i + seg] for i in range(0, n, seg)]
    approx = np.concatenate([[0.0], np.cumsum([float(np.sum(s)) for s in segs])[:-1]]) + guess_bias
    s, fast = 0.0, 0
    for c, part in enumerate(segs):
        gs, ge, _ = dec(float(approx[c]))
        r = record(part, gs, ge)
        sign, eb, S = dec(s)
        ok = r is not None and (sign, eb) == (gs, ge)
        if ok:
            K, mn, mx = r
            p = S & 1
            ok = S + mn[p] >= (1 << 52) + 1 and S + mx[p] <= (1 << 53) - 1
        if ok:
            s = enc(sign, eb, S + K[p])
            fast += 1
        else:
            for x in part:
                s = s + float(x)
    return s, fast


def inputs():
    r = np.random.default_rng(20260)
    n = 6000
    yield "normal+5", r.normal(5, 1, n)
    yield "zero-mean", r.normal(0, 1, n)
    yield "ties/256", np.round(r.normal(0, 1, n) * 256) / 256
    yield "ties/16+3", np.round(r.normal(3, 1, n) * 16) / 16
    yield "integers", r.integers(0, 256, n).astype(float)
    yield "sine+noise", np.sin(np.arange(n) * 0.01) + r.normal(0, 0.05, n)
    yield "negative", -np.abs(r.normal(0, 1, n)) - 0.5
    yield "dynamic-range", r.normal(0, 1, n) * np.exp(r.normal(0, 10, n))


@pytest.mark.parametrize("name,v", list(inputs()), ids=[n for n, _ in inputs()])
def test_binade_locked_sum_equals_sequential_sum(name, v):
    want = float(np.cumsum(v)[-1])  # numpy's cumsum adds left to right
    mean = want / len(v)
    w = (v - mean) * (v - mean)
    want2 = float(np.cumsum(w)[-1])
    for seg in (64, 512):
        got, fast = seq_sum(v, seg)
        assert got == want, (name, seg)
        got2, fast2 = seq_sum(w, seg)
        assert got2 == want2, (name, seg)
        if name in ("normal+5", "integers", "negative"):
            assert fast + fast2 > 0  # the integer path is actually exercised
    # wrong guesses only cost speed, never bits
    assert seq_sum(v, 64, guess_bias=1e3)[0] == want
