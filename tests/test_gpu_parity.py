"""Parity of the sm_100a engine (through the C ABI) against the oracle and the
reference's golden vectors. Bar: bit-exact for indices, counts, traces and
values (EMD, serializer, spline, the noise stream, and EEMD / CEEMDAN with the
device's own noise, which reproduces glibc's log/sincos bit-for-bit); per-IMF
rel-L2 <= 1e-9 is the north_star floor where a test compares across orders.
"""
import os
import subprocess

import numpy as np
import pytest

from tests.conftest import ROOT, fromhex, sha, sort_trace
from tests.golden.inputs import TestRng, rng_signal, sine

pytestmark = pytest.mark.gpu

REL_L2 = 1e-9  # north_star tolerance for fp64 IMFs


def pickup_serialized(se, D):
    from paper_2106_15319_b200 import workloads as W
    return se.concatenate(W.pickup_signals(), D)


def rel_l2(a, b):
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


def hazards(se):
    return se.context().stats()["solve_hazards"]


# ------------------------------------------------------------------ primitives

def test_rng_stream_bit_exact(se, oracle, golden):
    c = se.context()
    assert int(c.mt19937_64(5489, 10000)[-1]) == 9981545732273789042
    for seed in (oracle.derive_seed(0, 0), 7, 0, 2**64 - 1):
        assert np.array_equal(c.mt19937_64(seed, 4096), oracle.mt19937_64(seed, 4096))


def test_white_noise(se, oracle, golden):
    """emd.cpp:181-200 bit-for-bit: the device runs glibc's log and sincos restated (semd_libm.cuh)."""
    for n, seed in [(4, oracle.derive_seed(0, 0)), (1001, 7), (100000, 3), (1_000_001, oracle.derive_seed(0, 793))]:
        assert np.array_equal(se.white_noise(n, seed), oracle.white_noise(n, seed)), (n, seed)
    kat = golden["white_noise_1001_seed7"]
    assert sha(se.white_noise(1001, 7)) == kat["sha256"]
    assert [v.hex() for v in se.white_noise(4, oracle.derive_seed(0, 0))] == golden["white_noise_4_seed_ds00"]
    assert np.array_equal(se.white_noise(1001, 7, 0.37), oracle.white_noise(1001, 7, 0.37))
    assert abs(np.std(se.white_noise(100000, 3)) - 1.0) <= 0.02  # test_emd.cpp:224-227
    assert np.array_equal(se.white_noise(64, 5, 0.0), np.zeros(64))
    with pytest.raises(se.InvalidInput, match="white_noise: std must be non-negative"):
        se.white_noise(8, 0, -1.0)


def test_signal_std_bit_exact(se, oracle):
    for n in (1, 5, 6250, 100003, 2_000_001, 5_000_011):
        x = np.random.default_rng(n).standard_normal(n) * 3 + 1
        assert se.signal_std(x) == oracle.signal_std(x)


def test_find_extrema_golden(se, golden):
    for case in golden["find_extrema"]:
        x = fromhex(case["x"])
        mi, mv, ni, nv = se.find_extrema(x)
        assert mi.tolist() == case["max_idx"], case["name"]
        assert ni.tolist() == case["min_idx"], case["name"]
        assert np.array_equal(mv, fromhex(case["max_val"])) and np.array_equal(nv, fromhex(case["min_val"]))
    with pytest.raises(se.InvalidInput, match="find_extrema: signal too short"):
        se.find_extrema([1.0, 2.0])


def test_find_extrema_random_and_plateaus(se, oracle):
    rng = np.random.default_rng(1)
    for trial in range(40):
        n = int(rng.integers(3, 9000))
        x = rng.integers(-2, 3, size=n).astype(float) if trial % 2 else rng.standard_normal(n)
        a, b = se.find_extrema(x), oracle.find_extrema(x)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)
    # a plateau run crossing many eval tiles (2048 samples each)
    x = np.concatenate([np.zeros(10), np.ones(5000), np.zeros(3000), -np.ones(7001), np.zeros(3)])
    for u, v in zip(se.find_extrema(x), oracle.find_extrema(x)):
        assert np.array_equal(u, v)


def test_envelope_golden_and_random(se, oracle, golden):
    for case in golden["envelope"]:
        out = se.envelope(case["idx"], fromhex(case["val"]), case["length"])
        assert np.array_equal(out, fromhex(case["out"])), case["name"]
    rng = np.random.default_rng(2)
    for _ in range(30):
        length = int(rng.integers(5, 3000))
        k = int(rng.integers(2, min(200, length)))
        idx = np.sort(rng.choice(length, size=k, replace=False))
        val = rng.standard_normal(k)
        assert np.array_equal(se.envelope(idx, val, length), oracle.envelope(idx, val, length))
    with pytest.raises(se.InsufficientExtrema, match="envelope: need at least 2 extrema, got 1"):
        se.envelope([4], [1.0], 10)


# ------------------------------------------------------------------ sifting

def test_extract_imf(se, oracle):
    from oracle.ffi import OracleError
    for seed, n, iters in [(11, 600, 300), (5, 5000, 3), (9, 20000, 300), (3, 7, 300), (8, 12, 300)]:
        x = rng_signal(seed, n)
        try:
            oimf, ocnt = oracle.extract_imf(x, iters=iters)
        except OracleError as e:
            with pytest.raises(se.InvalidInput) as g:
                se.extract_imf(x, max_sift_iters=iters)
            assert str(g.value) == str(e)
            continue
        imf, cnt = se.extract_imf(x, max_sift_iters=iters)
        assert cnt == ocnt and np.array_equal(imf, oimf)
    x = sine(8.0, 1000, 1000.0)
    imf, _ = se.extract_imf(x)
    assert np.corrcoef(imf, x)[0, 1] >= 0.99  # test_emd.cpp:114-118
    with pytest.raises(se.InsufficientExtrema):
        se.extract_imf(np.arange(50.0))
    imf, cnt = se.extract_imf(rng_signal(4, 100), max_sift_iters=0)
    assert cnt == 0 and np.array_equal(imf, rng_signal(4, 100))


def test_emd_golden_random(se, golden):
    for case in golden["emd_random"]:
        x = rng_signal(case["seed"], case["n"])
        if case["n"] < 4:
            continue
        d = se.decompose_full(x, "emd", max_imfs=case["max_imfs"], trace_cap=100000)
        assert d["imfs"].shape[0] == case["K"]
        assert d["sift_counts"].tolist() == case["counts"]
        assert sha(d["imfs"]) == case["imfs_sha256"] and sha(d["residue"]) == case["residue_sha256"]
        got = [[int(t[k]) for k in ("k", "iter", "n_max", "n_min", "hash")] for t in sort_trace(d["trace"])]
        assert got == case["trace"]
    assert hazards(se) == 0


@pytest.mark.parametrize("n", [4, 5, 17, 2047, 2048, 2049, 6001, 40961, 250_000])
def test_emd_bit_exact_lengths(se, oracle, n):
    x = rng_signal(1000 + n, n) + 0.001 * np.arange(n)
    d = se.decompose_full(x, "emd", trace_cap=200000)
    o = oracle.emd(x, trace_cap=200000)
    assert d["imfs"].shape == o[0].shape
    assert np.array_equal(d["imfs"], o[0]) and np.array_equal(d["residue"], o[1])
    assert d["sift_counts"].tolist() == o[2].tolist()
    assert np.array_equal(sort_trace(d["trace"]), sort_trace(o[3]))
    assert hazards(se) == 0


def test_solve_repair_path_bit_exact(se, oracle):
    """Force the speculative-solve repair (exact sequential Thomas) on every multi-block envelope."""
    ctx = se.context()
    x = rng_signal(77, 120_000) + 0.001 * np.arange(120_000)
    ctx.lib.semd_set_debug(ctx.ptr, 1)
    try:
        d = se.decompose_full(x, "emd", trace_cap=200000)
        st = ctx.stats()
    finally:
        ctx.lib.semd_set_debug(ctx.ptr, 0)
    o = oracle.emd(x, trace_cap=200000)
    assert st["solve_hazards"] > 0  # the repair ran
    assert np.array_equal(d["imfs"], o[0]) and np.array_equal(d["residue"], o[1])
    assert np.array_equal(sort_trace(d["trace"]), sort_trace(o[3]))


def test_emd_edge_cases(se, oracle):
    ramp = 0.25 * np.arange(64)
    d = se.decompose(ramp)
    assert d["imfs"].shape[0] == 0 and np.array_equal(d["residue"], ramp)  # test_emd.cpp:144-150
    with pytest.raises(se.InvalidInput, match="emd: signal too short"):
        se.decompose([1.0, 2.0, 1.0])
    x = rng_signal(12, 500)
    d = se.decompose(x, max_imfs=2)
    assert d["imfs"].shape[0] == 2
    assert np.max(np.abs(d["imfs"].sum(0) + d["residue"] - x)) <= 1e-8
    const = np.full(100, 3.5)
    assert se.decompose(const)["imfs"].shape[0] == 0
    # clipped / plateau-rich input (exact equality runs)
    y = np.clip(np.round(4 * np.sin(np.arange(3000) * 0.01) + rng_signal(3, 3000)), -3, 3)
    d, o = se.decompose_full(y, "emd", trace_cap=100000), oracle.emd(y, trace_cap=100000)
    assert np.array_equal(d["imfs"], o[0]) and np.array_equal(d["residue"], o[1])


def test_c1_serial_emd(se, golden, golden_traces):
    c = golden["configs"]["c1_emd_D50"]
    s = pickup_serialized(se, 50)
    assert sha(s) == c["input_sha256"]
    d = se.decompose_full(s, "emd", max_sift_iters=1000, trace_cap=10000)
    assert d["imfs"].shape[0] == 6 and d["sift_counts"].tolist() == c["counts"] == [2, 2, 2, 2, 1, 1]
    assert sha(d["imfs"]) == c["imfs_sha256"] and sha(d["residue"]) == c["residue_sha256"]
    assert np.array_equal(sort_trace(d["trace"]), sort_trace(golden_traces["c1_emd_D50"]))
    assert d["stats"]["sifted_samples"] == c["sifted_samples"] == 62_500


# ------------------------------------------------------------------ ensembles

@pytest.mark.parametrize("name", ["c2_eemd_D1", "c2_eemd_D50", "c2_eemd_D500"])
def test_c2_eemd(se, oracle, golden, golden_traces, name):
    c = golden["configs"][name]
    s = pickup_serialized(se, c["D"])
    d = se.decompose_full(s, "eemd", max_imfs=c["imfs"], nr=c["nr"], trace_cap=100000)
    o_imfs, o_res, _, _ = oracle.decompose(s, 1, imfs=c["imfs"], nr=c["nr"])
    assert d["imfs"].shape == o_imfs.shape and d["imfs"].shape[0] == c["K"]
    assert np.array_equal(sort_trace(d["trace"]), sort_trace(golden_traces[name]))  # extrema + sift counts
    for k in range(c["K"]):
        assert rel_l2(d["imfs"][k], o_imfs[k]) <= REL_L2
    assert rel_l2(d["residue"], o_res) <= REL_L2
    assert d["stats"]["sifted_samples"] == c["sifted_samples"]
    # with the reference's own noise injected, the whole ensemble is bit-exact
    ctx = se.context()
    ctx.set_noise_override(np.stack([oracle.white_noise(s.size, oracle.derive_seed(0, m)) for m in range(c["nr"])]))
    try:
        e = se.decompose(s, "eemd", max_imfs=c["imfs"], nr=c["nr"])
    finally:
        ctx.set_noise_override(None)
    assert sha(e["imfs"]) == c["imfs_sha256"] and sha(e["residue"]) == c["residue_sha256"]
    assert hazards(se) == 0


def test_c3_ceemdan(se, oracle, golden, golden_traces):
    c = golden["configs"]["c3_ceemdan_D50"]
    s = pickup_serialized(se, 50)
    d = se.decompose_full(s, "ceemdan", max_sift_iters=5000, nr=500, trace_cap=100000)
    assert d["imfs"].shape[0] == c["K"] == 9
    assert np.array_equal(sort_trace(d["trace"]), sort_trace(golden_traces["c3_ceemdan_D50"]))
    o_imfs, o_res, _, _ = oracle.decompose(s, 2, iters=5000, nr=500)
    for k in range(9):
        assert rel_l2(d["imfs"][k], o_imfs[k]) <= REL_L2
    ctx = se.context()
    ctx.set_noise_override(np.stack([oracle.white_noise(s.size, oracle.derive_seed(0, m)) for m in range(500)]))
    try:
        e = se.decompose(s, "ceemdan", max_sift_iters=5000, nr=500)
    finally:
        ctx.set_noise_override(None)
    assert sha(e["imfs"]) == c["imfs_sha256"] and sha(e["residue"]) == c["residue_sha256"]


def test_small_ensembles_golden(se, oracle, golden):
    ctx = se.context()
    for case in golden["ensembles_small"]:
        x = rng_signal(case["seed"], case["n"])
        ctx.set_noise_override(np.stack([oracle.white_noise(x.size, oracle.derive_seed(0, m))
                                         for m in range(case["nr"])]))
        try:
            d = se.decompose(x, ["emd", "eemd", "ceemdan"][case["algo"]], nr=case["nr"])
        finally:
            ctx.set_noise_override(None)
        assert sha(d["imfs"]) == case["imfs_sha256"] and sha(d["residue"]) == case["residue_sha256"]


def test_ensemble_properties(se):
    x = rng_signal(22, 300)
    a, b = se.eemd(x, nr=10), se.eemd(x, nr=10)
    assert np.array_equal(a["imfs"], b["imfs"]) and np.array_equal(a["residue"], b["residue"])  # deterministic
    assert np.max(np.abs(a["imfs"].sum(0) + a["residue"] - x)) <= 1e-8 * np.max(np.abs(x))
    c1, c2 = se.ceemdan(x, nr=8), se.ceemdan(x, nr=8)
    assert np.array_equal(c1["imfs"], c2["imfs"])
    assert np.max(np.abs(c1["imfs"].sum(0) + c1["residue"] - x)) <= 1e-8 * np.max(np.abs(x))
    # nstd = 0 degenerates to plain emd exactly (acceptance criterion 9)
    e = se.emd(x)
    for algo in ("eemd", "ceemdan"):
        d = se.decompose(x, algo, nstd=0.0, nr=3)
        assert np.array_equal(d["imfs"], e["imfs"]) and np.array_equal(d["residue"], e["residue"])
    with pytest.raises(se.InvalidInput, match="ensemble: nr must be at least 1"):
        se.eemd(x, nr=0)
    with pytest.raises(se.InvalidInput, match="ensemble: nstd must be non-negative"):
        se.ceemdan(x, nstd=-1.0)
    with pytest.raises(se.InvalidInput, match="ceemdan: signal too short"):
        se.ceemdan([1.0, 2.0, 3.0])


# ------------------------------------------------------------------ serializer

def test_concatenate_sweep(se, oracle):
    g = TestRng(34)
    for _ in range(120):
        m, n = g.range(4, 60), g.range(1, 8)
        d = g.range(1, m)
        x = np.array([g.uniform() for _ in range(m * n)]).reshape(n, m)  # channel rows
        ms = np.ascontiguousarray(x.T)  # (M, N) samples x channels
        a = se.concatenate(ms, d)
        assert np.array_equal(a, oracle.concatenate(x, m, n, d))
        assert np.array_equal(se.concatenate_naive(ms, d), a)
    with pytest.raises(se.InvalidInput, match="concatenate: transition longer than channel"):
        se.concatenate(np.ones((10, 2)), 11)
    with pytest.raises(se.InvalidInput, match="concatenate: D must be at least 1"):
        se.concatenate(np.ones((10, 2)), 0)
    assert np.array_equal(se.transition_weights(4), [0.2, 0.4, 0.6, 0.8])
    assert se.default_transition_length(1000) == 200


def test_deconcatenate_and_serial(se, oracle):
    m, n, d = 10, 3, 4
    mode = np.zeros(m * n + d * (n - 1))
    for j in range(n - 1):
        mode[j * (m + d) + m: j * (m + d) + m + d] = 999.0  # poisoned transitions never leak
    t = se.deconcatenate(mode[:, None], m, n, d)
    assert t.shape == (m, n, 1) and np.all(t == 0.0)
    with pytest.raises(se.InvalidInput, match="deconcatenate: mode length 11 does not match"):
        se.deconcatenate(np.zeros((11, 1)), 10, 1, 2)
    x6 = oracle.multivariate_sinusoids()
    t, _ = se.serial_decompose_full(np.ascontiguousarray(x6.T), 50, "emd")
    o, _ = oracle.serial_decompose(x6, 1000, 6, 50, 0)
    assert np.array_equal(t, o.transpose(2, 1, 0))
    assert np.max(np.abs(t.sum(axis=2) - x6.T)) <= 1e-8 * np.max(np.abs(x6))
    te = se.serial_decompose(np.ascontiguousarray(x6.T), 50, "eemd", nr=8)
    assert np.max(np.abs(te.sum(axis=2) - x6.T)) <= 1e-8 * np.max(np.abs(x6))


def _slicewise_expected(per):
    """baseline.cpp:17-27 assembly of per-channel decompositions -> (M, N, K) tensor."""
    common = max(1, max(d[0].shape[0] + 1 for d in per))
    M = per[0][1].size
    t = np.zeros((M, len(per), common))
    for j, (imfs, res) in enumerate(per):
        if imfs.shape[0]:
            t[:, j, :imfs.shape[0]] = imfs.T
        t[:, j, common - 1] = res
    return t


def test_slicewise(se, oracle):
    rng = np.random.default_rng(11)
    x = rng.standard_normal((300, 5)) + np.sin(np.arange(300) / 9.0)[:, None]
    x[:, 4] = np.arange(300) * 0.1  # monotone channel: no IMFs, residue = x
    t = se.slicewise_decompose(x)
    per = [oracle.emd(x[:, j])[:2] for j in range(x.shape[1])]
    assert np.array_equal(t, _slicewise_expected(per))  # batched EMD == reference per channel, bit-exact
    assert np.max(np.abs(t.sum(axis=2) - x)) <= 1e-10 * np.max(np.abs(x))
    with pytest.raises(se.InvalidInput, match="slicewise_decompose: empty input"):
        se.slicewise_decompose(np.zeros((0, 3)))


def test_slicewise_ensembles(se, oracle):
    """baseline.cpp:5-29: slicewise EEMD (every channel x realization in one batched engine pass) and
    channel-by-channel CEEMDAN equal the oracle's decompose() of each channel bit-for-bit (the same
    seeds per realization, the same realization-ordered sums), and the per-channel GPU calls."""
    rng = np.random.default_rng(12)
    x = rng.standard_normal((256, 4)) + np.cos(np.arange(256) / 7.0)[:, None]
    for algo, code, nr in (("eemd", 1, 6), ("ceemdan", 2, 5)):
        t = se.slicewise_decompose(x, algo, nr=nr)
        ref = [oracle.decompose(np.ascontiguousarray(x[:, j]), code, nr=nr)[:2] for j in range(x.shape[1])]
        assert np.array_equal(t, _slicewise_expected(ref)), algo
        per = []
        for j in range(x.shape[1]):
            d = se.decompose(x[:, j], algo, nr=nr)
            per.append((d["imfs"], d["residue"]))
        assert np.array_equal(t, _slicewise_expected(per)), algo


# ------------------------------------------------------------------ full-size properties

def _c4_serialized(se):
    from paper_2106_15319_b200 import workloads as W
    return se.concatenate(W.image_batch(), 10)


@pytest.mark.slow
def test_c4_one_realization_bit_exact(se, oracle):
    s = _c4_serialized(se)
    assert s.size == 2_924_534
    ctx = se.context()
    ctx.set_noise_override(oracle.white_noise(s.size, oracle.derive_seed(0, 0))[None, :])
    try:
        d = se.decompose_full(s, "eemd", nr=1, trace_cap=2000)
    finally:
        ctx.set_noise_override(None)
    o = oracle.decompose(s, 1, nr=1, trace_cap=2000)
    assert np.array_equal(d["imfs"], o[0]) and np.array_equal(d["residue"], o[1])
    assert np.array_equal(sort_trace(d["trace"]), sort_trace(o[3]))
    assert hazards(se) == 0


@pytest.mark.slow
def test_c4_full_ensemble_properties(se):
    s = _c4_serialized(se)
    a = se.decompose_full(s, "eemd", nr=100)
    assert np.max(np.abs(a["imfs"].sum(0) + a["residue"] - s)) <= 1e-8 * np.max(np.abs(s))
    b = se.decompose(s, "eemd", nr=100)
    assert np.array_equal(a["imfs"], b["imfs"])  # bit-reproducible run to run
    assert a["stats"]["solve_hazards"] == 0


@pytest.mark.slow
def test_c5_realizations(se, oracle):
    from paper_2106_15319_b200 import workloads as W
    s = se.concatenate(W.sine_variates(), 64)
    assert s.size == 17_039_296
    d = se.decompose_full(s, "eemd", nr=2, trace_cap=4000)
    assert np.max(np.abs(d["imfs"].sum(0) + d["residue"] - s)) <= 1e-8 * np.max(np.abs(s))
    assert d["stats"]["solve_hazards"] == 0
    # realization-level trace parity for one realization against the oracle
    # (the oracle runs the same x + beta*w_0 with the device noise injected)
    ctx = se.context()
    w0 = se.white_noise(s.size, oracle.derive_seed(0, 0))
    ctx.set_noise_override(w0[None, :])
    try:
        g = se.decompose_full(s, "eemd", nr=1, trace_cap=4000)
    finally:
        ctx.set_noise_override(None)
    beta = 0.2 * se.signal_std(s)
    o = oracle.emd(s + beta * w0, trace_cap=4000)
    assert np.array_equal(sort_trace(g["trace"]), sort_trace(o[3]))
    for k in range(o[0].shape[0]):
        assert rel_l2(g["imfs"][k], o[0][k]) <= REL_L2


def test_unbounded_imf_loop(se, oracle):
    """The reference's IMF loop (emd.cpp:160-169) is unbounded when max_imfs == 0; on a near-constant
    signal with ulp-level wiggles every residue keeps extrema and it never terminates. With a cap the
    engine matches the oracle bit-for-bit; without one it fails with a capacity error (after growing
    its IMF store) instead of hanging."""
    x = 1.0 + np.spacing(1.0) * np.random.default_rng(0).integers(0, 3, 500)
    d = se.decompose_full(x, "emd", max_imfs=40, trace_cap=100000)
    o = oracle.emd(x, imfs=40, trace_cap=100000)
    assert d["imfs"].shape[0] == o[0].shape[0] == 40
    assert np.array_equal(d["imfs"], o[0]) and np.array_equal(d["residue"], o[1])
    assert d["sift_counts"].tolist() == o[2].tolist()
    assert np.array_equal(sort_trace(d["trace"]), sort_trace(o[3]))
    with pytest.raises(Exception, match="IMF capacity"):
        se.decompose(x)
    with pytest.raises(Exception, match="IMF capacity"):
        se.decompose(x, "eemd", nr=3)


def test_c5_realization_793(se, oracle):
    """C5 realization 793 with the device noise stream ran away when beta came from a parallel
    (non-sequential) std; with the reference's sequential std it ends at K=16 like its neighbours."""
    import ctypes as C

    import torch

    from paper_2106_15319_b200 import _native as N
    from paper_2106_15319_b200 import workloads as W
    s = se.concatenate(W.sine_variates(), 64)
    assert se.signal_std(s) == oracle.signal_std(s)
    ctx = se.context()
    sd = torch.from_numpy(s).cuda()
    sums = torch.zeros((32, s.size), dtype=torch.float64, device="cuda")
    k = C.c_size_t()
    ctx.check(ctx.lib.semd_eemd_partial_device(ctx.ptr, C.c_void_p(sd.data_ptr()), s.size,
                                               C.byref(N.SiftCfg(0.2, 300, 0)), C.byref(N.EnsCfg(0.2, 1000, 0, 0)),
                                               793, 794, C.c_void_p(sums.data_ptr()), 32, C.byref(k)))
    assert k.value == 16
    w = se.white_noise(s.size, oracle.derive_seed(0, 793))
    o = oracle.emd(s + 0.2 * oracle.signal_std(s) * w)
    assert o[0].shape[0] == 16
    for i in range(16):
        assert rel_l2(sums[i].cpu().numpy(), o[0][i]) <= REL_L2


def test_cpp_mirror_runs(se):
    from paper_2106_15319_b200 import _native
    exe = "/tmp/test_semd_cpp"
    src = os.path.join(ROOT, "tests", "cpp", "test_semd_cpp.cpp")
    libdir = os.path.dirname(_native.LIB_PATH)
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"), src, "-o", exe,
                        "-L" + libdir, "-lsemd_b200", "-Wl,-rpath," + libdir], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().splitlines()[-1].startswith("OK"), r.stdout


class _GpuCeemdanShard:
    """parallel.sharded_ceemdan's engine contract over the C ABI stage entry points
    (semd_ceemdan_shard_*), with torch CUDA tensors as the device buffers (test harness)."""

    def __init__(self, ctx, x_dev, n, nr):
        import ctypes as C

        from paper_2106_15319_b200 import _native as N
        self.C, self.c, self.x, self.n, self.nr = C, ctx, x_dev, n, nr
        self.scfg, self.ecfg = N.SiftCfg(0.2, 300, 0), N.EnsCfg(0.2, nr, 0, 0)
        self.modes = []

    def begin(self, mb, me):
        C = self.C
        self.c.run("semd_ceemdan_shard_begin", C.c_void_p(self.x.data_ptr()), self.n, C.byref(self.scfg),
                   C.byref(self.ecfg), mb, me)

    def stage(self):
        import torch
        part = torch.empty(self.n, dtype=torch.float64, device=self.x.device)
        self.c.run("semd_ceemdan_shard_stage", self.C.c_void_p(part.data_ptr()))
        return part

    def finish(self, total, check_zero):
        import torch
        C = self.C
        mode = torch.empty(self.n, dtype=torch.float64, device=self.x.device)
        ok = C.c_int32()
        self.c.run("semd_ceemdan_shard_finish_stage", C.c_void_p(total.data_ptr()), self.nr, int(check_zero),
                   C.c_void_p(mode.data_ptr()), C.byref(ok))
        if ok.value:
            self.modes.append(mode)
        return bool(ok.value)

    def residue_extrema(self):
        t = self.C.c_size_t()
        self.c.run("semd_ceemdan_shard_residue_extrema", self.C.byref(t))
        return int(t.value)

    def result(self):
        import torch
        res = torch.empty(self.n, dtype=torch.float64, device=self.x.device)
        self.c.run("semd_ceemdan_shard_residue", self.C.c_void_p(res.data_ptr()))
        return torch.stack(self.modes), res


def test_ceemdan_stage_api_matches_monolithic(se, oracle):
    """The per-stage CEEMDAN API driven by parallel.sharded_ceemdan (world 1) is the monolithic
    CEEMDAN bit-for-bit, and both are the oracle's CEEMDAN bit-for-bit (same noise: the device's
    Box-Muller reproduces glibc's)."""
    import torch

    from paper_2106_15319_b200.parallel import sharded_ceemdan
    x = pickup_serialized(se, 50)[:3000].copy()
    nr = 24
    ctx = se.context()
    mono = se.decompose(x, "ceemdan", nr=nr)
    xd = torch.from_numpy(x).cuda()
    imfs, res = sharded_ceemdan(nr, 0, 1, _GpuCeemdanShard(ctx, xd, x.size, nr), lambda p: p)
    o = oracle.decompose(x, 2, nr=nr)
    assert np.array_equal(imfs.cpu().numpy(), mono["imfs"]) and np.array_equal(res.cpu().numpy(), mono["residue"])
    assert np.array_equal(mono["imfs"], o[0]) and np.array_equal(mono["residue"], o[1])


def test_reconstruction_all_algorithms_and_pipelines(se):
    """Acceptance criterion 1's shape (acceptance.cpp:74-116): every algorithm (EMD, EEMD,
    CEEMDAN) through every pipeline (direct, serial, slicewise) reconstructs its input to 1e-8
    (relative to max |x|), on seeded noisy multi-tone inputs of varying length and channel count."""
    rng = np.random.default_rng(2106)
    algos = ("emd", "eemd", "ceemdan")
    for i in range(27):
        n = 80 + (i * 13) % 180
        algo = algos[i % 3]
        pipeline = (i // 3) % 3  # 0 direct, 1 serial, 2 slicewise
        kw = {} if algo == "emd" else {"nr": 6, "seed": 5000 + i}
        if pipeline == 0:
            x = rng.standard_normal(n) + np.sin(np.arange(n) * rng.uniform(0.05, 0.5))
            d = se.decompose(x, algo, **kw)
            rec = d["imfs"].sum(0) + d["residue"]
            err = np.max(np.abs(rec - x)) / np.max(np.abs(x))
        else:
            ch = 1 + i % 4
            t = np.arange(n)[:, None]
            x = rng.standard_normal((n, ch)) + np.sin(t * rng.uniform(0.05, 0.5, size=ch)[None, :])
            dd = max(1, n // 5)
            tens = se.serial_decompose(x, dd, algo, **kw) if pipeline == 1 else se.slicewise_decompose(x, algo, **kw)
            err = np.max(np.abs(tens.sum(axis=2) - x)) / np.max(np.abs(x))
        assert err <= 1e-8, (i, algo, pipeline, n, err)


def test_frequency_recovery_and_serial_vs_slicewise(se, oracle):
    """Acceptance criteria 4 and 5 (acceptance.cpp:179-220) on the pick-up signals (BASELINE
    configs 1-3: 6 variates x 1000 samples, 32/16/8/2 Hz by the mask): serial EMD with D=50 puts
    32 Hz in IMF1 of every 32 Hz variate and the common 8 Hz tone in some IMF of every variate;
    serial and slicewise IMF1 / IMF2 correlate per variate at r >= 0.9 / 0.7."""
    x6 = np.ascontiguousarray(oracle.multivariate_sinusoids().T)  # (1000 samples, 6 variates)
    mask32 = [1, 1, 0, 1, 0, 0]  # row 0 of the pick-up mask (32 Hz)
    serial = se.serial_decompose(x6, 50, "emd")
    sliced = se.slicewise_decompose(x6, "emd")

    def dominant(sig):  # Hz at fs = 1000, n = 1000 (1 Hz bins)
        mag = np.abs(np.fft.rfft(sig))
        mag[0] = 0.0
        return float(np.argmax(mag))

    for j in range(6):
        if mask32[j]:
            assert abs(dominant(serial[:, j, 0]) - 32.0) <= 1.0, j
        assert any(abs(dominant(serial[:, j, k]) - 8.0) <= 1.0 for k in range(serial.shape[2] - 1)), j
    for k, need in ((0, 0.9), (1, 0.7)):
        for j in range(6):
            r = np.corrcoef(serial[:, j, k], sliced[:, j, k])[0, 1]
            assert r >= need, (k, j, r)


def test_ceemdan_residue_extrema_count(se, oracle):
    """CEEMDAN's residue test (emd.cpp:311) counts find_extrema's maxima + minima with one kernel
    when untraced: equal to the oracle's find_extrema on plateau-rich and smooth signals."""
    import torch

    ctx = se.context()
    rng = np.random.default_rng(7)
    cases = [rng.integers(-2, 3, size=int(rng.integers(4, 9000))).astype(float) for _ in range(6)]
    cases += [rng.standard_normal(int(rng.integers(4, 9000))) for _ in range(4)]
    cases += [np.concatenate([np.zeros(10), np.ones(5000), np.zeros(3000), -np.ones(7001), np.zeros(3)]),
              np.array([1.0, 1.0, 1.0, 1.0]), np.array([0.0, 1.0, 1.0, 0.0, 2.0, 2.0, 2.0])]
    for x in cases:
        eng = _GpuCeemdanShard(ctx, torch.from_numpy(x).cuda(), x.size, 2)
        eng.begin(0, 2)  # the shard's residue starts as x
        max_idx, _, min_idx, _ = oracle.find_extrema(x)
        assert eng.residue_extrema() == len(max_idx) + len(min_idx)


def test_eemd_shards_sum_to_whole(se):
    """Realization sharding (the multi-GPU split) on one GPU: the partial sums of
    [0, m) and [m, nr) add up to the partial sums of [0, nr), and K is the max of the shards' K."""
    import ctypes as C

    import torch

    from paper_2106_15319_b200 import _native as N
    x = pickup_serialized(se, 50)
    n, nr = x.size, 12
    ctx = se.context()
    xd = torch.from_numpy(x).cuda()

    def part(mb, me):
        sums = torch.zeros((32, n), dtype=torch.float64, device="cuda")
        k = C.c_size_t()
        ctx.check(ctx.lib.semd_eemd_partial_device(ctx.ptr, C.c_void_p(xd.data_ptr()), n,
                                                   C.byref(N.SiftCfg(0.2, 300, 10)), C.byref(N.EnsCfg(0.2, nr, 0, 0)),
                                                   mb, me, C.c_void_p(sums.data_ptr()), 32, C.byref(k)))
        return sums.cpu().numpy(), int(k.value)

    whole, kw = part(0, nr)
    a, ka = part(0, 5)
    b, kb = part(5, nr)
    assert kw == max(ka, kb)
    assert np.max(np.abs((a + b) - whole)) <= 1e-12 * np.max(np.abs(whole))


def test_sd_stop_adversarial_thresholds(se, oracle):
    """The SD stop test (emd.cpp:150) at thresholds equal to, and one ulp above, the reference's
    own num/den of a sift: the engine's tree-summed ratio can differ from the reference's
    sequential one in the last bits, so these decisions are uncertifiable and must be redone with
    the reference's sequential sums (semd_stats.sd_rechecks counts them). Sift counts and IMFs
    must equal the oracle's at every such threshold."""
    rng = np.random.default_rng(150)
    c = se.context()
    rechecks = 0
    for n in (700, 3001, 200_003):
        t = np.arange(n)
        x = np.sin(0.07 * t) + 0.5 * np.sin(0.011 * t + 1.0) + 0.3 * rng.standard_normal(n)
        _, cnt, ratios = oracle.sd_ratios(x)
        thresholds = sorted({float(r) for r in ratios} | {float(np.nextafter(r, np.inf)) for r in ratios})
        for thr in thresholds:
            gi, gc = se.extract_imf(x, sd_threshold=thr)
            rechecks += c.stats()["sd_rechecks"]
            oi, oc = oracle.extract_imf(x, sd=thr)
            assert gc == oc, (n, thr, gc, oc)
            assert np.array_equal(gi, oi), (n, thr)
    assert rechecks > 0  # the uncertain branch ran


def test_sd_forced_sequential_sums_identical(se):
    """Debug bit 2 redoes every SD test with the sequential sums: results are unchanged."""
    from tests.golden.inputs import rng_signal
    x = rng_signal(31, 2500)
    c = se.context()
    a = se.decompose_full(x, "eemd", nr=6)
    c.run("semd_set_debug", 4)
    try:
        b = se.decompose_full(x, "eemd", nr=6)
    finally:
        c.run("semd_set_debug", 0)
    assert b["stats"]["sd_rechecks"] == b["stats"]["sift_iterations"] > 0
    assert np.array_equal(a["imfs"], b["imfs"]) and np.array_equal(a["residue"], b["residue"])
