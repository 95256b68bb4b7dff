"""Pin the oracle (the plain-C restatement) to the golden vectors produced by
the reference itself (tests/golden/make_golden.py)."""
import numpy as np
import pytest

from tests.conftest import fromhex, sha, sort_trace
from tests.golden.inputs import C_CONFIGS, pickup_serialized, rng_signal


def test_derive_seed_and_mt19937_64(oracle, golden):
    for b, i, v in golden["derive_seed"]:
        assert oracle.derive_seed(b, i) == v
    # [rand.predef]: 10000th draw of a default-constructed mt19937_64
    assert int(oracle.mt19937_64(5489, 10000)[-1]) == golden["mt19937_64_default_10000th"] == 9981545732273789042
    for seed, draws in golden["mt19937_64_seed_first"].items():
        assert [int(v) for v in oracle.mt19937_64(int(seed), 8)] == draws


def test_white_noise_known_answers(oracle, golden):
    w = oracle.white_noise(4, oracle.derive_seed(0, 0))
    assert np.array_equal(w, fromhex(golden["white_noise_4_seed_ds00"]))
    assert np.array_equal(w, [0.42398543408524497, -0.2190339834701002, -0.57701778896195799, -0.42265740857495115])
    w = oracle.white_noise(1001, 7)
    assert sha(w) == golden["white_noise_1001_seed7"]["sha256"]
    assert np.array_equal(oracle.white_noise(5, 42, 0.0), np.zeros(5))


def test_find_extrema_cases(oracle, golden):
    for case in golden["find_extrema"]:
        x = fromhex(case["x"])
        mi, mv, ni, nv = oracle.find_extrema(x)
        assert mi.tolist() == case["max_idx"], case["name"]
        assert ni.tolist() == case["min_idx"], case["name"]
        assert np.array_equal(mv, fromhex(case["max_val"]))
        assert np.array_equal(nv, fromhex(case["min_val"]))


def test_envelope_cases(oracle, golden):
    for case in golden["envelope"]:
        out = oracle.envelope(case["idx"], fromhex(case["val"]), case["length"])
        assert np.array_equal(out, fromhex(case["out"])), case["name"]


def test_serializer_known_answers(oracle, golden):
    for m, d in golden["default_transition_length"]:
        assert oracle.default_transition_length(m) == d
    assert np.array_equal(oracle.concatenate(np.array([[0.0, 3.0], [6.0, 9.0]]), 2, 2, 2),
                          fromhex(golden["concat_hand"]))
    assert np.array_equal(fromhex(golden["concat_hand"]), [0.0, 3.0, 5.0, 4.0, 6.0, 9.0])  # test_serialize.cpp:41-52


def test_emd_random_signals(oracle, golden):
    for case in golden["emd_random"]:
        x = rng_signal(case["seed"], case["n"])
        if case["n"] < 4:
            continue
        imfs, res, counts, tr = oracle.emd(x, imfs=case["max_imfs"], trace_cap=100000)
        assert imfs.shape[0] == case["K"]
        assert counts.tolist() == case["counts"]
        assert sha(imfs) == case["imfs_sha256"]
        assert sha(res) == case["residue_sha256"]
        got = [[int(t[k]) for k in ("k", "iter", "n_max", "n_min", "hash")] for t in tr]
        assert got == case["trace"]


def test_small_ensembles(oracle, golden):
    for case in golden["ensembles_small"]:
        x = rng_signal(case["seed"], case["n"])
        imfs, res, _, _ = oracle.decompose(x, case["algo"], nr=case["nr"])
        assert sha(imfs) == case["imfs_sha256"]
        assert sha(res) == case["residue_sha256"]


@pytest.mark.parametrize("name", ["c1_emd_D50", "c2_eemd_D1", "c2_eemd_D50", "c2_eemd_D500"])
def test_baseline_configs(oracle, golden, golden_traces, name):
    c = golden["configs"][name]
    s = pickup_serialized(oracle, c["D"])
    assert s.size == c["L"] and sha(s) == c["input_sha256"]
    imfs, res, counts, tr = oracle.decompose(s, c["algo"], iters=c["iters"], imfs=c["imfs"], nr=c["nr"],
                                             trace_cap=1_000_000)
    assert imfs.shape[0] == c["K"]
    assert sha(imfs) == c["imfs_sha256"]
    assert sha(res) == c["residue_sha256"]
    assert np.array_equal(sort_trace(tr), sort_trace(golden_traces[name]))
    if c["algo"] == 0:
        assert counts.tolist() == c["counts"]


def test_c3_ceemdan(oracle, golden, golden_traces):
    c = golden["configs"]["c3_ceemdan_D50"]
    s = pickup_serialized(oracle, c["D"])
    imfs, res, _, tr = oracle.decompose(s, 2, iters=c["iters"], imfs=c["imfs"], nr=c["nr"], trace_cap=1_000_000)
    assert imfs.shape[0] == c["K"] == 9
    assert sha(imfs) == c["imfs_sha256"]
    assert sha(res) == c["residue_sha256"]
    assert np.array_equal(sort_trace(tr), sort_trace(golden_traces["c3_ceemdan_D50"]))
    # 110,387,500 sifted samples
    sifted = int(s.size) * int(((tr["task"] != 3) & (tr["n_max"] >= 2) & (tr["n_min"] >= 2)).sum())
    assert sifted == c["sifted_samples"] == 110_387_500


def test_sifted_sample_counts(golden):
    # SURVEY.md §8(d) probe counts
    cf = golden["configs"]
    assert cf["c1_emd_D50"]["sifted_samples"] == 62_500
    assert cf["c2_eemd_D1"]["sifted_samples"] == 9_517_925
    assert cf["c2_eemd_D50"]["sifted_samples"] == 10_043_750
    assert cf["c2_eemd_D500"]["sifted_samples"] == 13_974_000
