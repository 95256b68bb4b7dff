"""The oracle restatement against the reference library itself (oracle/_ref,
compiled from /root/reference by oracle/Makefile): bit-identical results on
randomized sweeps. Skipped where the reference is not built."""
import numpy as np
import pytest

from tests.golden.inputs import TestRng, rng_signal


def test_concatenate_sweep(oracle, ref):
    g = TestRng(34)  # test_serialize.cpp:107-121 / acceptance criterion 2
    for _ in range(200):
        m = g.range(4, 60)
        n = g.range(1, 8)
        d = g.range(1, m)
        x = np.array([g.uniform() for _ in range(m * n)])
        a = oracle.concatenate(x, m, n, d)
        assert np.array_equal(a, ref.concatenate(x, m, n, d))
        assert np.array_equal(a, oracle.concatenate(x, m, n, d, naive=True))
        assert np.array_equal(a, ref.concatenate(x, m, n, d, naive=True))


def test_deconcatenate_roundtrip(oracle, ref):
    g = TestRng(35)
    for _ in range(50):
        m, n = g.range(4, 40), g.range(1, 6)
        d = g.range(1, m)
        x = np.array([g.uniform() for _ in range(m * n)])
        s = oracle.concatenate(x, m, n, d)
        modes = np.stack([s, s * 2.0])
        a = oracle.deconcatenate(modes, m, n, d)
        assert np.array_equal(a, ref.deconcatenate(modes, m, n, d))
        assert np.array_equal(a[0], x.reshape(n, m))


def test_find_extrema_plateaus(oracle, ref):
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = int(rng.integers(3, 60))
        x = rng.integers(-3, 4, size=n).astype(float)  # many exact plateaus
        a, b = oracle.find_extrema(x), ref.find_extrema(x)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)


def test_envelope_random(oracle, ref):
    rng = np.random.default_rng(6)
    for _ in range(200):
        length = int(rng.integers(5, 200))
        k = int(rng.integers(2, min(12, length)))
        idx = np.sort(rng.choice(length, size=k, replace=False))
        val = rng.standard_normal(k)
        assert np.array_equal(oracle.envelope(idx, val, length), ref.envelope(idx, val, length))


@pytest.mark.parametrize("seed", range(8))
def test_emd_random(oracle, ref, seed):
    n = 50 + 97 * seed
    x = rng_signal(100 + seed, n)
    a = oracle.emd(x, iters=300 if seed % 2 else 7)
    b = ref.decompose(x, 0, iters=300 if seed % 2 else 7)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("algo", [1, 2])
def test_ensembles_random(oracle, ref, algo):
    for seed in range(3):
        x = rng_signal(200 + seed, 150 + 40 * seed)
        a = oracle.decompose(x, algo, nr=4 + seed, seed=seed)
        b = ref.decompose(x, algo, nr=4 + seed, seed=seed)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_serial_decompose(oracle, ref):
    x = oracle.multivariate_sinusoids()
    a, _ = oracle.serial_decompose(x, 1000, 6, 50, 0)
    assert np.array_equal(a, ref.serial_decompose(x, 1000, 6, 50, 0))


def test_errors_match(oracle, ref):
    from oracle.ffi import OracleError
    for fn in (lambda o: o.find_extrema([1.0, 2.0]), lambda o: o.emd(np.zeros(3)),
               lambda o: o.concatenate(np.zeros(20), 10, 2, 11), lambda o: o.envelope([4], [1.0], 10)):
        with pytest.raises(OracleError) as e1:
            fn(oracle)
        with pytest.raises(OracleError) as e2:
            fn(ref)
        assert str(e1.value) == str(e2.value)
        assert e1.value.code == e2.value.code
