"""The resident engine (semd_resident.cu: one persistent CTA per job, candidate and segment tables
in shared memory) against the lockstep engine, the oracle and the reference's golden data.

The default engine choice sends signals of at most SEMD_RESIDENT_MAX_L samples to the resident
engine, so the C1-C3 golden tests in test_gpu_parity.py already run on it; here both engines are
forced and compared bit for bit, the repair paths are forced, and the shared-memory overflow
fallback is exercised."""
import numpy as np
import pytest

from tests.conftest import sort_trace
from tests.golden.inputs import rng_signal

pytestmark = pytest.mark.gpu

AUTO, LOCKSTEP, RESIDENT = 0, 1, 2


def bits(a):
    return np.ascontiguousarray(a).view(np.int64)


def run(se, engine, x, algo, debug=0, **kw):
    c = se.context()
    c.check(c.lib.semd_set_engine(c.ptr, engine))
    c.check(c.lib.semd_set_debug(c.ptr, debug))
    try:
        return se.decompose_full(x, algo, trace_cap=200000, **kw)
    finally:
        c.check(c.lib.semd_set_debug(c.ptr, 0))
        c.check(c.lib.semd_set_engine(c.ptr, AUTO))


def same(a, b):
    assert a["imfs"].shape == b["imfs"].shape
    assert np.array_equal(bits(a["imfs"]), bits(b["imfs"]))
    assert np.array_equal(bits(a["residue"]), bits(b["residue"]))
    assert np.array_equal(sort_trace(a["trace"]), sort_trace(b["trace"]))


def pickup(se, D=50):
    from paper_2106_15319_b200 import workloads as W
    return se.concatenate(W.pickup_signals(), D)


@pytest.mark.parametrize("algo,kw", [("emd", dict(max_sift_iters=1000)),
                                     ("eemd", dict(max_sift_iters=300, max_imfs=10, nr=100)),
                                     ("ceemdan", dict(max_sift_iters=5000, nr=100))])
def test_resident_equals_lockstep_pickup(se, algo, kw):
    """C1-C3 inputs: IMFs, residue and the full parity trace bit-identical across the two engines."""
    s = pickup(se)
    a = run(se, LOCKSTEP, s, algo, **kw)
    b = run(se, RESIDENT, s, algo, **kw)
    assert a["stats"]["resident_jobs"] == 0 and b["stats"]["resident_jobs"] > 0
    same(a, b)
    if algo == "emd":
        assert np.array_equal(a["sift_counts"], b["sift_counts"])


def test_resident_emd_vs_oracle_many_lengths(se, oracle):
    """Plain EMD, bit-exact against the oracle at lengths 4 .. the resident maximum (white noise of
    8188 samples has ~5.5k extrema: its tables outgrow the shared memory and the call falls back)."""
    for n in (4, 5, 7, 64, 129, 1000, 3001, 6250, 8188):
        x = rng_signal(n, n)
        d = run(se, RESIDENT, x, "emd", max_sift_iters=300)
        oi, ores, _, otr = oracle.decompose(x, 0, trace_cap=100000)
        assert d["stats"]["resident_jobs"] == (1 if n <= 6250 else 0), n
        assert np.array_equal(bits(d["imfs"]), bits(oi)), n
        assert np.array_equal(bits(d["residue"]), bits(ores)), n
        assert np.array_equal(sort_trace(d["trace"]), sort_trace(otr)), n


def test_resident_plateaus_vs_oracle(se, oracle):
    """find_extrema's plateau rule (emd.cpp:16-33) inside the resident detection."""
    rng = np.random.default_rng(7)
    for n in (300, 2500):
        x = np.round(rng.standard_normal(n).cumsum() * 2) / 2  # many equal neighbours
        x[100:140] = x[99]  # one long plateau
        d = run(se, RESIDENT, x, "emd", max_sift_iters=50)
        oi, ores, _, otr = oracle.decompose(x, 0, iters=50, trace_cap=100000)
        assert np.array_equal(bits(d["imfs"]), bits(oi)) and np.array_equal(bits(d["residue"]), bits(ores))
        assert np.array_equal(sort_trace(d["trace"]), sort_trace(otr))


def test_resident_forced_replays_bit_exact(se):
    """Debug bit 0: two-row warm-ups make the speculative chains disagree at their boundaries; the
    in-order replay must restore the sequential Thomas result exactly."""
    s = pickup(se)
    a = run(se, LOCKSTEP, s, "eemd", max_imfs=10, nr=20)
    b = run(se, RESIDENT, s, "eemd", debug=1, max_imfs=10, nr=20)
    assert b["stats"]["solve_hazards"] > 0
    same(a, b)


def test_resident_sd_sequential_path(se):
    """Debug bit 2: every SD decision redone with the reference's left-to-right sums."""
    s = pickup(se)
    a = run(se, LOCKSTEP, s, "emd", max_sift_iters=1000)
    b = run(se, RESIDENT, s, "emd", debug=4, max_sift_iters=1000)
    assert b["stats"]["sd_rechecks"] == b["stats"]["sift_iterations"] > 0
    same(a, b)


def test_resident_smem_overflow_falls_back(se, oracle):
    """Segment tables larger than the shared memory (every sample an extremum) rerun the call on the
    lockstep engine; the result is still the reference's."""
    n = 8188
    x = np.where(np.arange(n) % 2 == 0, 1.0, -1.0) + np.arange(n) * 1e-6
    d = run(se, RESIDENT, x, "emd", max_sift_iters=20)
    oi, ores, _, otr = oracle.decompose(x, 0, iters=20, trace_cap=100000)
    assert np.array_equal(bits(d["imfs"]), bits(oi)) and np.array_equal(bits(d["residue"]), bits(ores))
    assert np.array_equal(sort_trace(d["trace"]), sort_trace(otr))
    assert d["stats"]["steps"] > 0  # the lockstep engine ran


def test_resident_ceemdan_vs_oracle(se, oracle):
    """CEEMDAN task jobs (noise modes in place, first modes accumulated in realization order)."""
    s = pickup(se)[:3000]
    d = run(se, RESIDENT, s, "ceemdan", max_sift_iters=300, nr=16)
    oi, ores, _, otr = oracle.decompose(s, 2, nr=16, trace_cap=200000)
    assert np.array_equal(bits(d["imfs"]), bits(oi)) and np.array_equal(bits(d["residue"]), bits(ores))
    assert np.array_equal(sort_trace(d["trace"]), sort_trace(otr))


@pytest.mark.parametrize("n,nr,max_imfs,iters", [(12, 5, 0, 300), (64, 3, 0, 300), (200, 1, 0, 50),
                                                 (700, 8, 2, 300), (1500, 6, 0, 1000)])
def test_resident_ceemdan_edges_vs_lockstep_and_oracle(se, oracle, n, nr, max_imfs, iters):
    """The fused device CEEMDAN (k_res_ceemdan) on small cases: noise modes running out (alive
    flags), residue checks ending the stage loop, nr = 1 and a max_imfs limit -- IMFs, residue and
    the full trace bit-identical to the lockstep per-stage drivers and to the oracle."""
    rng = np.random.default_rng(n)
    x = np.sin(np.arange(n) * 0.3) + 0.5 * rng.standard_normal(n)
    kw = dict(nr=nr, max_imfs=max_imfs, max_sift_iters=iters)
    a = run(se, LOCKSTEP, x, "ceemdan", **kw)
    b = run(se, RESIDENT, x, "ceemdan", **kw)
    assert b["stats"]["resident_jobs"] > 0
    same(a, b)
    oi, ores, _, otr = oracle.decompose(x, 2, iters=iters, imfs=max_imfs, nr=nr, trace_cap=200000)
    assert np.array_equal(bits(b["imfs"]), bits(oi)) and np.array_equal(bits(b["residue"]), bits(ores))
    assert np.array_equal(sort_trace(b["trace"]), sort_trace(otr))


@pytest.mark.parametrize("n,nr", [(16, 4), (500, 3)])
def test_resident_eemd_small_vs_oracle(se, oracle, n, nr):
    """EEMD job queue + realization-ordered accumulation on small signals (IMF counts that differ
    between realizations: shorter lists count as zeros, emd.cpp:246-251)."""
    rng = np.random.default_rng(n + 1)
    x = np.cos(np.arange(n) * 0.2) + 0.4 * rng.standard_normal(n)
    b = run(se, RESIDENT, x, "eemd", nr=nr, max_sift_iters=300)
    oi, ores, _, otr = oracle.decompose(x, 1, nr=nr, trace_cap=200000)
    assert b["stats"]["resident_jobs"] == nr
    assert np.array_equal(bits(b["imfs"]), bits(oi)) and np.array_equal(bits(b["residue"]), bits(ores))
    assert np.array_equal(sort_trace(b["trace"]), sort_trace(otr))


def test_smoke_in_fresh_process():
    """__graft_entry__.smoke() as the driver runs it: a fresh process whose first decomposition is
    on the resident engine (the control block's trace counter must start reset)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke()"], cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "smoke ok" in r.stdout


@pytest.mark.parametrize("algo,kw", [("eemd", dict(max_sift_iters=300, max_imfs=10, nr=100)),
                                     ("ceemdan", dict(max_sift_iters=5000, nr=500))])
def test_resident_untraced_equals_lockstep(se, algo, kw):
    """C2/C3 without tracing (the bench's and the CLI's mode, where the resident kernels take their
    untraced paths): IMFs and residue bit-identical to the lockstep engine."""
    s = pickup(se)
    c = se.context()
    out = {}
    for eng in (LOCKSTEP, RESIDENT):
        c.check(c.lib.semd_set_engine(c.ptr, eng))
        try:
            out[eng] = se.decompose_full(s, algo, **kw)
        finally:
            c.check(c.lib.semd_set_engine(c.ptr, AUTO))
    a, b = out[LOCKSTEP], out[RESIDENT]
    assert b["stats"]["resident_jobs"] > 0 and a["stats"]["resident_jobs"] == 0
    assert a["imfs"].shape == b["imfs"].shape
    assert np.array_equal(bits(a["imfs"]), bits(b["imfs"])) and np.array_equal(bits(a["residue"]), bits(b["residue"]))


def _fuzz_signal(rng, n, kind):
    t = np.arange(n, dtype=np.float64)
    if kind == "noise":
        return rng.standard_normal(n)
    if kind == "chirp":
        return np.sin(t * t * 1e-4 * rng.uniform(0.5, 2)) + 0.1 * rng.standard_normal(n)
    if kind == "steps":  # long plateaus and equal neighbours
        return np.round(np.cumsum(rng.standard_normal(n)) * rng.uniform(0.5, 2)) / 2
    if kind == "spikes":
        x = 0.01 * rng.standard_normal(n)
        x[rng.integers(0, n, max(1, n // 50))] += rng.uniform(-1e3, 1e3, max(1, n // 50))
        return x
    # mixed scales
    return np.sin(t * 0.02) * 1e6 + rng.standard_normal(n) * 1e-3


@pytest.mark.parametrize("case", range(24))
def test_resident_fuzz_vs_oracle(se, oracle, case):
    """Seeded random lengths (4 .. the resident maximum), algorithms and signal shapes (noise,
    chirps, plateaus/steps, spikes, mixed scales): the resident engine's IMFs, residue and trace
    equal the oracle's bit for bit."""
    rng = np.random.default_rng(1000 + case)
    kind = ["noise", "chirp", "steps", "spikes", "mixed"][case % 5]
    algo = ["emd", "eemd", "ceemdan"][case % 3]
    n = int(rng.integers(4, 7000 if algo == "emd" else 2500))
    x = _fuzz_signal(rng, n, kind)
    iters = int(rng.choice([3, 50, 300]))
    imfs = int(rng.choice([0, 0, 2, 5]))
    nr = int(rng.integers(1, 6))
    code = {"emd": 0, "eemd": 1, "ceemdan": 2}[algo]
    try:
        oi, ores, _, otr = oracle.decompose(x, code, iters=iters, imfs=imfs, nr=nr, trace_cap=400000)
    except Exception as e:  # the reference rejects the input: so must the engine, with the same message
        with pytest.raises(se.InvalidInput, match=str(e).split(": ", 1)[-1][:40] if ": " in str(e) else None):
            run(se, RESIDENT, x, algo, max_sift_iters=iters, max_imfs=imfs, nr=nr)
        return
    d = run(se, RESIDENT, x, algo, max_sift_iters=iters, max_imfs=imfs, nr=nr)
    assert d["imfs"].shape == oi.shape, (n, kind, algo)
    assert np.array_equal(bits(d["imfs"]), bits(oi)), (n, kind, algo)
    assert np.array_equal(bits(d["residue"]), bits(ores)), (n, kind, algo)
    assert np.array_equal(sort_trace(d["trace"]), sort_trace(otr)), (n, kind, algo)


def test_python_set_engine(se):
    """Context.set_engine: the Python mirror of semd_set_engine."""
    c = se.context()
    s = pickup(se)
    try:
        c.set_engine("lockstep")
        assert se.decompose_full(s, "emd")["stats"]["resident_jobs"] == 0
        c.set_engine("resident")
        assert se.decompose_full(s, "emd")["stats"]["resident_jobs"] == 1
        with pytest.raises(se.InvalidInput, match="unknown engine"):
            c.set_engine("fast")
    finally:
        c.set_engine("auto")
