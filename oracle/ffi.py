"""TEST INFRASTRUCTURE ONLY: ctypes front-ends for the parity checkers.

* ``Oracle`` -- the plain-C restatement (oracle/semd_oracle.c, liboracle.so).
* ``Ref``    -- the unmodified reference compiled from /root/reference by
  oracle/Makefile into oracle/_ref/libsemd_ref.so (present only where it was
  built; it travels to the GPU box as a prebuilt file).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module. The product (paper_2106_15319_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsemd_ref.so")

TRACE_DTYPE = np.dtype([("task", "<i4"), ("m", "<i4"), ("k", "<i4"), ("iter", "<i4"),
                        ("n_max", "<u4"), ("n_min", "<u4"), ("hash", "<u8")])

_dp = C.POINTER(C.c_double)
_szp = C.POINTER(C.c_size_t)
_u64p = C.POINTER(C.c_uint64)
_i32p = C.POINTER(C.c_int32)


def build(quiet: bool = True) -> None:
    """Build liboracle.so (and oracle/_ref when the reference sources exist)."""
    out = subprocess.run(["make", "-f", os.path.join(HERE, "Makefile"), "all"], cwd=HERE,
                         capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _f64(x) -> np.ndarray:
    return np.ascontiguousarray(x, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class _SiftCfg(C.Structure):
    _fields_ = [("sd_threshold", C.c_double), ("max_sift_iters", C.c_int32), ("max_imfs", C.c_int32)]


class _EnsCfg(C.Structure):
    _fields_ = [("nstd", C.c_double), ("nr", C.c_int32), ("_pad", C.c_int32), ("base_seed", C.c_uint64)]


class _Decomp(C.Structure):
    _fields_ = [("K", C.c_size_t), ("n", C.c_size_t), ("imfs", _dp), ("residue", _dp), ("sift_counts", _i32p)]


class _Trace(C.Structure):
    _fields_ = [("rec", C.c_void_p), ("count", C.c_size_t), ("cap", C.c_size_t)]


class Oracle:
    """The C restatement. Results are bit-identical to the reference (pinned by tests)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = L = C.CDLL(path)
        L.so_last_error.restype = C.c_char_p
        L.so_derive_seed.restype = C.c_uint64
        L.so_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.so_signal_std.restype = C.c_double
        L.so_signal_std.argtypes = [_dp, C.c_size_t]
        L.so_trace_hash.restype = C.c_uint64
        L.so_default_transition_length.restype = C.c_size_t
        L.so_default_transition_length.argtypes = [C.c_size_t]

    def _chk(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self.lib.so_last_error().decode())

    @staticmethod
    def _trace(cap: int):
        buf = np.zeros(cap, dtype=TRACE_DTYPE)
        t = _Trace(buf.ctypes.data, 0, cap)
        return buf, t

    def _take(self, d: _Decomp, rc: int):
        self._chk(rc)
        n, K = d.n, d.K
        imfs = np.ctypeslib.as_array(d.imfs, shape=(K * n,)).copy().reshape(K, n) if K else np.zeros((0, n))
        residue = np.ctypeslib.as_array(d.residue, shape=(n,)).copy()
        counts = np.ctypeslib.as_array(d.sift_counts, shape=(K,)).copy() if K else np.zeros(0, np.int32)
        self.lib.so_decomp_free(C.byref(d))
        return imfs, residue, counts

    # --- primitives ---------------------------------------------------------------
    def derive_seed(self, base: int, index: int) -> int:
        return self.lib.so_derive_seed(base, index)

    def mt19937_64(self, seed: int, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.uint64)
        self.lib.so_mt19937_64(C.c_uint64(seed), C.c_size_t(n), out.ctypes.data_as(_u64p))
        return out

    def white_noise(self, n: int, seed: int, std: float = 1.0) -> np.ndarray:
        out = np.zeros(n)
        self._chk(self.lib.so_white_noise(C.c_size_t(n), C.c_uint64(seed), C.c_double(std), _d(out)))
        return out

    def signal_std(self, x) -> float:
        x = _f64(x)
        return self.lib.so_signal_std(_d(x), x.size)

    def trace_hash(self, max_idx, min_idx) -> int:
        a = np.ascontiguousarray(max_idx, dtype=np.uint64)
        b = np.ascontiguousarray(min_idx, dtype=np.uint64)
        return self.lib.so_trace_hash(a.ctypes.data_as(_szp), C.c_size_t(a.size), b.ctypes.data_as(_szp),
                                      C.c_size_t(b.size))

    def find_extrema(self, x):
        x = _f64(x)
        n = x.size
        mi, ni = np.zeros(max(n, 1), np.uint64), np.zeros(max(n, 1), np.uint64)
        mv, nv = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        a, b = C.c_size_t(), C.c_size_t()
        self._chk(self.lib.so_find_extrema(_d(x), C.c_size_t(n), mi.ctypes.data_as(_szp), _d(mv), C.byref(a),
                                           ni.ctypes.data_as(_szp), _d(nv), C.byref(b)))
        return mi[:a.value].astype(np.int64), mv[:a.value], ni[:b.value].astype(np.int64), nv[:b.value]

    def envelope(self, idx, val, length: int) -> np.ndarray:
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        val = _f64(val)
        out = np.zeros(length)
        self._chk(self.lib.so_envelope(idx.ctypes.data_as(_szp), _d(val), C.c_size_t(idx.size),
                                       C.c_size_t(length), _d(out)))
        return out

    def extract_imf(self, x, sd=0.2, iters=300, imfs=0, trace_cap=0):
        x = _f64(x)
        out = np.zeros(x.size)
        cnt = C.c_int32()
        buf, tr = self._trace(trace_cap)
        cfg = _SiftCfg(sd, iters, imfs)
        self._chk(self.lib.so_extract_imf(_d(x), C.c_size_t(x.size), C.byref(cfg), _d(out), C.byref(cnt),
                                          C.byref(tr) if trace_cap else None))
        return out, cnt.value

    def decompose(self, x, algo=0, sd=0.2, iters=300, imfs=0, nstd=0.2, nr=100, seed=0, trace_cap=0):
        """Returns (imfs KxL, residue L, sift_counts K, trace records)."""
        x = _f64(x)
        d = _Decomp()
        buf, tr = self._trace(trace_cap)
        cfg, ens = _SiftCfg(sd, iters, imfs), _EnsCfg(nstd, nr, 0, seed)
        rc = self.lib.so_decompose(_d(x), C.c_size_t(x.size), algo, C.byref(cfg), C.byref(ens), C.byref(d),
                                   C.byref(tr) if trace_cap else None)
        imfs_, res, counts = self._take(d, rc)
        if trace_cap and tr.count > trace_cap:
            raise OracleError(5, f"trace capacity {trace_cap} < {tr.count}")
        return imfs_, res, counts, buf[:tr.count].copy()

    def emd(self, x, **kw):
        return self.decompose(x, 0, **kw)

    def eemd_partial(self, x, m_begin, m_end, sd=0.2, iters=300, imfs=0, nstd=0.2, nr=100, seed=0, trace_cap=0):
        x = _f64(x)
        d = _Decomp()
        buf, tr = self._trace(trace_cap)
        cfg, ens = _SiftCfg(sd, iters, imfs), _EnsCfg(nstd, nr, 0, seed)
        rc = self.lib.so_eemd_partial(_d(x), C.c_size_t(x.size), C.byref(cfg), C.byref(ens), m_begin, m_end,
                                      C.byref(d), C.byref(tr) if trace_cap else None)
        sums, _, _ = self._take(d, rc)
        return sums, buf[:tr.count].copy()

    def sd_ratios(self, x, sd=0.2, iters=300):
        """extract_imf -> (imf, sift_count, the reference's num/den of every sift)."""
        x = _f64(x)
        out = np.zeros(x.size)
        cnt = C.c_int32()
        r = np.zeros(max(iters, 1) + 1)
        k = C.c_size_t()
        cfg = _SiftCfg(sd, iters, 0)
        self._chk(self.lib.so_sd_ratios(_d(x), C.c_size_t(x.size), C.byref(cfg), _d(out), C.byref(cnt), _d(r),
                                        C.c_size_t(r.size), C.byref(k)))
        return out, cnt.value, r[:k.value].copy()

    # --- serializer ---------------------------------------------------------------
    def concatenate(self, x_cm: np.ndarray, M: int, N: int, D: int, naive: bool = False) -> np.ndarray:
        x = _f64(x_cm).ravel()
        out = np.zeros(max(M * N + D * (N - 1), 1))
        fn = self.lib.so_concatenate_naive if naive else self.lib.so_concatenate
        self._chk(fn(_d(x), C.c_size_t(M), C.c_size_t(N), C.c_size_t(D), _d(out)))
        return out[:M * N + D * (N - 1)]

    def deconcatenate(self, modes: np.ndarray, M: int, N: int, D: int) -> np.ndarray:
        modes = _f64(modes)
        K, L = modes.shape
        out = np.zeros(max(K * M * N, 1))
        self._chk(self.lib.so_deconcatenate(_d(modes), C.c_size_t(K), C.c_size_t(L), C.c_size_t(M), C.c_size_t(N),
                                            C.c_size_t(D), _d(out)))
        return out[:K * M * N].reshape(K, N, M)

    def serial_decompose(self, x_cm, M, N, D, algo=0, sd=0.2, iters=300, imfs=0, nstd=0.2, nr=100, seed=0,
                         trace_cap=0):
        x = _f64(x_cm).ravel()
        p = _dp()
        k1 = C.c_size_t()
        buf, tr = self._trace(trace_cap)
        cfg, ens = _SiftCfg(sd, iters, imfs), _EnsCfg(nstd, nr, 0, seed)
        self._chk(self.lib.so_serial_decompose(_d(x), C.c_size_t(M), C.c_size_t(N), C.c_size_t(D), algo,
                                               C.byref(cfg), C.byref(ens), C.byref(p), C.byref(k1),
                                               C.byref(tr) if trace_cap else None))
        t = np.ctypeslib.as_array(p, shape=(k1.value * M * N,)).copy().reshape(k1.value, N, M)
        self.lib.so_free(p)
        return t, buf[:tr.count].copy()

    def multivariate_sinusoids(self, n: int = 1000, fs: float = 1000.0) -> np.ndarray:
        """Channel-contiguous (6, n) array (row j = variate j)."""
        out = np.zeros(6 * n)
        self._chk(self.lib.so_multivariate_sinusoids(C.c_size_t(n), C.c_double(fs), _d(out)))
        return out.reshape(6, n)

    def default_transition_length(self, rows: int) -> int:
        return self.lib.so_default_transition_length(rows)


class Ref:
    """The unmodified reference (oracle/_ref/libsemd_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        for f in ("ref_out_imfs", "ref_out_residue"):
            getattr(L, f).restype = _dp
            getattr(L, f).argtypes = [C.c_void_p]
        L.ref_out_counts.restype = _i32p
        L.ref_out_counts.argtypes = [C.c_void_p]
        L.ref_out_trace.restype = C.c_void_p
        L.ref_out_trace.argtypes = [C.c_void_p]
        for f in ("ref_out_K", "ref_out_ncounts", "ref_out_ntrace"):
            getattr(L, f).restype = C.c_size_t
            getattr(L, f).argtypes = [C.c_void_p]
        L.ref_out_new.restype = C.c_void_p
        L.ref_out_free.argtypes = [C.c_void_p]
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_signal_std.restype = C.c_double
        L.ref_signal_std.argtypes = [_dp, C.c_size_t]
        L.ref_default_transition_length.restype = C.c_size_t
        L.ref_default_transition_length.argtypes = [C.c_size_t]
        L.ref_decompose.argtypes = [_dp, C.c_size_t, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                                    C.c_uint64, C.c_void_p]
        L.ref_emd_traced.argtypes = [_dp, C.c_size_t, C.c_double, C.c_int, C.c_int, C.c_void_p]
        L.ref_eemd_traced.argtypes = [_dp, C.c_size_t, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                                      C.c_uint64, C.c_int, C.c_int, C.c_void_p]
        L.ref_ceemdan_traced.argtypes = [_dp, C.c_size_t, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                                         C.c_uint64, C.c_void_p]
        L.ref_emd_realizations.argtypes = [_dp, C.c_size_t, C.c_double, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                           C.c_int, C.c_int, C.c_int, _dp]
        L.ref_serial_decompose.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, C.c_double, C.c_int,
                                           C.c_int, C.c_double, C.c_int, C.c_uint64, C.c_void_p]
        L.ref_realization_summary.argtypes = [_dp, C.c_size_t, C.c_double, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                              C.c_int, C.c_int, _u64p, C.c_size_t, C.c_void_p]
        L.ref_eemd_stream.argtypes = [_dp, C.c_size_t, C.c_double, C.c_int, C.c_int, C.c_double, C.c_int,
                                      C.c_uint64, C.c_int, C.c_void_p]
        L.ref_realization_sifts.argtypes = [_dp, C.c_size_t, C.c_double, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                            C.c_int, C.c_int, C.c_int, _u64p, _i32p]

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def _out(self, o, n):
        L = self.lib
        K = L.ref_out_K(o)
        imfs = np.ctypeslib.as_array(L.ref_out_imfs(o), shape=(K * n,)).copy().reshape(K, n) if K else np.zeros((0, n))
        rp = L.ref_out_residue(o)
        residue = np.ctypeslib.as_array(rp, shape=(n,)).copy() if rp else None
        nc = L.ref_out_ncounts(o)
        counts = np.ctypeslib.as_array(L.ref_out_counts(o), shape=(nc,)).copy() if nc else np.zeros(0, np.int32)
        nt = L.ref_out_ntrace(o)
        trace = np.frombuffer(C.string_at(L.ref_out_trace(o), nt * TRACE_DTYPE.itemsize), dtype=TRACE_DTYPE).copy() \
            if nt else np.zeros(0, TRACE_DTYPE)
        return imfs, residue, counts, trace

    def derive_seed(self, base, index):
        return self.lib.ref_derive_seed(base, index)

    def mt19937_64(self, seed, n):
        out = np.zeros(n, dtype=np.uint64)
        self.lib.ref_mt19937_64(C.c_uint64(seed), C.c_size_t(n), out.ctypes.data_as(_u64p))
        return out

    def white_noise(self, n, seed, std=1.0):
        out = np.zeros(n)
        self._chk(self.lib.ref_white_noise(C.c_size_t(n), C.c_uint64(seed), C.c_double(std), _d(out)))
        return out

    def signal_std(self, x):
        x = _f64(x)
        return self.lib.ref_signal_std(_d(x), x.size)

    def find_extrema(self, x):
        x = _f64(x)
        n = x.size
        mi, ni = np.zeros(max(n, 1), np.uint64), np.zeros(max(n, 1), np.uint64)
        mv, nv = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        a, b = C.c_size_t(), C.c_size_t()
        self._chk(self.lib.ref_find_extrema(_d(x), C.c_size_t(n), mi.ctypes.data_as(_szp), _d(mv), C.byref(a),
                                            ni.ctypes.data_as(_szp), _d(nv), C.byref(b)))
        return mi[:a.value].astype(np.int64), mv[:a.value], ni[:b.value].astype(np.int64), nv[:b.value]

    def envelope(self, idx, val, length):
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        val = _f64(val)
        out = np.zeros(length)
        self._chk(self.lib.ref_envelope(idx.ctypes.data_as(_szp), _d(val), C.c_size_t(idx.size),
                                        C.c_size_t(length), _d(out)))
        return out

    def extract_imf(self, x, sd=0.2, iters=300, imfs=0):
        x = _f64(x)
        out = np.zeros(x.size)
        cnt = C.c_int32()
        self._chk(self.lib.ref_extract_imf(_d(x), C.c_size_t(x.size), C.c_double(sd), iters, imfs, _d(out),
                                           C.byref(cnt)))
        return out, cnt.value

    def decompose(self, x, algo=0, sd=0.2, iters=300, imfs=0, nstd=0.2, nr=100, seed=0):
        x = _f64(x)
        o = self.lib.ref_out_new()
        try:
            self._chk(self.lib.ref_decompose(_d(x), x.size, algo, sd, iters, imfs, nstd, nr, seed, o))
            imfs_, res, _, _ = self._out(o, x.size)
        finally:
            self.lib.ref_out_free(o)
        return imfs_, res

    def emd(self, x, **kw):
        return self.decompose(x, 0, **kw)

    def emd_traced(self, x, sd=0.2, iters=300, imfs=0):
        x = _f64(x)
        o = self.lib.ref_out_new()
        try:
            self._chk(self.lib.ref_emd_traced(_d(x), x.size, sd, iters, imfs, o))
            return self._out(o, x.size)
        finally:
            self.lib.ref_out_free(o)

    def eemd_traced(self, x, m_begin, m_end, sd=0.2, iters=300, imfs=0, nstd=0.2, nr=100, seed=0):
        """Unscaled realization sums over [m_begin, m_end), per-realization [K_m, counts...], traces."""
        x = _f64(x)
        o = self.lib.ref_out_new()
        try:
            self._chk(self.lib.ref_eemd_traced(_d(x), x.size, sd, iters, imfs, nstd, nr, seed, m_begin, m_end, o))
            sums, _, counts, trace = self._out(o, x.size)
            return sums, counts, trace
        finally:
            self.lib.ref_out_free(o)

    def ceemdan_traced(self, x, sd=0.2, iters=300, imfs=0, nstd=0.2, nr=100, seed=0):
        x = _f64(x)
        o = self.lib.ref_out_new()
        try:
            self._chk(self.lib.ref_ceemdan_traced(_d(x), x.size, sd, iters, imfs, nstd, nr, seed, o))
            imfs_, res, _, trace = self._out(o, x.size)
            return imfs_, res, trace
        finally:
            self.lib.ref_out_free(o)

    def emd_realizations(self, x, m_begin, count, threads, sd=0.2, iters=300, imfs=0, nstd=0.2, seed=0) -> float:
        x = _f64(x)
        chk = C.c_double()
        self._chk(self.lib.ref_emd_realizations(_d(x), x.size, sd, iters, imfs, nstd, seed, m_begin, count, threads,
                                                C.byref(chk)))
        return chk.value

    def realization_summary(self, x, m, sample_idx, check=False, sd=0.2, iters=300, imfs=0, nstd=0.2, seed=0):
        """EEMD realization m (emd.cpp:237-244) through the replayer: (sift counts per IMF, trace,
        per-IMF L2 norms, IMF values at sample_idx (K x ns)). check: also bit-compare with semd::emd."""
        x = _f64(x)
        idx = np.ascontiguousarray(sample_idx, dtype=np.uint64)
        o = self.lib.ref_out_new()
        try:
            self._chk(self.lib.ref_realization_summary(_d(x), x.size, sd, iters, imfs, nstd, seed, int(m), int(check),
                                                       idx.ctypes.data_as(_u64p), idx.size, o))
            L = self.lib
            K = L.ref_out_K(o)
            ns = idx.size
            samples = np.ctypeslib.as_array(L.ref_out_imfs(o), shape=(K * ns,)).copy().reshape(K, ns) if K * ns \
                else np.zeros((K, ns))
            norms = np.ctypeslib.as_array(L.ref_out_residue(o), shape=(K,)).copy() if K else np.zeros(0)
            nc = L.ref_out_ncounts(o)
            counts = np.ctypeslib.as_array(L.ref_out_counts(o), shape=(nc,)).copy() if nc else np.zeros(0, np.int32)
            nt = L.ref_out_ntrace(o)
            trace = np.frombuffer(C.string_at(L.ref_out_trace(o), nt * TRACE_DTYPE.itemsize), dtype=TRACE_DTYPE).copy()
            return counts, trace, norms, samples
        finally:
            self.lib.ref_out_free(o)

    def eemd_stream(self, x, threads, sd=0.2, iters=300, imfs=0, nstd=0.2, nr=100, seed=0):
        """semd::eemd (bit-identical) with realizations streamed in order over `threads` workers.
        Returns (imfs KxL, residue L, per-realization K)."""
        x = _f64(x)
        o = self.lib.ref_out_new()
        try:
            self._chk(self.lib.ref_eemd_stream(_d(x), x.size, sd, iters, imfs, nstd, nr, seed, threads, o))
            imfs_, res, counts, _ = self._out(o, x.size)
            return imfs_, res, counts
        finally:
            self.lib.ref_out_free(o)

    def realization_sifts(self, x, m_begin, count, threads, sd=0.2, iters=300, imfs=0, nstd=0.2, seed=0):
        """(n x total sift iterations, per-realization sift totals) of EEMD realizations
        [m_begin, m_begin+count), computed on the CPU by the reference's extract_imf."""
        x = _f64(x)
        tot = C.c_uint64()
        per = np.zeros(max(count, 1), np.int32)
        self._chk(self.lib.ref_realization_sifts(_d(x), x.size, sd, iters, imfs, nstd, seed, m_begin, count, threads,
                                                 C.byref(tot), per.ctypes.data_as(_i32p)))
        return int(tot.value), per[:count]

    def concatenate(self, x_cm, M, N, D, naive=False):
        x = _f64(x_cm).ravel()
        out = np.zeros(max(M * N + D * (N - 1), 1))
        self._chk(self.lib.ref_concatenate(_d(x), C.c_size_t(M), C.c_size_t(N), C.c_size_t(D), int(naive), _d(out)))
        return out[:M * N + D * (N - 1)]

    def deconcatenate(self, modes, M, N, D):
        modes = _f64(modes)
        K, L = modes.shape
        out = np.zeros(max(K * M * N, 1))
        self._chk(self.lib.ref_deconcatenate(_d(modes), C.c_size_t(K), C.c_size_t(L), C.c_size_t(M), C.c_size_t(N),
                                             C.c_size_t(D), _d(out)))
        return out[:K * M * N].reshape(K, N, M)

    def serial_decompose(self, x_cm, M, N, D, algo=0, sd=0.2, iters=300, imfs=0, nstd=0.2, nr=100, seed=0):
        x = _f64(x_cm).ravel()
        o = self.lib.ref_out_new()
        try:
            self._chk(self.lib.ref_serial_decompose(_d(x), M, N, D, algo, sd, iters, imfs, nstd, nr, seed, o))
            K1 = self.lib.ref_out_K(o)
            t = np.ctypeslib.as_array(self.lib.ref_out_imfs(o), shape=(K1 * M * N,)).copy().reshape(K1, N, M)
        finally:
            self.lib.ref_out_free(o)
        return t

    def multivariate_sinusoids(self, n=1000, fs=1000.0):
        out = np.zeros(6 * n)
        self._chk(self.lib.ref_multivariate_sinusoids(C.c_size_t(n), C.c_double(fs), _d(out)))
        return out.reshape(6, n)

    def default_transition_length(self, rows):
        return self.lib.ref_default_transition_length(rows)


def ref_available() -> bool:
    return os.path.exists(REF_SO)
