"""Python mirror of the reference's public interface, running on the B200 engine.

Same names, argument meaning and error behaviour as the reference's Python
module (/root/reference/proj/python/module.cpp:108-227, serialemd/__init__.py)
and its C++ free functions (include/semd/emd.hpp, serialize.hpp):
InvalidInput -> ValueError (InsufficientExtrema is a ValueError subclass),
CUDA failures -> RuntimeError. Every call goes through the C ABI of
libsemd_b200.so; nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _native as N


class InvalidInput(ValueError):
    """types.hpp:15-17 semd::InvalidInput."""


class InsufficientExtrema(InvalidInput):
    """types.hpp:20-22 semd::InsufficientExtrema."""


class CapacityError(InvalidInput):
    pass


class EngineError(RuntimeError):
    pass


_ctx_lock = threading.Lock()
_ctxs: dict[int, "Context"] = {}


def _check(lib, rc: int) -> None:
    if rc == N.SEMD_OK:
        return
    msg = lib.semd_last_error().decode()
    if rc == N.SEMD_INSUFFICIENT_EXTREMA:
        raise InsufficientExtrema(msg)
    if rc == N.SEMD_INVALID_INPUT:
        raise InvalidInput(msg)
    if rc == N.SEMD_CAPACITY:
        raise CapacityError(msg)
    if rc == N.SEMD_NO_MEMORY:
        raise MemoryError(msg)
    raise EngineError(msg)


def _f64(x, ndim=None) -> np.ndarray:
    a = np.ascontiguousarray(x, dtype=np.float64)
    if ndim is not None and a.ndim != ndim:
        raise ValueError(f"expected a {ndim}D array")
    return a


def _dp(a: np.ndarray):
    return a.ctypes.data_as(N._dp)


class Context:
    """One engine context (device buffers, streams) on one GPU."""

    def __init__(self, device: int = 0):
        self.lib = N.load()
        # ctypes releases the GIL during foreign calls; one context's arena, pinned staging and
        # streams must not be entered by two threads at once (semd_b200.h: one context per host
        # thread, or external locking). Every call on this context holds this lock.
        self.lock = threading.RLock()
        p = C.c_void_p()
        _check(self.lib, self.lib.semd_ctx_create(device, C.byref(p)))
        self.ptr = p
        self.device = device

    def close(self):
        if self.ptr:
            self.lib.semd_ctx_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int):
        _check(self.lib, rc)

    def call(self, name: str, *args) -> int:
        """lib.<name>(ctx, *args) under the context lock; returns the status code."""
        with self.lock:
            return getattr(self.lib, name)(self.ptr, *args)

    def run(self, name: str, *args) -> None:
        self.check(self.call(name, *args))

    # ---- multi-GPU (semd_comm_*): one context per rank, NCCL communicator ----
    @staticmethod
    def comm_unique_id() -> bytes:
        lib = N.load()
        buf = C.create_string_buffer(N.SEMD_COMM_ID_BYTES)
        _check(lib, lib.semd_comm_unique_id(buf, N.SEMD_COMM_ID_BYTES))
        return buf.raw

    def comm_init(self, uid: bytes, rank: int, world: int, root: int = -1) -> None:
        buf = C.create_string_buffer(bytes(uid), N.SEMD_COMM_ID_BYTES)
        self.run("semd_comm_init", buf, N.SEMD_COMM_ID_BYTES, int(rank), int(world))
        self.run("semd_comm_set_root", int(root))

    def comm_info(self) -> tuple[int, int]:
        r, w = C.c_int(), C.c_int()
        self.run("semd_comm_info", C.byref(r), C.byref(w))
        return r.value, w.value

    def comm_allreduce(self, vals, op: str = "sum") -> np.ndarray:
        a = np.array(vals, dtype=np.float64).ravel().copy()
        self.run("semd_comm_allreduce_host", _dp(a), a.size, 0 if op == "sum" else 1)
        return a

    def comm_destroy(self) -> None:
        self.run("semd_comm_destroy")

    def stats(self) -> dict:
        s = N.Stats()
        self.run("semd_get_stats", C.byref(s))
        return {f: getattr(s, f) for f, _ in N.Stats._fields_}

    def set_timing(self, on: bool):
        self.run("semd_set_timing", int(on))

    def set_max_slots(self, g: int):
        self.run("semd_set_max_slots", int(g))

    ENGINES = {"auto": 0, "lockstep": 1, "resident": 2}

    def set_engine(self, engine: str):
        """'auto' (default: the resident engine for signals of at most 8188 samples, the lockstep
        engine above), 'lockstep' or 'resident' (include/semd_b200.h semd_set_engine)."""
        if engine not in self.ENGINES:
            raise InvalidInput(f"unknown engine '{engine}' (expected auto, lockstep or resident)")
        self.run("semd_set_engine", self.ENGINES[engine])

    def set_stream(self, stream_ptr: int | None):
        self.run("semd_set_stream", C.c_void_p(stream_ptr or 0))

    def mt19937_64(self, seed: int, n: int) -> np.ndarray:
        """TEST HOOK: raw device std::mt19937_64 draws."""
        out = np.zeros(max(n, 1), dtype=np.uint64)
        self.run("semd_mt19937_64_device_test", C.c_uint64(seed), n,
                                                        out.ctypes.data_as(C.POINTER(C.c_uint64)))
        return out[:n]

    def set_noise_override(self, noise: np.ndarray | None):
        """TEST HOOK: use the given (nr, n) noise instead of the device RNG."""
        if noise is None:
            self.run("semd_set_noise_override", None, 0, 0)
            return
        w = _f64(noise, 2)
        self.run("semd_set_noise_override", _dp(w), w.shape[0], w.shape[1])


def context(device: int = 0) -> Context:
    with _ctx_lock:
        c = _ctxs.get(device)
        if c is None:
            c = Context(device)
            _ctxs[device] = c
        return c


def _cfgs(sd_threshold, max_sift_iters, max_imfs, nstd, nr, seed):
    return (N.SiftCfg(sd_threshold, max_sift_iters, max_imfs), N.EnsCfg(nstd, nr, 0, seed))


def parse_algorithm(name: str) -> int:
    """emd.cpp:346-354 ("emd", "eemd", "ceemdan"/"eemdan", case-insensitive)."""
    lib = N.load()
    out = C.c_int()
    _check(lib, lib.semd_parse_algorithm(name.encode(), C.byref(out)))
    return out.value


def _algo(algo) -> int:
    return parse_algorithm(algo) if isinstance(algo, str) else int(algo)


# --------------------------------------------------------------------- emd.hpp

def derive_seed(base: int, index: int) -> int:
    return N.load().semd_derive_seed(base, index)


def find_extrema(x, device: int = 0):
    """emd.cpp:10-35 -> (max_idx, max_val, min_idx, min_val)."""
    c = context(device)
    x = _f64(x, 1)
    n = x.size
    mi, ni = np.zeros(max(n, 1), np.uint64), np.zeros(max(n, 1), np.uint64)
    mv, nv = np.zeros(max(n, 1)), np.zeros(max(n, 1))
    a, b = C.c_size_t(), C.c_size_t()
    c.run("semd_find_extrema", _dp(x), n, mi.ctypes.data_as(N._szp), _dp(mv), C.byref(a),
                                    ni.ctypes.data_as(N._szp), _dp(nv), C.byref(b))
    return (mi[:a.value].astype(np.int64), mv[:a.value], ni[:b.value].astype(np.int64), nv[:b.value])


def envelope(idx, val, length: int, device: int = 0) -> np.ndarray:
    """emd.cpp:91-125."""
    c = context(device)
    i = np.ascontiguousarray(idx, dtype=np.uint64)
    v = _f64(val, 1)
    if i.size != v.size:
        raise InvalidInput("envelope: index/value size mismatch")
    out = np.zeros(length)
    c.run("semd_envelope", i.ctypes.data_as(N._szp), _dp(v), i.size, length, _dp(out))
    return out


def extract_imf(x, sd_threshold=0.2, max_sift_iters=300, max_imfs=0, device: int = 0):
    """emd.cpp:127-153 -> (imf, sift_count)."""
    c = context(device)
    x = _f64(x, 1)
    out = np.zeros(x.size)
    cnt = C.c_int32()
    cfg = N.SiftCfg(sd_threshold, max_sift_iters, max_imfs)
    c.run("semd_extract_imf", _dp(x), x.size, C.byref(cfg), _dp(out), C.byref(cnt))
    return out, cnt.value


def decompose_full(x, algo="emd", sd_threshold=0.2, max_sift_iters=300, max_imfs=0, nstd=0.2, nr=100, seed=0,
                   trace_cap: int = 0, device: int = 0):
    """decompose + per-IMF sift counts (EMD) + parity trace. Returns a dict."""
    c = context(device)
    x = _f64(x, 1)
    n = x.size
    a = _algo(algo)
    cfg, ens = _cfgs(sd_threshold, max_sift_iters, max_imfs, nstd, nr, seed)
    k_cap = max(8, max_imfs) if max_imfs else 32
    while True:
        imfs = np.zeros((k_cap, max(n, 1)))
        res = np.zeros(max(n, 1))
        counts = np.zeros(k_cap, np.int32)
        kout = C.c_size_t()
        trace_buf = (N.TraceRec * trace_cap)() if trace_cap else None
        tr = N.Trace(C.cast(trace_buf, C.c_void_p) if trace_cap else None, trace_cap, 0)
        rc = c.call("semd_decompose", a, _dp(x), n, C.byref(cfg), C.byref(ens), _dp(imfs), k_cap, C.byref(kout),
                                  _dp(res), counts.ctypes.data_as(N._i32p), C.byref(tr) if trace_cap else None)
        if rc == N.SEMD_CAPACITY and kout.value > k_cap:
            k_cap = int(kout.value)
            continue
        c.check(rc)
        break
    K = int(kout.value)
    out = {"imfs": imfs[:K, :n].copy(), "residue": res[:n].copy(), "sift_counts": counts[:K].copy()}
    if trace_cap:
        cnt = min(tr.count, trace_cap)
        arr = np.frombuffer(C.string_at(trace_buf, cnt * C.sizeof(N.TraceRec)),
                            dtype=np.dtype([("task", "<i4"), ("m", "<i4"), ("k", "<i4"), ("iter", "<i4"),
                                            ("n_max", "<u4"), ("n_min", "<u4"), ("hash", "<u8")])).copy()
        out["trace"] = arr
        out["trace_count"] = int(tr.count)
    out["stats"] = c.stats()
    return out


def decompose(x, algo="emd", sd_threshold=0.2, max_sift_iters=300, max_imfs=0, nstd=0.2, nr=100, seed=0):
    """module.cpp:108-122 / emd.cpp:365-373 -> {'imfs': (K, n), 'residue': (n,)}."""
    d = decompose_full(x, algo, sd_threshold, max_sift_iters, max_imfs, nstd, nr, seed)
    return {"imfs": d["imfs"], "residue": d["residue"]}


def emd(x, sd_threshold=0.2, max_sift_iters=300, max_imfs=0):
    return decompose(x, "emd", sd_threshold, max_sift_iters, max_imfs)


def eemd(x, sd_threshold=0.2, max_sift_iters=300, max_imfs=0, nstd=0.2, nr=100, seed=0):
    return decompose(x, "eemd", sd_threshold, max_sift_iters, max_imfs, nstd, nr, seed)


def ceemdan(x, sd_threshold=0.2, max_sift_iters=300, max_imfs=0, nstd=0.2, nr=100, seed=0):
    return decompose(x, "ceemdan", sd_threshold, max_sift_iters, max_imfs, nstd, nr, seed)


def white_noise(n: int, seed: int, std: float = 1.0, device: int = 0) -> np.ndarray:
    """emd.cpp:181-200 (mt19937_64 + Box-Muller on the GPU)."""
    c = context(device)
    out = np.zeros(max(n, 1))
    c.run("semd_white_noise", n, C.c_uint64(seed), std, _dp(out))
    return out[:n]


def noise_mode(w, i: int, sd_threshold=0.2, max_sift_iters=300, max_imfs=0, device: int = 0) -> np.ndarray:
    """emd.cpp:202-207."""
    c = context(device)
    w = _f64(w, 1)
    out = np.zeros(w.size)
    cfg = N.SiftCfg(sd_threshold, max_sift_iters, max_imfs)
    c.run("semd_noise_mode", _dp(w), w.size, i, C.byref(cfg), _dp(out))
    return out


def signal_std(x, device: int = 0) -> float:
    """emd.cpp:209-217."""
    c = context(device)
    x = _f64(x, 1)
    out = C.c_double()
    c.run("semd_signal_std", _dp(x), x.size, C.byref(out))
    return out.value


# --------------------------------------------------------------- serialize.hpp

def transition_weights(d: int, device: int = 0) -> np.ndarray:
    c = context(device)
    out = np.zeros(max(d, 1))
    c.run("semd_transition_weights", d, _dp(out))
    return out[:d]


def default_transition_length(rows: int) -> int:
    return N.load().semd_default_transition_length(rows)


def _channel_major(x) -> tuple[np.ndarray, int, int]:
    a = _f64(x, 2)  # (M samples, N channels), as module.cpp:23-32
    M, Nc = a.shape
    return np.ascontiguousarray(a.T), M, Nc


def concatenate(x, d: int, naive: bool = False, device: int = 0) -> np.ndarray:
    """serialize.cpp:30-50 (naive: :52-71). x is (M, N) samples x channels."""
    c = context(device)
    cm, M, Nc = _channel_major(x)
    L = M * Nc + d * (Nc - 1) if M and Nc else 0
    out = np.zeros(max(L, 1))
    c.run("semd_concatenate_naive" if naive else "semd_concatenate", _dp(cm), M, Nc, d, _dp(out))
    return out[:L]


def concatenate_naive(x, d: int, device: int = 0) -> np.ndarray:
    return concatenate(x, d, naive=True, device=device)


def deconcatenate(modes, rows: int, channels: int, d: int, device: int = 0) -> np.ndarray:
    """serialize.cpp:73-95. modes is (length, K) as module.cpp:159-172; returns (M, N, K)."""
    c = context(device)
    m = _f64(modes, 2)
    L, K = m.shape
    km = np.ascontiguousarray(m.T)
    out = np.zeros(max(K * rows * channels, 1))
    c.run("semd_deconcatenate", _dp(km), K, L, rows, channels, d, _dp(out))
    return out[:K * rows * channels].reshape(K, channels, rows).transpose(2, 1, 0).copy()


def serial_decompose_full(x, d: int, algo="emd", sd_threshold=0.2, max_sift_iters=300, max_imfs=0, nstd=0.2, nr=100,
                          seed=0, trace_cap: int = 0, device: int = 0):
    c = context(device)
    cm, M, Nc = _channel_major(x)
    a = _algo(algo)
    cfg, ens = _cfgs(sd_threshold, max_sift_iters, max_imfs, nstd, nr, seed)
    k_cap = (max_imfs + 1) if max_imfs else 33
    while True:
        t = np.zeros(max(k_cap * M * Nc, 1))
        mo = C.c_size_t()
        trace_buf = (N.TraceRec * trace_cap)() if trace_cap else None
        tr = N.Trace(C.cast(trace_buf, C.c_void_p) if trace_cap else None, trace_cap, 0)
        rc = c.call("semd_serial_decompose", a, _dp(cm), M, Nc, d, C.byref(cfg), C.byref(ens), _dp(t), k_cap,
                                         C.byref(mo), C.byref(tr) if trace_cap else None)
        if rc == N.SEMD_CAPACITY and mo.value > k_cap:
            k_cap = int(mo.value)
            continue
        c.check(rc)
        break
    K1 = int(mo.value)
    tensor = t[:K1 * M * Nc].reshape(K1, Nc, M).transpose(2, 1, 0).copy()
    return tensor, c.stats()


def serial_decompose(x, d: int, algo="emd", sd_threshold=0.2, max_sift_iters=300, max_imfs=0, nstd=0.2, nr=100,
                     seed=0):
    """serialize.cpp:97-105 / module.cpp:124-137 -> (M, N, K+1) tensor, residue last."""
    return serial_decompose_full(x, d, algo, sd_threshold, max_sift_iters, max_imfs, nstd, nr, seed)[0]


def slicewise_decompose(x, algo="emd", sd_threshold=0.2, max_sift_iters=300, max_imfs=0, nstd=0.2, nr=100, seed=0,
                        device: int = 0):
    """baseline.cpp:5-29: each channel of the (M, N) multi-signal decomposed independently; returns the
    (M, N, K) tensor (IMFs zero-padded to a common count, residue last). EMD / EEMD run every channel
    (x every realization) as one batched engine pass on the GPU."""
    c = context(device)
    cm, M, Nc = _channel_major(x)
    if M == 0 or Nc == 0:
        raise InvalidInput("slicewise_decompose: empty input")
    a = _algo(algo)
    cfg, ens = _cfgs(sd_threshold, max_sift_iters, max_imfs, nstd, nr, seed)
    k_cap = (max_imfs + 1) if max_imfs else 33
    while True:
        t = np.zeros(max(k_cap * M * Nc, 1))
        mo = C.c_size_t()
        rc = c.call("semd_slicewise_decompose", a, _dp(cm), M, Nc, C.byref(cfg), C.byref(ens), _dp(t), k_cap,
                                            C.byref(mo))
        if rc == N.SEMD_CAPACITY and mo.value > k_cap:
            k_cap = int(mo.value)
            continue
        c.check(rc)
        break
    K1 = int(mo.value)
    return t[:K1 * M * Nc].reshape(K1, Nc, M).transpose(2, 1, 0).copy()
