"""ctypes binding of the C ABI (include/semd_b200.h) -> libsemd_b200.so.

The shared library is built in-tree by csrc/build.py (sm_100a, nvcc). If it
is missing or no CUDA device is usable, calls fail loudly: there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# SEMD_LIB: an alternative in-tree build of the same library (A/B tuning runs)
LIB_PATH = os.environ.get("SEMD_LIB") or os.path.join(HERE, "libsemd_b200.so")

SEMD_OK = 0
SEMD_INVALID_INPUT = 1
SEMD_INSUFFICIENT_EXTREMA = 2
SEMD_CAPACITY = 3
SEMD_CUDA_ERROR = 4
SEMD_NO_MEMORY = 5
SEMD_COMM_ID_BYTES = 128

ALGOS = {"emd": 0, "eemd": 1, "ceemdan": 2}

_dp = C.POINTER(C.c_double)
_szp = C.POINTER(C.c_size_t)
_i32p = C.POINTER(C.c_int32)


class SiftCfg(C.Structure):
    """emd.hpp:10-18 SiftConfig."""
    _fields_ = [("sd_threshold", C.c_double), ("max_sift_iters", C.c_int32), ("max_imfs", C.c_int32)]


class EnsCfg(C.Structure):
    """emd.hpp:21-28 EnsembleConfig."""
    _fields_ = [("nstd", C.c_double), ("nr", C.c_int32), ("reserved", C.c_int32), ("base_seed", C.c_uint64)]


class TraceRec(C.Structure):
    _fields_ = [("task", C.c_int32), ("m", C.c_int32), ("k", C.c_int32), ("iter", C.c_int32),
                ("n_max", C.c_uint32), ("n_min", C.c_uint32), ("hash", C.c_uint64)]


class Trace(C.Structure):
    _fields_ = [("rec", C.c_void_p), ("cap", C.c_size_t), ("count", C.c_size_t)]


class Stats(C.Structure):
    _fields_ = [("sifted_samples", C.c_uint64), ("sift_iterations", C.c_uint64), ("steps", C.c_uint64),
                ("kernel_launches", C.c_uint64), ("solve_hazards", C.c_uint64), ("slots", C.c_int32),
                ("waves", C.c_int32), ("eval_ms", C.c_double), ("eval_launches", C.c_uint64),
                ("sd_rechecks", C.c_uint64), ("resident_jobs", C.c_uint64)]


# name -> (restype, argtypes); every symbol declared in include/semd_b200.h
SIGNATURES = {
    "semd_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "semd_ctx_destroy": (None, [C.c_void_p]),
    "semd_last_error": (C.c_char_p, []),
    "semd_get_stats": (C.c_int, [C.c_void_p, C.POINTER(Stats)]),
    "semd_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "semd_set_timing": (C.c_int, [C.c_void_p, C.c_int]),
    "semd_set_max_slots": (C.c_int, [C.c_void_p, C.c_int]),
    "semd_set_engine": (C.c_int, [C.c_void_p, C.c_int]),
    "semd_find_extrema": (C.c_int, [C.c_void_p, _dp, C.c_size_t, _szp, _dp, _szp, _szp, _dp, _szp]),
    "semd_envelope": (C.c_int, [C.c_void_p, _szp, _dp, C.c_size_t, C.c_size_t, _dp]),
    "semd_extract_imf": (C.c_int, [C.c_void_p, _dp, C.c_size_t, C.POINTER(SiftCfg), _dp, _i32p]),
    "semd_decompose": (C.c_int, [C.c_void_p, C.c_int, _dp, C.c_size_t, C.POINTER(SiftCfg), C.POINTER(EnsCfg), _dp,
                                 C.c_size_t, _szp, _dp, _i32p, C.POINTER(Trace)]),
    "semd_white_noise": (C.c_int, [C.c_void_p, C.c_size_t, C.c_uint64, C.c_double, _dp]),
    "semd_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "semd_noise_mode": (C.c_int, [C.c_void_p, _dp, C.c_size_t, C.c_size_t, C.POINTER(SiftCfg), _dp]),
    "semd_signal_std": (C.c_int, [C.c_void_p, _dp, C.c_size_t, _dp]),
    "semd_parse_algorithm": (C.c_int, [C.c_char_p, C.POINTER(C.c_int)]),
    "semd_transition_weights": (C.c_int, [C.c_void_p, C.c_size_t, _dp]),
    "semd_default_transition_length": (C.c_size_t, [C.c_size_t]),
    "semd_concatenate": (C.c_int, [C.c_void_p, _dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp]),
    "semd_concatenate_naive": (C.c_int, [C.c_void_p, _dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp]),
    "semd_deconcatenate": (C.c_int, [C.c_void_p, _dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                     _dp]),
    "semd_serial_decompose": (C.c_int, [C.c_void_p, C.c_int, _dp, C.c_size_t, C.c_size_t, C.c_size_t,
                                        C.POINTER(SiftCfg), C.POINTER(EnsCfg), _dp, C.c_size_t, _szp,
                                        C.POINTER(Trace)]),
    "semd_decompose_device": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t, C.POINTER(SiftCfg),
                                        C.POINTER(EnsCfg), C.c_void_p, C.c_size_t, _szp, C.c_void_p]),
    "semd_eemd_partial_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(SiftCfg), C.POINTER(EnsCfg),
                                           C.c_int32, C.c_int32, C.c_void_p, C.c_size_t, _szp]),
    "semd_eemd_partial_traced_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(SiftCfg),
                                                  C.POINTER(EnsCfg), C.c_int32, C.c_int32, C.c_void_p, C.c_size_t,
                                                  _szp, C.POINTER(Trace)]),
    "semd_ensemble_finish_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_int32,
                                              C.c_void_p]),
    "semd_concatenate_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_void_p]),
    "semd_deconcatenate_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                            C.c_size_t, C.c_void_p]),
    "semd_serial_decompose_device": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t,
                                               C.POINTER(SiftCfg), C.POINTER(EnsCfg), C.c_void_p, C.c_size_t,
                                               _szp]),
    "semd_slicewise_decompose": (C.c_int, [C.c_void_p, C.c_int, _dp, C.c_size_t, C.c_size_t, C.POINTER(SiftCfg),
                                           C.POINTER(EnsCfg), _dp, C.c_size_t, _szp]),
    "semd_slicewise_decompose_device": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_size_t, C.c_size_t,
                                                  C.POINTER(SiftCfg), C.POINTER(EnsCfg), C.c_void_p, C.c_size_t,
                                                  _szp]),
    "semd_serial_decompose_batch": (C.c_int, [C.c_void_p, C.c_int, _dp, C.c_size_t, C.c_size_t, C.c_size_t,
                                              C.c_size_t, C.POINTER(SiftCfg), C.POINTER(EnsCfg), _dp, C.c_size_t,
                                              _szp]),
    "semd_ceemdan_shard_begin": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(SiftCfg), C.POINTER(EnsCfg),
                                           C.c_int32, C.c_int32]),
    "semd_ceemdan_shard_residue_extrema": (C.c_int, [C.c_void_p, _szp]),
    "semd_ceemdan_shard_stage": (C.c_int, [C.c_void_p, C.c_void_p]),
    "semd_ceemdan_shard_finish_stage": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                                  C.POINTER(C.c_int32)]),
    "semd_ceemdan_shard_residue": (C.c_int, [C.c_void_p, C.c_void_p]),
    "semd_comm_unique_id": (C.c_int, [C.c_void_p, C.c_size_t]),
    "semd_comm_init": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int]),
    "semd_comm_set_root": (C.c_int, [C.c_void_p, C.c_int]),
    "semd_comm_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "semd_comm_allreduce_host": (C.c_int, [C.c_void_p, _dp, C.c_size_t, C.c_int]),
    "semd_comm_destroy": (C.c_int, [C.c_void_p]),
    "semd_device_alloc": (C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "semd_device_free": (C.c_int, [C.c_void_p, C.c_void_p]),
    "semd_host_alloc": (C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "semd_host_free": (C.c_int, [C.c_void_p, C.c_void_p]),
    "semd_memcpy": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]),
    "semd_timer_start": (C.c_int, [C.c_void_p]),
    "semd_timer_stop": (C.c_int, [C.c_void_p, _dp]),
}
# test-only hook (not part of the reference API)
EXTRA = {"semd_set_noise_override": (C.c_int, [C.c_void_p, _dp, C.c_size_t, C.c_size_t]),
         "semd_set_debug": (C.c_int, [C.c_void_p, C.c_int]),
         "semd_solve_profile": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
         "semd_resident_profile": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
         "semd_kernel_spans": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]),
         "semd_std_stats": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
         "semd_hazard_log": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]),
         "semd_mt19937_64_device_test": (C.c_int, [C.c_void_p, C.c_uint64, C.c_size_t, C.POINTER(C.c_uint64)])}

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libsemd_b200.so (building it first if the sources are newer)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path) or os.environ.get("SEMD_REBUILD"):
            from .csrc import build as _b
            _b.build()
        lib = C.CDLL(path)
        for name, (res, args) in {**SIGNATURES, **EXTRA}.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
        return lib
