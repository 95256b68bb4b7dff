"""The C-ABI library: builds for sm_100a, loads, exports every symbol that
include/semd_b200.h declares, and fails loudly (no CPU fallback) where no GPU
is present. No GPU compute here."""
import ctypes as C
import os
import re
import subprocess

import pytest

from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "semd_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(semd_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2106_15319_b200 import _native
    return _native.load()


def test_every_declared_symbol_is_exported(lib):
    from paper_2106_15319_b200 import _native
    names = declared()
    assert len(names) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (semd_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(names) <= set(_native.SIGNATURES), "ctypes binding misses a declared symbol"
    for n in names:
        getattr(lib, n)


def test_library_is_sm100a(lib):
    from paper_2106_15319_b200 import _native
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_pure_functions_match_oracle(lib, oracle):
    for b, i in [(0, 0), (0, 1), (123, 456), (2**63, 7)]:
        assert lib.semd_derive_seed(b, i) == oracle.derive_seed(b, i)
    for m in (1000, 112, 92, 4, 2, 1, 3, 0):
        assert lib.semd_default_transition_length(m) == (oracle.default_transition_length(m) if m else 0)
    a = C.c_int()
    for name, v in [("emd", 0), ("EEMD", 1), ("ceemdan", 2), ("eemdan", 2)]:
        assert lib.semd_parse_algorithm(name.encode(), C.byref(a)) == 0 and a.value == v
    assert lib.semd_parse_algorithm(b"vmd", C.byref(a)) == 1
    assert lib.semd_last_error() == b"unknown algorithm 'vmd' (expected emd, eemd, or ceemdan)"


def test_context_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    p = C.c_void_p()
    rc = lib.semd_ctx_create(0, C.byref(p))
    assert rc == 4  # SEMD_CUDA_ERROR: no CPU fallback
    assert b"no CPU fallback" in lib.semd_last_error()
    import paper_2106_15319_b200 as se
    with pytest.raises(se.EngineError):
        se.decompose([1.0, 2.0, 3.0, 4.0, 5.0])


def test_cpp_mirror_compiles():
    """include/semd/*.hpp (the reference-signature C++ API) compiles against the C ABI."""
    src = os.path.join(ROOT, "tests", "cpp", "test_semd_cpp.cpp")
    out = "/tmp/test_semd_cpp.o"
    r = subprocess.run(["g++", "-std=c++20", "-c", "-I" + os.path.join(ROOT, "include"), src, "-o", out],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
