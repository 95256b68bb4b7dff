"""build_feature_bank (recognition.cpp:281-298) over the GPU: the C++ mirror (include/semd/
recognition.hpp) decomposes every image of the set in ONE batched engine pass
(semd_serial_decompose_batch); the banked features must be bit-identical to the reference's own
build_feature_bank (tests/golden/bank.json, from oracle/_ref), with and without speckle, for EMD,
EEMD and CEEMDAN, on the reference test's synthetic faces and on 112x92 images."""
import hashlib
import json
import math
import os
import subprocess

import numpy as np
import pytest

from tests.conftest import GOLDEN, ROOT
from tests.golden.make_golden_bank import inputs


def _build(tmp_path):
    from paper_2106_15319_b200 import _native
    exe = str(tmp_path / "feature_bank")
    libdir = os.path.dirname(_native.LIB_PATH)
    r = subprocess.run(["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "feature_bank.cpp"), "-o", exe, "-L" + libdir,
                        "-lsemd_b200", "-Wl,-rpath," + libdir], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_feature_bank_mirror_compiles(tmp_path):
    _build(tmp_path)


@pytest.mark.gpu
def test_feature_bank_bit_identical_to_reference(se, tmp_path):
    exe = _build(tmp_path)
    for case in json.load(open(os.path.join(GOLDEN, "bank.json"))):
        imgs = np.ascontiguousarray(inputs(case["images"]), dtype=np.float64)
        assert hashlib.sha256(imgs.astype("<f8").tobytes()).hexdigest() == case["input_sha256"]
        B, rows, cols = imgs.shape
        fin, fout = tmp_path / "in.bin", tmp_path / "out.bin"
        imgs.tofile(fin)
        snr = "inf" if case["snr_db"] is None else repr(case["snr_db"])
        argv = [exe, fin, fout, B, rows, cols, case["algo"], case["d"], repr(case["nstd"]), case["nr"], case["seed"],
                snr, case["speckle_seed"], case["target"]]
        r = subprocess.run(list(map(str, argv)), capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        feats = np.fromfile(fout, dtype="<f8")
        assert [float(v).hex() for v in feats.reshape(B, case["target"], -1)[0, -1, :8]] == case["features_head"]
        assert hashlib.sha256(feats.tobytes()).hexdigest() == case["features_sha256"], case
