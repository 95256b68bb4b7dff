"""Golden feature banks (recognition.cpp:281-298 build_feature_bank) from the REFERENCE ITSELF
(oracle/_ref ref_feature_bank) for tests/test_feature_bank.py.

    python tests/golden/make_golden_bank.py      (build container only)

Inputs: the reference test's synthetic_faces clusters (test_recognition.cpp:30-47, 16x12) and six
112x92 images of BASELINE config 4's generator (the face database itself is not in the image).
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "bank.json")

# (images, algo, d, nstd, nr, seed, snr_db, speckle_seed, target)
CASES = [
    ("synthetic_faces", 0, 3, 0.2, 100, 0, math.inf, 0, 10),
    ("synthetic_faces", 1, 4, 0.2, 8, 5, -6.0, 77, 10),
    ("synthetic_faces", 2, 3, 0.2, 4, 1, -6.0, 9, 6),
    ("images112x92", 0, 20, 0.2, 100, 0, -6.0, 0xFACE, 10),
    ("images112x92", 1, 20, 0.2, 6, 0, math.inf, 0, 10),
]


def synthetic_faces(subjects: int = 3, per_subject: int = 4) -> np.ndarray:
    """test_recognition.cpp:30-47 (TestRng, 16 x 12 images, subject-level offsets)."""
    from tests.golden.inputs import TestRng
    two_pi = 6.283185307179586476925286766559
    out = []
    for s in range(1, subjects + 1):
        for p in range(per_subject):
            rng = TestRng(1000 * s + p)
            img = np.empty((16, 12))
            for r in range(16):
                for c in range(12):
                    img[r, c] = 10.0 * s + math.sin(two_pi * float(r * 12 + c) / 16.0) + 0.01 * rng.uniform()
            out.append(img)
    return np.stack(out)


def images112x92() -> np.ndarray:
    from paper_2106_15319_b200 import workloads as W
    b = W.image_batch(n_images=6)  # (92, 112*6): channel (image, row) = 92 pixels
    return np.ascontiguousarray(b.T.reshape(6, 112, 92))


def inputs(name: str) -> np.ndarray:
    return synthetic_faces() if name == "synthetic_faces" else images112x92()


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def main() -> None:
    from oracle.ffi import REF_SO
    lib = C.CDLL(REF_SO)
    lib.ref_feature_bank.argtypes = [C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, C.c_size_t, C.c_double,
                                     C.c_int, C.c_uint64, C.c_double, C.c_uint64, C.c_size_t, C.c_void_p]
    lib.ref_last_error.restype = C.c_char_p
    out = []
    for name, algo, d, nstd, nr, seed, snr, sseed, target in CASES:
        imgs = np.ascontiguousarray(inputs(name), dtype=np.float64)
        B, rows, cols = imgs.shape
        feats = np.zeros((B, target, rows * cols))
        rc = lib.ref_feature_bank(imgs.ctypes.data, B, rows, cols, algo, d, nstd, nr, seed, snr, sseed, target,
                                  feats.ctypes.data)
        assert rc == 0, lib.ref_last_error()
        out.append({"images": name, "input_sha256": sha(imgs), "algo": algo, "d": d, "nstd": nstd, "nr": nr,
                    "seed": seed, "snr_db": None if math.isinf(snr) else snr, "speckle_seed": sseed, "target": target,
                    "features_sha256": sha(feats), "features_head": [float(v).hex() for v in feats[0, -1, :8]]})
        print(name, algo, "B", B, "ok")
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
