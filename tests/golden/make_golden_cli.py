"""Golden outputs of the reference CLI's `decompose` (cli.cpp:93-134) for tests/test_cli.py, from
the REFERENCE ITSELF: oracle/_ref's ref_cli_decompose runs cli.cpp's steps over the reference's own
read_csv / read_pgm, serial_decompose, write_csv / write_pgm and nlohmann::json sidecar.

    python tests/golden/make_golden_cli.py      (build container only: needs oracle/_ref)
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cli.json")

# (input, algo, d, nstd, nr, seed, sd, iters, imfs)
CASES = [
    ("signals.csv", "emd", "50", 0.2, 100, 0, 0.2, 1000, 0),      # BASELINE config 1
    ("signals.csv", "eemd", "auto", 0.2, 20, 0, 0.2, 300, 10),    # config 2 shape, fewer realizations
    ("signals.csv", "ceemdan", "50", 0.2, 8, 3, 0.2, 300, 0),     # config 3 shape
    ("texture.pgm", "emd", "10", 0.2, 100, 0, 0.2, 300, 0),       # image input: CSV + PGM per mode
    ("texture.pgm", "eemd", "auto", 0.25, 6, 11, 0.2, 300, 0),
]
JSON_VALUES = [0.2, 0.25, 1.0, 0.0, 1e-5, 1e-4, 0.001, 123456789012.0, 1e15, 1e16, 2.5e-7, 1.0 / 3.0, 0.1, 100.0,
               6.02e23, 5e-324, 1.7976931348623157e308, 12.5, 0.30000000000000004]


def texture_image(rows: int = 40, cols: int = 48) -> np.ndarray:
    """A small deterministic 8-bit test image (gratings + a blob), as in BASELINE config 4."""
    y, x = np.mgrid[0:rows, 0:cols].astype(float)
    img = 128 + 50 * np.sin(2 * np.pi * x / 12.0) + 30 * np.cos(2 * np.pi * (x + y) / 5.0)
    img += 40 * np.exp(-((y - 15) ** 2 + (x - 30) ** 2) / 50.0)
    return np.clip(np.round(img), 0, 255).astype(np.uint8)


def write_pgm(path: str, img: np.ndarray) -> None:
    with open(path, "wb") as f:
        f.write(b"P5\n%d %d\n255\n" % (img.shape[1], img.shape[0]))
        f.write(img.tobytes())


def sha_file(path: str) -> str:
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


def make_inputs(d: str, ref_lib=None) -> dict:
    """signals.csv (the reference's synth signals) and texture.pgm into directory d."""
    if ref_lib is not None:
        assert ref_lib.ref_synth_signals_csv(C.c_size_t(1000), C.c_double(1000.0),
                                             os.path.join(d, "signals.csv").encode()) == 0
    write_pgm(os.path.join(d, "texture.pgm"), texture_image())
    return {f: sha_file(os.path.join(d, f)) for f in ("signals.csv", "texture.pgm") if os.path.exists(os.path.join(d, f))}


def main() -> None:
    from oracle.ffi import REF_SO
    lib = C.CDLL(REF_SO)
    lib.ref_cli_decompose.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_double, C.c_int, C.c_uint64, C.c_double,
                                      C.c_int, C.c_int, C.c_char_p]
    lib.ref_last_error.restype = C.c_char_p
    out = {"inputs": {}, "cases": [], "json_double": []}
    with tempfile.TemporaryDirectory() as d:
        out["inputs"] = make_inputs(d, lib)
        for i, (inp, algo, dflag, nstd, nr, seed, sd, iters, imfs) in enumerate(CASES):
            od = os.path.join(d, f"out{i}")
            rc = lib.ref_cli_decompose(os.path.join(d, inp).encode(), algo.encode(), dflag.encode(), nstd, nr, seed, sd,
                                       iters, imfs, od.encode())
            assert rc == 0, lib.ref_last_error()
            files = {f: sha_file(os.path.join(od, f)) for f in sorted(os.listdir(od))}
            out["cases"].append({"input": inp, "args": {"algo": algo, "d": dflag, "nstd": nstd, "nr": nr, "seed": seed,
                                                        "sd-threshold": sd, "max-sift-iters": iters, "max-imfs": imfs},
                                 "files": files,
                                 "sidecar": open(os.path.join(od, os.path.splitext(inp)[0] + "_decomposition.json")).read()})
    buf = C.create_string_buffer(64)
    for v in JSON_VALUES:
        assert lib.ref_json_double(C.c_double(v), buf, 64) == 0
        out["json_double"].append([v.hex(), buf.value.decode()])
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", OUT, [len(c["files"]) for c in out["cases"]])


if __name__ == "__main__":
    main()
