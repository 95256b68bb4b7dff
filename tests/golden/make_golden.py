"""Generate the golden vectors in tests/golden/ from the REFERENCE ITSELF.

Runs only in the build container, where /root/reference exists and
oracle/Makefile has compiled it into oracle/_ref/libsemd_ref.so. Every value
written here comes from the unmodified reference library (or the reference's
public find_extrema/envelope driven by the trace replayer in
oracle/ref_shim.cpp, which checks itself bit-for-bit against semd::emd).

    python tests/golden/make_golden.py

The reference ships no golden files; its unit-test inputs are
reproduced from their definitions (test_emd.cpp, test_serialize.cpp,
test_helpers.hpp TestRng) and its known answers are recorded as computed.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.ffi import Ref  # noqa: E402
from tests.golden.inputs import (C_CONFIGS, kat_envelope_cases, kat_extrema_cases, rng_signal,  # noqa: E402
                                 pickup_serialized)

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def hexs(a) -> list[str]:
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).ravel()]


def main() -> None:
    r = Ref()
    kat: dict = {}
    kat["derive_seed"] = [[b, i, r.derive_seed(b, i)] for b, i in [(0, 0), (0, 1), (1, 0), (42, 7), (5000, 99)]]
    kat["mt19937_64_default_10000th"] = int(r.mt19937_64(5489, 10000)[-1])
    kat["mt19937_64_seed_first"] = {str(s): [int(v) for v in r.mt19937_64(s, 8)]
                                    for s in (r.derive_seed(0, 0), 7, 0)}
    kat["mt19937_64_seed7_sha_first_4096"] = hashlib.sha256(r.mt19937_64(7, 4096).astype("<u8").tobytes()).hexdigest()
    kat["white_noise_4_seed_ds00"] = hexs(r.white_noise(4, r.derive_seed(0, 0)))
    wn = r.white_noise(1001, 7)
    kat["white_noise_1001_seed7"] = {"sha256": sha(wn), "head": hexs(wn[:16]), "tail": hexs(wn[-3:])}
    kat["white_noise_std0"] = hexs(r.white_noise(5, 42, 0.0))

    ext = []
    for name, x in kat_extrema_cases():
        mi, mv, ni, nv = r.find_extrema(x)
        ext.append({"name": name, "x": hexs(x), "max_idx": mi.tolist(), "max_val": hexs(mv),
                    "min_idx": ni.tolist(), "min_val": hexs(nv)})
    kat["find_extrema"] = ext
    env = []
    for name, idx, val, length in kat_envelope_cases(r):
        env.append({"name": name, "idx": [int(v) for v in idx], "val": hexs(val), "length": length,
                    "out": hexs(r.envelope(idx, val, length))})
    kat["envelope"] = env
    kat["default_transition_length"] = [[m, r.default_transition_length(m)] for m in (1000, 112, 92, 4, 2, 1, 3)]
    kat["concat_hand"] = hexs(r.concatenate(np.array([[0.0, 3.0], [6.0, 9.0]]), 2, 2, 2))

    # random-signal EMD cases: TestRng seeds/lengths of test_emd.cpp
    rnd = []
    for seed, n, imfs in [(11, 600, 0), (12, 500, 2), (21, 400, 0), (23, 400, 0), (31, 37, 0), (99, 4, 0),
                          (98, 5, 0), (97, 64, 0)]:
        x = rng_signal(seed, n)
        imf, res, counts, trace = r.emd_traced(x, imfs=imfs)
        rnd.append({"seed": seed, "n": n, "max_imfs": imfs, "K": int(imf.shape[0]), "counts": counts.tolist(),
                    "imfs_sha256": sha(imf), "residue_sha256": sha(res),
                    "trace": [[int(t[k]) for k in ("k", "iter", "n_max", "n_min", "hash")] for t in trace]})
    kat["emd_random"] = rnd

    # small ensembles (test_emd.cpp:281-293, :330-343)
    ens = []
    for algo, seed, n, nr in [(1, 22, 300, 10), (2, 24, 300, 8), (1, 21, 400, 3), (2, 23, 200, 5)]:
        x = rng_signal(seed, n)
        imf, res = r.decompose(x, algo, nr=nr)
        ens.append({"algo": algo, "seed": seed, "n": n, "nr": nr, "K": int(imf.shape[0]),
                    "imfs_sha256": sha(imf), "residue_sha256": sha(res),
                    "imf_norms": hexs(np.sqrt((imf ** 2).sum(axis=1)))})
    kat["ensembles_small"] = ens

    # BASELINE configs 1-3
    cfgs = {}
    traces = {}
    for name, c in C_CONFIGS.items():
        s = pickup_serialized(r, c["D"])
        ent = {"L": int(s.size), "input_sha256": sha(s), **{k: v for k, v in c.items()}}
        if c["algo"] == 0:
            imf, res, counts, trace = r.emd_traced(s, iters=c["iters"], imfs=c["imfs"])
            ent.update(K=int(imf.shape[0]), counts=counts.tolist(), imfs_sha256=sha(imf), residue_sha256=sha(res))
        elif c["algo"] == 1:
            sums, kc, trace = r.eemd_traced(s, 0, c["nr"], iters=c["iters"], imfs=c["imfs"], nr=c["nr"])
            imf, res = r.decompose(s, 1, iters=c["iters"], imfs=c["imfs"], nr=c["nr"])
            ent.update(K=int(imf.shape[0]), realization_counts=kc.tolist(), imfs_sha256=sha(imf),
                       residue_sha256=sha(res), imf_norms=hexs(np.sqrt((imf ** 2).sum(axis=1))))
        else:
            imf, res, trace = r.ceemdan_traced(s, iters=c["iters"], imfs=c["imfs"], nr=c["nr"])
            ent.update(K=int(imf.shape[0]), imfs_sha256=sha(imf), residue_sha256=sha(res),
                       imf_norms=hexs(np.sqrt((imf ** 2).sum(axis=1))))
        if trace is not None:
            traces[name] = trace
            ent["sifted_samples"] = int(s.size) * int((trace["iter"] >= 0).sum() - count_failed(trace))
        cfgs[name] = ent
    kat["configs"] = cfgs

    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(kat, f, indent=1)
    np.savez_compressed(os.path.join(OUT, "traces.npz"), **traces)
    print("wrote", os.path.join(OUT, "golden.json"), "and traces.npz:", {k: len(v) for k, v in traces.items()})


def count_failed(trace) -> int:
    """find_extrema calls that did not lead to a subtraction: insufficient extrema, or CEEMDAN stage checks."""
    return int((((trace["n_max"] < 2) | (trace["n_min"] < 2)) | (trace["task"] == 3)).sum())


if __name__ == "__main__":
    main()
