"""Full-size ensemble goldens for C4 and C5 (BASELINE.json configs[3], configs[4]) from the
REFERENCE ITSELF, with the reference's own noise (glibc Box-Muller, emd.cpp:181-200).

Runs only in the build container (oracle/_ref/libsemd_ref.so compiled from /root/reference):

    python tests/golden/make_golden_ensembles.py realizations   # C4 m=0..99, C5 64 realizations
    python tests/golden/make_golden_ensembles.py c4-ensemble    # the whole C4 eemd() (NR=100)
    python tests/golden/make_golden_ensembles.py c5-ensemble    # the whole C5 eemd() (NR=1000, ~1 h on 6 cores)

Per realization m (w = white_noise(L, derive_seed(0, m)), x_m = x + beta*w, emd(x_m)) it records,
through the replayer in oracle/ref_shim.cpp: K_m, the sift count of every IMF, the parity trace
(one record per find_extrema call: extrema counts + order-sensitive hash of both index lists),
each IMF's L2 norm, and each IMF's values at fixed sample indices. A subset is also checked
bit-for-bit against the unmodified semd::emd. The whole ensembles come from ref_eemd_stream,
semd::eemd with its NR x K x L store replaced by in-order accumulation (bit-identical to
eemd(); tested against it on C2). Everything lands in tests/golden/ensembles.npz (+ .json).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

OUT = os.path.dirname(os.path.abspath(__file__))
NPZ = os.path.join(OUT, "ensembles.npz")
JSN = os.path.join(OUT, "ensembles.json")
WORKERS = int(os.environ.get("GOLDEN_WORKERS", "6"))

# realization sets (VERDICT r1 "next round" #1): all 100 C4 realizations; C5 m=0..31 plus 32
# spread over [32, 999] including 793 (the realization that ran away under a 1-ulp beta change)
C4_MS = list(range(100))
C5_MS = sorted(set(range(32)) | {793, 999} | set(int(v) for v in np.linspace(40, 990, 30).round()))
CHECK_MS = {0, 1, 793}  # also bit-compared with the unmodified semd::emd
N_SAMPLES_REAL = 64
N_SAMPLES_ENS = 1024


def serialized(key: str) -> np.ndarray:
    from oracle.ffi import Ref
    from paper_2106_15319_b200 import workloads as W
    x = W.config_input(key)
    M, N = x.shape
    return Ref().concatenate(np.ascontiguousarray(x.T), M, N, W.CONFIGS[key]["D"])


def sample_idx(L: int, n: int, seed: int) -> np.ndarray:
    return np.unique(np.random.default_rng(seed).integers(0, L, size=n)).astype(np.uint64)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


_S = {}


def _one(args):
    key, m = args
    from oracle.ffi import Ref
    if key not in _S:
        _S[key] = serialized(key)
    s = _S[key]
    t0 = time.time()
    counts, trace, norms, samples = Ref().realization_summary(s, m, sample_idx(s.size, N_SAMPLES_REAL, 7),
                                                              check=m in CHECK_MS)
    return key, m, counts, trace, norms, samples, time.time() - t0


def load() -> tuple[dict, dict]:
    arrs = dict(np.load(NPZ)) if os.path.exists(NPZ) else {}
    meta = json.load(open(JSN)) if os.path.exists(JSN) else {}
    return arrs, meta


def save(arrs: dict, meta: dict) -> None:
    np.savez_compressed(NPZ, **arrs)
    with open(JSN, "w") as f:
        json.dump(meta, f, indent=1)


def realizations() -> None:
    arrs, meta = load()
    jobs = [("c5", m) for m in C5_MS] + [("c4", m) for m in C4_MS]
    res = {"c4": {}, "c5": {}}
    with Pool(WORKERS) as p:
        for key, m, counts, trace, norms, samples, dt in p.imap_unordered(_one, jobs):
            res[key][m] = (counts, trace, norms, samples)
            print(f"{key} m={m} K={len(counts)} sifts={int(counts.sum())} {dt:.1f}s", flush=True)
    for key, ms in (("c4", C4_MS), ("c5", C5_MS)):
        s = serialized(key)
        ks = np.array([len(res[key][m][0]) for m in ms], np.int32)
        arrs[f"{key}_real_m"] = np.array(ms, np.int32)
        arrs[f"{key}_real_K"] = ks
        arrs[f"{key}_real_counts"] = np.concatenate([res[key][m][0] for m in ms]).astype(np.int32)
        arrs[f"{key}_real_trace"] = np.concatenate([res[key][m][1] for m in ms])
        arrs[f"{key}_real_norms"] = np.concatenate([res[key][m][2] for m in ms])
        arrs[f"{key}_real_samples"] = np.concatenate([res[key][m][3] for m in ms], axis=0)
        arrs[f"{key}_real_sample_idx"] = sample_idx(s.size, N_SAMPLES_REAL, 7)
        meta[f"{key}_realizations"] = {
            "L": int(s.size), "input_sha256": sha(s), "ms": ms, "checked_against_semd_emd": sorted(CHECK_MS & set(ms)),
            "sifted_samples": int(s.size) * int(arrs[f"{key}_real_counts"].sum()),
            "note": "per-realization emd() of x + beta*white_noise(L, derive_seed(0, m)), reference noise"}
    save(arrs, meta)


def ensemble(key: str) -> None:
    from oracle.ffi import Ref
    from paper_2106_15319_b200 import workloads as W
    c = W.CONFIGS[key]
    s = serialized(key)
    t0 = time.time()
    imfs, res, kper = Ref().eemd_stream(s, WORKERS, iters=c["max_sift_iters"], imfs=c["max_imfs"], nr=c["nr"])
    dt = time.time() - t0
    arrs, meta = load()
    idx = sample_idx(s.size, N_SAMPLES_ENS, 11)
    arrs[f"{key}_ens_sample_idx"] = idx
    arrs[f"{key}_ens_samples"] = imfs[:, idx.astype(np.int64)]
    arrs[f"{key}_ens_residue_samples"] = res[idx.astype(np.int64)]
    arrs[f"{key}_ens_norms"] = np.sqrt((imfs ** 2).sum(axis=1))
    arrs[f"{key}_ens_K_per_realization"] = kper.astype(np.int32)
    meta[f"{key}_ensemble"] = {"L": int(s.size), "input_sha256": sha(s), "NR": c["nr"], "K": int(imfs.shape[0]),
                               "imfs_sha256": sha(imfs), "residue_sha256": sha(res), "seconds": round(dt, 1),
                               "workers": WORKERS,
                               "note": "semd::eemd semantics (realization-ordered sums), reference noise"}
    save(arrs, meta)
    print(key, "K", imfs.shape[0], "seconds", round(dt, 1))


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "realizations"
    if what == "realizations":
        realizations()
    elif what == "c4-ensemble":
        ensemble("c4")
    elif what == "c5-ensemble":
        ensemble("c5")
    else:
        raise SystemExit(__doc__)
