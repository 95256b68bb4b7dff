"""Full-size parity of the headline configs (BASELINE.json configs[3] = C4, configs[4] = C5) against
the REFERENCE ITSELF with its own noise: tests/golden/ensembles.{npz,json}, written by
tests/golden/make_golden_ensembles.py from oracle/_ref (the reference built from its sources).

Per realization m (x + beta * white_noise(L, derive_seed(0, m)), emd.cpp:237-244) the engine must
reproduce the reference's IMF count, every IMF's sift count, every find_extrema record (extrema
counts + hash of both index lists) and the IMF values: all 100 C4 realizations and 64 C5 ones
(m = 0..31 and 32 spread over 40..999, including 793). The device draws its own noise
(mt19937_64 + the glibc log/sincos restatement), so this checks the noise stream too. The whole
ensembles (C4 NR=100, C5 NR=1000: realization-ordered sums, emd.cpp:246-261) must be identical
to the reference's eemd() down to the sha256 of the IMF and residue arrays.
"""
import ctypes as C
import hashlib
import json
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

REL_L2 = 1e-9


@pytest.fixture(scope="module")
def eg():
    npz = os.path.join(GOLDEN, "ensembles.npz")
    arrs = dict(np.load(npz))
    meta = json.load(open(os.path.join(GOLDEN, "ensembles.json")))
    return arrs, meta


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def serialized(se, key, meta_entry):
    from paper_2106_15319_b200 import workloads as W
    s = se.concatenate(W.config_input(key), W.CONFIGS[key]["D"])
    assert s.size == meta_entry["L"]
    assert sha(s) == meta_entry["input_sha256"], "synthetic input differs from the one the goldens were made on"
    return s


def run_realization(se, d_x, n, m, k_cap, trace_cap=2000):
    """Realization m alone through semd_eemd_partial_traced_device: its IMFs (unscaled sum of one)
    on the device, K and its trace records."""
    import torch

    from paper_2106_15319_b200 import _native as N
    c = se.context(0)
    sums = torch.empty((k_cap, n), dtype=torch.float64, device="cuda")
    buf = (N.TraceRec * trace_cap)()
    tr = N.Trace(C.cast(buf, C.c_void_p), trace_cap, 0)
    k = C.c_size_t()
    c.run("semd_eemd_partial_traced_device", C.c_void_p(d_x.data_ptr()), n, C.byref(N.SiftCfg(0.2, 300, 0)),
          C.byref(N.EnsCfg(0.2, 1000, 0, 0)), m, m + 1, C.c_void_p(sums.data_ptr()), k_cap, C.byref(k),
          C.byref(tr))
    assert tr.count <= trace_cap
    rec = np.frombuffer(C.string_at(buf, tr.count * C.sizeof(N.TraceRec)),
                        dtype=[("task", "<i4"), ("m", "<i4"), ("k", "<i4"), ("iter", "<i4"), ("n_max", "<u4"),
                               ("n_min", "<u4"), ("hash", "<u8")]).copy()
    return sums[:k.value], rec


def check_realizations(se, key, eg, ms_subset=None):
    import torch
    arrs, meta = eg
    ent = meta[f"{key}_realizations"]
    s = serialized(se, key, ent)
    d_x = torch.from_numpy(s).cuda()
    ms = arrs[f"{key}_real_m"].tolist()
    Ks = arrs[f"{key}_real_K"]
    off_k = np.concatenate([[0], np.cumsum(Ks)])
    tr_all = arrs[f"{key}_real_trace"]
    idx = torch.from_numpy(arrs[f"{key}_real_sample_idx"].astype(np.int64)).cuda()
    bad = []
    for j, m in enumerate(ms):
        if ms_subset is not None and m not in ms_subset:
            continue
        imfs, rec = run_realization(se, d_x, s.size, m, 40)
        K = int(Ks[j])
        gold_tr = np.sort(tr_all[tr_all["m"] == m], order=["k", "iter"])
        got_tr = np.sort(rec, order=["k", "iter"])
        counts = arrs[f"{key}_real_counts"][off_k[j]:off_k[j + 1]]
        ok_rows = (got_tr["n_max"] >= 2) & (got_tr["n_min"] >= 2)
        got_counts = [int((ok_rows & (got_tr["k"] == k)).sum()) for k in range(imfs.shape[0])]
        norms = torch.linalg.norm(imfs, dim=1).cpu().numpy()
        samples = imfs[:, idx].cpu().numpy()
        gold_norms = arrs[f"{key}_real_norms"][off_k[j]:off_k[j + 1]]
        gold_samples = arrs[f"{key}_real_samples"][off_k[j]:off_k[j + 1]]
        why = []
        if imfs.shape[0] != K:
            why.append(f"K {imfs.shape[0]} != {K}")
        else:
            if got_counts != counts.tolist():
                why.append("sift counts")
            if not np.array_equal(got_tr, gold_tr):
                why.append("trace")
            if np.max(np.abs(norms - gold_norms) / gold_norms) > REL_L2:
                why.append("norms")
            if not np.array_equal(samples, gold_samples):  # identical noise -> identical IMF values
                why.append(f"samples (max rel {np.max(np.abs(samples - gold_samples)) / np.max(gold_norms):.2e})")
        if why:
            bad.append((m, why))
    assert not bad, f"{len(bad)} mismatching {key} realizations: {bad[:8]}"


def test_c4_all_realizations_vs_reference(se, eg):
    check_realizations(se, "c4", eg)


def test_c5_64_realizations_vs_reference(se, eg):
    check_realizations(se, "c5", eg)


def _ensemble(se, key, eg):
    import torch

    from paper_2106_15319_b200 import _native as N
    from paper_2106_15319_b200 import workloads as W
    arrs, meta = eg
    ent = meta.get(f"{key}_ensemble")
    if ent is None:
        pytest.skip(f"no {key} ensemble golden committed")
    s = serialized(se, key, ent)
    cfg = W.CONFIGS[key]
    c = se.context(0)
    d_x = torch.from_numpy(s).cuda()
    k_cap = 40
    imfs = torch.empty((k_cap, s.size), dtype=torch.float64, device="cuda")
    res = torch.empty(s.size, dtype=torch.float64, device="cuda")
    k = C.c_size_t()
    c.run("semd_decompose_device", 1, C.c_void_p(d_x.data_ptr()), s.size,
          C.byref(N.SiftCfg(0.2, cfg["max_sift_iters"], cfg["max_imfs"])), C.byref(N.EnsCfg(0.2, cfg["nr"], 0, 0)),
          C.c_void_p(imfs.data_ptr()), k_cap, C.byref(k), C.c_void_p(res.data_ptr()))
    K = int(k.value)
    assert K == ent["K"]
    hi, hr = imfs[:K].cpu().numpy(), res.cpu().numpy()
    idx = arrs[f"{key}_ens_sample_idx"].astype(np.int64)
    norms = np.sqrt((hi ** 2).sum(axis=1))
    assert np.max(np.abs(norms - arrs[f"{key}_ens_norms"]) / arrs[f"{key}_ens_norms"]) <= REL_L2
    assert np.array_equal(hi[:, idx], arrs[f"{key}_ens_samples"])
    assert np.array_equal(hr[idx], arrs[f"{key}_ens_residue_samples"])
    assert sha(hi) == ent["imfs_sha256"] and sha(hr) == ent["residue_sha256"], "ensemble not bit-identical"


def test_c4_ensemble_bit_identical_to_reference(se, eg):
    _ensemble(se, "c4", eg)


def test_c5_ensemble_bit_identical_to_reference(se, eg):
    _ensemble(se, "c5", eg)
