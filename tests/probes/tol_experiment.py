"""Experiment: a tolerance-mode spline (reciprocal multiplications + FMAs instead of the
correctly rounded divisions; build with -DSEMD_TOL_SPLINE, select with SEMD_LIB) against the reference goldens.

    python tests/probes/tol_experiment.py real  c4|c5        per-realization K / sift counts / traces / values
    python tests/probes/tol_experiment.py dump  c4|c5 out    whole ensemble with every realization's trace -> out.npz/.npy
    python tests/probes/tol_experiment.py cmp   a b          two dumps: traces equal? per-IMF rel-L2
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

DT = [("task", "<i4"), ("m", "<i4"), ("k", "<i4"), ("iter", "<i4"), ("n_max", "<u4"), ("n_min", "<u4"), ("hash", "<u8")]
mode = sys.argv[1]

if mode == "cmp":
    a, b = sys.argv[2], sys.argv[3]
    ta, tb = np.load(a + ".npz")["trace"], np.load(b + ".npz")["trace"]
    key = ["m", "k", "iter"]
    ta, tb = np.sort(ta, order=key), np.sort(tb, order=key)
    print("records", ta.size, tb.size)
    ms = sorted(set(ta["m"].tolist()) | set(tb["m"].tolist()))
    diff = [m for m in ms if not np.array_equal(ta[ta["m"] == m], tb[tb["m"] == m])]
    print("realizations with a differing trace: %d of %d" % (len(diff), len(ms)), diff[:40])
    for m in diff[:6]:
        x, y = ta[ta["m"] == m], tb[tb["m"] == m]
        n = min(x.size, y.size)
        j = next((i for i in range(n) if x[i] != y[i]), n)
        print("  m", m, "records", x.size, y.size, "first difference at", j, x[j] if j < x.size else None, y[j] if j < y.size else None)
    ia, ib = np.load(a + ".npy", mmap_mode="r"), np.load(b + ".npy", mmap_mode="r")
    print("K", ia.shape[0], ib.shape[0])
    for k in range(min(ia.shape[0], ib.shape[0])):
        d = np.linalg.norm(np.asarray(ia[k]) - np.asarray(ib[k]))
        print("  mode %2d rel-L2 %.3e" % (k, d / max(np.linalg.norm(np.asarray(ia[k])), 1e-300)))
    sys.exit(0)

import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import _native as N
from paper_2106_15319_b200 import workloads as W

key = sys.argv[2]
cfg = W.CONFIGS[key]
s = se.concatenate(W.config_input(key), cfg["D"])
c = se.context(0)
print("library", N.LIB_PATH, flush=True)

if mode == "dump":
    out = sys.argv[3]
    cap = 120 * cfg["nr"]
    buf = (N.TraceRec * cap)()
    tr = N.Trace(C.cast(buf, C.c_void_p), cap, 0)
    k = C.c_size_t()
    kc = 40
    imfs = np.zeros((kc, s.size))
    res = np.zeros(s.size)
    c.run("semd_decompose", 1, s.ctypes.data_as(N._dp), s.size, C.byref(N.SiftCfg(0.2, cfg["max_sift_iters"], cfg["max_imfs"])),
          C.byref(N.EnsCfg(0.2, cfg["nr"], 0, 0)), imfs.ctypes.data_as(N._dp), kc, C.byref(k), res.ctypes.data_as(N._dp),
          None, C.byref(tr))
    assert tr.count <= cap, tr.count
    rec = np.frombuffer(C.string_at(buf, tr.count * C.sizeof(N.TraceRec)), dtype=DT).copy()
    K = int(k.value)
    np.savez(out + ".npz", trace=rec)
    np.save(out + ".npy", np.concatenate([imfs[:K], res[None]]))
    print("K", K, "records", rec.size, "stats", c.stats(), flush=True)
    sys.exit(0)

# mode == "real": the golden realizations
import torch
GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "golden")
arrs = dict(np.load(os.path.join(GOLDEN, "ensembles.npz")))
ms = arrs[f"{key}_real_m"].tolist()
Ks = arrs[f"{key}_real_K"]
off_k = np.concatenate([[0], np.cumsum(Ks)])
tr_all = arrs[f"{key}_real_trace"]
idx = torch.from_numpy(arrs[f"{key}_real_sample_idx"].astype(np.int64)).cuda()
d_x = torch.from_numpy(s).cuda()
n = s.size
cnt = {"K": 0, "counts": 0, "trace": 0, "norms": 0, "values_exact": 0}
worst = 0.0
for j, m in enumerate(ms):
    sums = torch.empty((40, n), dtype=torch.float64, device="cuda")
    cap = 2000
    buf = (N.TraceRec * cap)()
    tr = N.Trace(C.cast(buf, C.c_void_p), cap, 0)
    k = C.c_size_t()
    c.run("semd_eemd_partial_traced_device", C.c_void_p(d_x.data_ptr()), n, C.byref(N.SiftCfg(0.2, 300, 0)),
          C.byref(N.EnsCfg(0.2, 1000, 0, 0)), m, m + 1, C.c_void_p(sums.data_ptr()), 40, C.byref(k), C.byref(tr))
    rec = np.frombuffer(C.string_at(buf, tr.count * C.sizeof(N.TraceRec)), dtype=DT).copy()
    imfs = sums[:k.value]
    K = int(Ks[j])
    gold_tr = np.sort(tr_all[tr_all["m"] == m], order=["k", "iter"])
    got_tr = np.sort(rec, order=["k", "iter"])
    why = []
    if imfs.shape[0] != K:
        cnt["K"] += 1
        why.append("K %d vs %d" % (imfs.shape[0], K))
    else:
        if not np.array_equal(got_tr, gold_tr):
            cnt["trace"] += 1
            n_ = min(got_tr.size, gold_tr.size)
            jj = next((i for i in range(n_) if got_tr[i] != gold_tr[i]), n_)
            why.append("trace differs from record %d of %d (k=%d iter=%d)" % (jj, gold_tr.size, gold_tr[min(jj, gold_tr.size - 1)]["k"],
                                                                            gold_tr[min(jj, gold_tr.size - 1)]["iter"]))
        norms = torch.linalg.norm(imfs, dim=1).cpu().numpy()
        gold_norms = arrs[f"{key}_real_norms"][off_k[j]:off_k[j + 1]]
        samples = imfs[:, idx].cpu().numpy()
        gold_samples = arrs[f"{key}_real_samples"][off_k[j]:off_k[j + 1]]
        rel = float(np.max(np.abs(norms - gold_norms) / gold_norms))
        srel = float(np.max(np.max(np.abs(samples - gold_samples), axis=1) / (gold_norms / np.sqrt(n))))
        worst = max(worst, srel)
        if rel > 1e-9:
            cnt["norms"] += 1
            why.append("norm rel %.2e" % rel)
        if np.array_equal(samples, gold_samples):
            cnt["values_exact"] += 1
    if why:
        print("m", m, why, flush=True)
print(key, "realizations", len(ms), "mismatches:", cnt, "worst sampled |diff| / rms %.2e" % worst, flush=True)
