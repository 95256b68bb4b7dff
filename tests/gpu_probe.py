"""Quick GPU probe (dev aid): parity of the engine against the oracle on C1 and small cases."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2106_15319_b200 as se
from oracle.ffi import Oracle
from tests.golden.inputs import pickup_serialized, test_rng_signal
o = Oracle()
def srt(t):
    return np.sort(t, order=["task", "m", "k", "iter"])
def cmp(name, a, b):
    print(name, "K", a[0].shape[0], b[0].shape[0], "imfs_eq", a[0].shape == b[0].shape and np.array_equal(a[0], b[0]),
          "res_eq", np.array_equal(a[1], b[1]), flush=True)
x = test_rng_signal(11, 600)
t = time.time(); d = se.decompose_full(x, "emd", trace_cap=10000); print("emd600", time.time() - t)
od = o.emd(x, trace_cap=10000)
cmp("emd600", (d["imfs"], d["residue"]), od)
print("counts", d["sift_counts"], od[2], "trace eq", np.array_equal(srt(d["trace"]), srt(od[3])), d["stats"])
s = pickup_serialized(o, 50)
t = time.time(); d = se.decompose_full(s, "emd", max_sift_iters=1000, trace_cap=10000); print("C1", time.time() - t)
od = o.emd(s, iters=1000, trace_cap=10000)
cmp("C1", (d["imfs"], d["residue"]), od)
print("counts", d["sift_counts"], od[2], "trace eq", np.array_equal(srt(d["trace"]), srt(od[3])), d["stats"])
for D in (50,):
    s = pickup_serialized(o, D)
    t = time.time(); d = se.decompose_full(s, "eemd", max_imfs=10, nr=100, trace_cap=100000); el = time.time() - t
    od = o.decompose(s, 1, imfs=10, nr=100, trace_cap=100000)
    rel = [np.linalg.norm(d["imfs"][k] - od[0][k]) / np.linalg.norm(od[0][k]) for k in range(min(len(od[0]), len(d["imfs"])))]
    print("C2 D", D, "time", el, "K", d["imfs"].shape[0], od[0].shape[0], "max relL2", max(rel), "trace eq",
          np.array_equal(srt(d["trace"]), srt(od[3])), len(d["trace"]), len(od[3]), d["stats"], flush=True)
    # bit-exact with injected noise
    c = se.context()
    noise = np.stack([o.white_noise(s.size, o.derive_seed(0, m)) for m in range(100)])
    c.set_noise_override(noise)
    d2 = se.decompose_full(s, "eemd", max_imfs=10, nr=100)
    c.set_noise_override(None)
    print("C2 injected noise bit-exact:", np.array_equal(d2["imfs"], od[0]), np.array_equal(d2["residue"], od[1]))
    w = se.white_noise(1001, 7); ow = o.white_noise(1001, 7)
    print("noise max ulp diff", np.max(np.abs(w - ow) / np.spacing(np.abs(ow))), "n differing", np.sum(w != ow))
