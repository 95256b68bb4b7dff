"""Dev probe: one C5 realization (argv m) -- determinism + first trace divergence vs the oracle."""
import sys, time, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W, _native as N
from oracle.ffi import Oracle  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 793
x = W.config_input("c5")
s_h = se.concatenate(x, 64)
s = torch.from_numpy(s_h).cuda()
n = s.numel()
c = se.context()
sums = torch.zeros((64, n), dtype=torch.float64, device="cuda")
k = C.c_size_t()


def part(m0, m1):
    rc = c.lib.semd_eemd_partial_device(c.ptr, C.c_void_p(s.data_ptr()), n, C.byref(N.SiftCfg(0.2, 300, 0)),
                                        C.byref(N.EnsCfg(0.2, 1000, 0, 0)), m0, m1, C.c_void_p(sums.data_ptr()), 64,
                                        C.byref(k))
    return rc, (c.lib.semd_last_error().decode() if rc else c.stats()["steps"])


for r in [(m - 1, m + 2), (m, m + 1)]:
    print("partial", r, part(*r), flush=True)

o = Oracle()
w = se.white_noise(n, o.derive_seed(0, m))
c.set_noise_override(w[None, :])
try:
    g = se.decompose_full(s_h, "eemd", nr=1, trace_cap=200000, max_imfs=20)
except Exception as e:  # noqa: BLE001
    print("gpu override run failed:", e)
    g = None
finally:
    c.set_noise_override(None)
beta = 0.2 * se.signal_std(s_h)
t = time.time()
oi = o.emd(s_h + beta * w, imfs=20, trace_cap=200000)
print("oracle K", oi[0].shape[0], "time %.1f" % (time.time() - t), flush=True)
ot = oi[3]
if g is not None:
    gt = g["trace"]
    print("gpu trace count", g["trace_count"], "oracle", len(ot), "K gpu", g["imfs"].shape[0])
    ok = sorted(map(tuple, ot[["k", "iter", "n_max", "n_min", "hash"]].tolist()))
    gk = sorted(map(tuple, gt[["k", "iter", "n_max", "n_min", "hash"]].tolist()))
    for i, (a, b) in enumerate(zip(ok, gk)):
        if a != b:
            print("first diff at", i, "oracle", a, "gpu", b)
            print("context oracle", ok[max(0, i - 3):i + 3])
            print("context gpu", gk[max(0, i - 3):i + 3])
            break
    else:
        print("traces identical over", min(len(ok), len(gk)))
