"""Dev probe: is realization m of C5 deterministic across call sequences?"""
import sys, time, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W, _native as N
from oracle.ffi import Oracle

m = int(sys.argv[1]) if len(sys.argv) > 1 else 793
imfs = int(sys.argv[2]) if len(sys.argv) > 2 else 0
s_h = se.concatenate(W.sine_variates(), 64)
s = torch.from_numpy(s_h).cuda()
n = s.numel()
c = se.context()
sums = torch.zeros((256, n), dtype=torch.float64, device="cuda")
k = C.c_size_t()
o = Oracle()


def part(tag):
    t = time.time()
    rc = c.lib.semd_eemd_partial_device(c.ptr, C.c_void_p(s.data_ptr()), n, C.byref(N.SiftCfg(0.2, 300, imfs)),
                                        C.byref(N.EnsCfg(0.2, 1000, 0, 0)), m, m + 1, C.c_void_p(sums.data_ptr()),
                                        256, C.byref(k))
    st = c.stats()
    h = float(sums[:max(1, k.value)].sum().item()) if rc == 0 else None
    print(tag, "rc", rc, "K", k.value, "sifted", st["sifted_samples"], "steps", st["steps"], "sum", h,
          "%.1fs" % (time.time() - t), c.lib.semd_last_error().decode()[:200] if rc else "", flush=True)


print("std gpu %r oracle %r" % (se.signal_std(s_h), o.signal_std(s_h)), flush=True)
for i in range(3):
    part("fresh%d" % i)
w = se.white_noise(n, o.derive_seed(0, m))
c.set_noise_override(w[None, :])
try:
    g = se.decompose_full(s_h, "eemd", nr=1, max_imfs=imfs)
    print("override K", g["imfs"].shape[0], "sifted", g["stats"]["sifted_samples"], flush=True)
except Exception as e:  # noqa: BLE001
    print("override failed", str(e)[:200], flush=True)
finally:
    c.set_noise_override(None)
for i in range(3):
    part("after%d" % i)
print("std gpu %r" % se.signal_std(s_h), flush=True)
