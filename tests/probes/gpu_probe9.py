"""Dev probe: run an EEMD config's realizations in chunks; report per-chunk steps and any engine stall."""
import sys, time, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W, _native as N
key = sys.argv[1] if len(sys.argv) > 1 else "c5"
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 30
x = W.config_input(key)
D = W.CONFIGS[key]["D"]
s = torch.from_numpy(se.concatenate(x, D)).cuda()
n = s.numel()
c = se.context()
sums = torch.zeros((64, n), dtype=torch.float64, device="cuda")
k = C.c_size_t()
imfs = int(sys.argv[4]) if len(sys.argv) > 4 else 0
passes = int(sys.argv[5]) if len(sys.argv) > 5 else 1
fails = 0
t0 = time.time()
seen = {}
for m0 in [a for _ in range(passes) for a in range(0, nr, chunk)]:
    m1 = min(nr, m0 + chunk)
    rc = c.lib.semd_eemd_partial_device(c.ptr, C.c_void_p(s.data_ptr()), n, C.byref(N.SiftCfg(0.2, 300, imfs)),
                                        C.byref(N.EnsCfg(0.2, nr, 0, 0)), m0, m1, C.c_void_p(sums.data_ptr()), 64,
                                        C.byref(k))
    st = c.stats()
    if rc != 0:
        fails += 1
        print("FAIL", m0, m1, rc, c.lib.semd_last_error().decode(), flush=True)
    else:
        h = float(sums[:k.value].sum().item())
        key = (st["sifted_samples"], k.value, h)
        if m0 in seen and seen[m0] != key:
            print("NONDETERMINISTIC", m0, seen[m0], key, flush=True)
        seen[m0] = key
        print("ok", m0, m1, "steps", st["steps"], "waves", st["waves"], "sifted %.4e" % st["sifted_samples"],
              "K", k.value, "sum %r" % h, flush=True)
print("done fails", fails, "time %.1f" % (time.time() - t0))
