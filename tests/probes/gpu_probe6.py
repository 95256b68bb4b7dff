"""Dev probe: device-API EEMD (like bench) host vs device time, with per-phase host timing."""
import sys, time, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W, _native as N
key = sys.argv[1] if len(sys.argv) > 1 else "c4"
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 100
x = W.config_input(key)
D = W.CONFIGS[key]["D"]
s = torch.from_numpy(se.concatenate(x, D)).cuda()
n = s.numel()
c = se.context()
sums = torch.zeros((64, n), dtype=torch.float64, device="cuda")
k = C.c_size_t()
def run(nr):
    c.check(c.lib.semd_eemd_partial_device(c.ptr, C.c_void_p(s.data_ptr()), n, C.byref(N.SiftCfg(0.2, 300, 0)),
                                           C.byref(N.EnsCfg(0.2, nr, 0, 0)), 0, nr, C.c_void_p(sums.data_ptr()), 64,
                                           C.byref(k)))
run(4)
for nr_ in (nr, nr):
    torch.cuda.synchronize()
    t = time.time(); run(nr_); torch.cuda.synchronize(); el = time.time() - t
    st = c.stats()
    print(key, "nr", nr_, "wall %.1f ms" % (el * 1e3), "steps", st["steps"], "waves", st["waves"], "sifted %.3e" % st["sifted_samples"],
          "rate %.3e" % (st["sifted_samples"] / el), flush=True)
