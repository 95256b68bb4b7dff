"""Dev probe: C5 realizations with device noise vs injected noise (no side-stream generator)."""
import sys, time, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W, _native as N
nr = int(sys.argv[1]) if len(sys.argv) > 1 else 12
s_h = se.concatenate(W.config_input("c5"), 64)
s = torch.from_numpy(s_h).cuda()
n = s.numel()
c = se.context()
sums = torch.zeros((64, n), dtype=torch.float64, device="cuda")
k = C.c_size_t()
def run(tag):
    torch.cuda.synchronize(); t = time.time()
    c.check(c.lib.semd_eemd_partial_device(c.ptr, C.c_void_p(s.data_ptr()), n, C.byref(N.SiftCfg(0.2, 300, 0)),
                                           C.byref(N.EnsCfg(0.2, nr, 0, 0)), 0, nr, C.c_void_p(sums.data_ptr()), 64, C.byref(k)))
    torch.cuda.synchronize(); el = time.time() - t
    st = c.stats()
    print(tag, "wall %.1f ms" % (el * 1e3), "steps", st["steps"], "sifted %.4e" % st["sifted_samples"], "rate %.3e" % (st["sifted_samples"] / el), flush=True)
run("device-noise warm"); run("device-noise")
w = np.stack([se.white_noise(n, se.derive_seed(0, m)) for m in range(nr)])
c.set_noise_override(w)
run("injected warm"); run("injected")
c.set_noise_override(None)
