"""Dev probe: a full C5 decomposition (NR=1000 by default) through semd_decompose_device with the
per-kernel device spans, steps, waves and wall time -- where the bench step's time goes.
    python tests/probes/gpu_probe19.py [config] [nr]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch

import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import _native as N
from paper_2106_15319_b200 import workloads as W

key = sys.argv[1] if len(sys.argv) > 1 else "c5"
nr = int(sys.argv[2]) if len(sys.argv) > 2 else W.CONFIGS[key]["nr"]
cfg = W.CONFIGS[key]
s = torch.from_numpy(se.concatenate(W.config_input(key), cfg["D"])).cuda()
n = s.numel()
c = se.context()
imfs = torch.empty((40, n), dtype=torch.float64, device="cuda")
res = torch.empty(n, dtype=torch.float64, device="cuda")
k = C.c_size_t()
ms = (C.c_double * 5)()
strips = (C.c_uint64 * 4)()
sc = N.SiftCfg(0.2, cfg["max_sift_iters"], cfg["max_imfs"])
for rep in range(2):
    c.run("semd_kernel_spans", ms, strips)
    torch.cuda.synchronize()
    t = time.time()
    c.run("semd_decompose_device", 1, C.c_void_p(s.data_ptr()), n, C.byref(sc), C.byref(N.EnsCfg(0.2, nr, 0, 0)),
          C.c_void_p(imfs.data_ptr()), 40, C.byref(k), C.c_void_p(res.data_ptr()))
    torch.cuda.synchronize()
    el = time.time() - t
    st = c.stats()
    c.run("semd_kernel_spans", ms, strips)
    names = ["solve", "eval", "scan", "compact", "final"]
    print(key, "nr", nr, "wall %.1f ms" % (el * 1e3), "steps", st["steps"], "waves", st["waves"], "slots", st["slots"],
          "sifted %.3e" % st["sifted_samples"], "rate %.3e" % (st["sifted_samples"] / el), flush=True)
    print("   spans ms: " + "  ".join("%s %.1f" % (a, b) for a, b in zip(names, ms)), " sum %.1f" % sum(ms),
          " other %.1f" % (el * 1e3 - sum(ms)), flush=True)
