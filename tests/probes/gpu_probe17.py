"""Dev probe: per-kernel device spans of the step kernels (semd_kernel_spans) on a config.

    python tests/probes/gpu_probe17.py [config] [nr]
"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import _native as N
from paper_2106_15319_b200 import workloads as W

key = sys.argv[1] if len(sys.argv) > 1 else "c5"
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 62
x = W.config_input(key)
D = W.CONFIGS[key]["D"]
s = torch.from_numpy(se.concatenate(x, D)).cuda()
n = s.numel()
c = se.context()
sums = torch.zeros((64, n), dtype=torch.float64, device="cuda")
k = C.c_size_t()
ms = (C.c_double * 5)()
strips = (C.c_uint64 * 4)()
spec = (C.c_uint64 * 4)()


def run(nr):
    c.check(c.lib.semd_eemd_partial_device(c.ptr, C.c_void_p(s.data_ptr()), n, C.byref(N.SiftCfg(0.2, 300, 0)),
                                           C.byref(N.EnsCfg(0.2, nr, 0, 0)), 0, nr, C.c_void_p(sums.data_ptr()), 64,
                                           C.byref(k)))


run(4)
c.check(c.lib.semd_kernel_spans(c.ptr, ms, strips))
getattr(c.lib, 'semd_spec_stats', lambda *a: 0)(c.ptr, spec)
for _ in range(2):
    torch.cuda.synchronize()
    t = time.time()
    run(nr)
    torch.cuda.synchronize()
    el = time.time() - t
    st = c.stats()
    c.check(c.lib.semd_kernel_spans(c.ptr, ms, strips))
    getattr(c.lib, 'semd_spec_stats', lambda *a: 0)(c.ptr, spec)
    names = ["solve", "eval", "scan", "compact", "final"]
    tot = sum(ms)
    print(key, "nr", nr, "wall %.1f ms" % (el * 1e3), "steps", st["steps"], "waves", st["waves"],
          "sifted %.3e" % st["sifted_samples"], "rate %.3e" % (st["sifted_samples"] / el), flush=True)
    print("   spans ms: " + "  ".join("%s %.1f (%.0f%%)" % (a, b, 100 * b / el / 1e3) for a, b in zip(names, ms)),
          " sum %.1f" % tot, " strips detect %d sift %d" % (strips[0], strips[1]),
          " warp-cycles/strip detect %.0f sift %.0f" % (strips[2] / max(1, strips[0]), strips[3] / max(1, strips[1])),
          flush=True)
    print("   speculative last sifts: run %d, stopped %d, continued %d; lockstep steps %d" % tuple(spec), flush=True)
