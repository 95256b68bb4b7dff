"""Dev probe: C3 (serial-CEEMDAN, NR=500) wall time, steps and per-kernel device spans."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W

s = se.concatenate(W.config_input("c3"), 50)
c = se.context()
ms = (C.c_double * 5)()
strips = (C.c_uint64 * 4)()
for it in range(int(os.environ.get("ITERS", "4"))):
    c.check(c.lib.semd_kernel_spans(c.ptr, ms, strips))
    t = time.time()
    d = se.decompose_full(s, "ceemdan", max_sift_iters=5000, nr=500)
    el = time.time() - t
    st = d["stats"]
    c.check(c.lib.semd_kernel_spans(c.ptr, ms, strips))
    print("c3 wall %.2f ms" % (el * 1e3), "K", d["imfs"].shape[0], "steps", st["steps"], "waves", st["waves"],
          "launches", st["kernel_launches"], "sifted %.3e" % st["sifted_samples"],
          "| spans ms solve %.2f eval %.2f scan %.2f compact %.2f final %.2f (sum %.2f)" % (*ms, sum(ms)), flush=True)
