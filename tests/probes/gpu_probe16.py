"""Dev probe: C3 (CEEMDAN) wall time vs engine steps/waves."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W
s = se.concatenate(W.config_input("c3"), 50)
for _ in range(3):
    t = time.time()
    d = se.decompose_full(s, "ceemdan", max_sift_iters=5000, nr=500)
    el = time.time() - t
    st = d["stats"]
    print("c3 wall %.1f ms" % (el * 1e3), "K", d["imfs"].shape[0], "steps", st["steps"], "waves", st["waves"],
          "launches", st["kernel_launches"], "sifted %.3e" % st["sifted_samples"], flush=True)
