"""Dev probe: one wave of C5 for kernel-level timing (ncu launch list)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W
x5 = W.sine_variates()
s5 = se.concatenate(x5, 64)
nr = int(sys.argv[1]) if len(sys.argv) > 1 else 3
t = time.time(); d = se.decompose_full(s5, "eemd", nr=nr); el = time.time() - t
st = d["stats"]
print("C5 nr", nr, "time", el, "rate %.3e" % (st["sifted_samples"] / el), st, flush=True)
