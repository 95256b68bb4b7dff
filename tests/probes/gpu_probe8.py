"""Dev probe: small workload for compute-sanitizer."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W
s = se.concatenate(W.pickup_signals(), 50)
d = se.decompose(s, "eemd", max_imfs=10, nr=8)
e = se.decompose(s, "emd")
x = np.random.default_rng(1).standard_normal(40000)
f = se.decompose(x, "eemd", nr=3)
g = se.decompose(s, "ceemdan", nr=4)
print("ok", d["imfs"].shape, e["imfs"].shape, f["imfs"].shape, g["imfs"].shape)
