"""Dev probe: one C4 decomposition (NR=100) for kernel-level timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W
s = se.concatenate(W.image_batch(), 10)
nr = int(sys.argv[1]) if len(sys.argv) > 1 else 100
se.decompose_full(s, "eemd", nr=4)
t = time.time(); d = se.decompose_full(s, "eemd", nr=nr); el = time.time() - t
st = d["stats"]
print("C4 nr", nr, "time", el, "rate %.3e" % (st["sifted_samples"] / el), st, flush=True)
