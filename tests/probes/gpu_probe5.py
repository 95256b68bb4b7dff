"""Dev probe: host loop vs device time for one C4 wave."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W
s = se.concatenate(W.image_batch(), 10)
c = se.context()
se.decompose_full(s, "eemd", nr=4)
for nr in (22, 100):
    c.set_timing(True)
    t = time.time(); d = se.decompose_full(s, "eemd", nr=nr); el = time.time() - t
    st = d["stats"]
    print("nr", nr, "wall %.1f ms" % (el * 1e3), "eval_ms %.1f" % st["eval_ms"], "steps", st["steps"], "waves", st["waves"],
          "wall/step %.3f ms" % (el * 1e3 / st["steps"]), flush=True)
    c.set_timing(False)
    t = time.time(); d = se.decompose_full(s, "eemd", nr=nr); el = time.time() - t
    print("   no timing wall %.1f ms" % (el * 1e3), flush=True)
x = np.random.default_rng(0).standard_normal(6250)
t = time.time()
for _ in range(20): se.decompose(x, "emd")
print("small emd x20: %.2f ms each" % ((time.time() - t) / 20 * 1e3))
