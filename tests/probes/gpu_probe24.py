"""Dev probe: slicewise_decompose (baseline.cpp:5-29) of the pick-up signals (6 channels x 1000) on
both engines: bit-identity and wall time (EMD, EEMD NR=100)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W

c = se.context()
x = W.pickup_signals()
for algo, kw in (("emd", {}), ("eemd", dict(nr=100, max_imfs=10))):
    out = {}
    for eng in (1, 2):
        c.check(c.lib.semd_set_engine(c.ptr, eng))
        se.slicewise_decompose(x, algo, **kw)
        ts = []
        for _ in range(5):
            t = time.perf_counter()
            out[eng] = se.slicewise_decompose(x, algo, **kw)
            ts.append(time.perf_counter() - t)
        print(algo, "lockstep" if eng == 1 else "resident", "ms min %.3f" % (1e3 * min(ts)), "resident_jobs",
              c.stats()["resident_jobs"], flush=True)
    print(algo, "bit-identical:", np.array_equal(out[1].view(np.int64), out[2].view(np.int64)), flush=True)
c.check(c.lib.semd_set_engine(c.ptr, 0))
