import sys; sys.path.insert(0,'.')
import numpy as np
import paper_2106_15319_b200 as se
from oracle.ffi import Oracle
from paper_2106_15319_b200 import workloads as W
o = Oracle()
x = W.pickup_signals()
s = se.concatenate(x, 50)
c = se.context()
key = ["task", "m", "k", "iter"]
oi, ores, _, otr = o.decompose(s, 1, imfs=10, nr=8, trace_cap=4096)
for eng in (1, 2):
    c.check(c.lib.semd_set_engine(c.ptr, eng))
    d = se.decompose_full(s, "eemd", max_imfs=10, nr=8, trace_cap=4096)
    a = np.sort(d["trace"], order=key); b = np.sort(otr, order=key)
    print("engine", eng, "n", len(a), len(b), "count", d["trace_count"], "equal", np.array_equal(a, b), "imfs", d["imfs"].shape, oi.shape,
          "maxdiff", np.abs(d["imfs"] - oi).max() if d["imfs"].shape == oi.shape else None)
    if not np.array_equal(a, b):
        sa = set(map(tuple, a.tolist())); sb = set(map(tuple, b.tolist()))
        print(" only gpu", sorted(sa - sb)[:5]); print(" only ref", sorted(sb - sa)[:5])
