"""Dev probe: where do speculative-solve hazards occur? (C5 realizations in chunks)"""
import sys, os, time, ctypes as C, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W, _native as N

key = sys.argv[1] if len(sys.argv) > 1 else "c5"
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 30
s = torch.from_numpy(se.concatenate(W.config_input(key), W.CONFIGS[key]["D"])).cuda()
n = s.numel()
c = se.context()
sums = torch.zeros((64, n), dtype=torch.float64, device="cuda")
k = C.c_size_t()
allrec = []
t0 = time.time()
for m0 in range(0, nr, chunk):
    m1 = min(nr, m0 + chunk)
    c.check(c.lib.semd_eemd_partial_device(c.ptr, C.c_void_p(s.data_ptr()), n, C.byref(N.SiftCfg(0.2, 300, 0)),
                                           C.byref(N.EnsCfg(0.2, nr, 0, 0)), m0, m1, C.c_void_p(sums.data_ptr()), 64,
                                           C.byref(k)))
    cnt = C.c_size_t()
    c.check(c.lib.semd_hazard_log(c.ptr, None, 0, C.byref(cnt)))
    if cnt.value:
        buf = np.zeros(cnt.value * 8, dtype=np.int32)
        c.check(c.lib.semd_hazard_log(c.ptr, buf.ctypes.data, cnt.value, C.byref(cnt)))
        allrec.append(buf.reshape(-1, 8))
    print("chunk", m0, "hazards", c.stats()["solve_hazards"], flush=True)
print("time %.1f" % (time.time() - t0))
if allrec:
    r = np.concatenate(allrec)
    print("records", len(r))
    print("by kind", collections.Counter(r[:, 7].tolist()))
    print("by k", sorted(collections.Counter(r[:, 1].tolist()).items()))
    print("by iter", sorted(collections.Counter(r[:, 2].tolist()).items())[:20])
    print("knots quantiles", np.percentile(r[:, 4], [0, 10, 50, 90, 100]).tolist())
    print("block/nb samples", r[:20, 5].tolist(), r[:20, 6].tolist())
    print("distinct (m,k,iter,side)", len({tuple(x) for x in r[:, :4].tolist()}))
    print("first rows", r[:10].tolist())
