"""Dev probe: per-step device time of bench.py's timed loop on a config (semd_timer around every
step), to look for outlier steps. python tests/probes/gpu_probe25.py [config] [steps]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import _native as N
from paper_2106_15319_b200 import workloads as W

key = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = W.CONFIGS[key]
x = W.config_input(key)
c = se.context()
c.set_timing(True)
M, Nch = x.shape
D = cfg["D"]
L = M * Nch + D * (Nch - 1)
xc = np.ascontiguousarray(x.T)
d_x = C.c_void_p(); c.run("semd_device_alloc", xc.nbytes, C.byref(d_x))
c.run("semd_memcpy", d_x, xc.ctypes.data_as(C.c_void_p), xc.nbytes)
d_s = C.c_void_p(); c.run("semd_device_alloc", L * 8, C.byref(d_s))
c.run("semd_concatenate_device", d_x, M, Nch, D, d_s)
d_i = C.c_void_p(); c.run("semd_device_alloc", 32 * L * 8, C.byref(d_i))
d_r = C.c_void_p(); c.run("semd_device_alloc", L * 8, C.byref(d_r))
k = C.c_size_t()
algo = {"emd": 0, "eemd": 1, "ceemdan": 2}[cfg["algo"]]
scfg = N.SiftCfg(0.2, cfg["max_sift_iters"], cfg["max_imfs"])
ens = N.EnsCfg(0.2, cfg["nr"], 0, 0)
ts = []
for i in range(steps):
    ms = C.c_double()
    c.run("semd_timer_start")
    c.run("semd_decompose_device", algo, d_s, L, C.byref(scfg), C.byref(ens), d_i, 32, C.byref(k), d_r)
    c.run("semd_timer_stop", C.byref(ms))
    ts.append(ms.value)
print(key, "per-step ms:", " ".join("%.2f" % t for t in ts))
