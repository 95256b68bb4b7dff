"""Dev probe: signal_std of the C5 / C4 serialized signals -- the parallel kernels against the single-thread
kernel (debug bit 32): equal bits, host wall time of semd_signal_std (the upload is common to both) and the
segments that took the slow path.
    python tests/probes/gpu_probe26.py [configs]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W

c = se.context()
for key in (sys.argv[1:] or ["c4", "c5"]):
    s = se.concatenate(W.config_input(key), W.CONFIGS[key]["D"])
    out = {}
    for name, bits in (("single", 32), ("parallel", 0), ("single", 32), ("parallel", 0)):
        c.run("semd_set_debug", bits)
        t = time.time()
        v = se.signal_std(s)
        el = time.time() - t
        buf = (C.c_uint64 * 3)()
        c.run("semd_std_stats", buf)
        out[name] = v
        print(key, "L", s.size, name, "std", v.hex(), "%.2f ms" % (el * 1e3), "slow segments", list(buf), flush=True)
    c.run("semd_set_debug", 0)
    assert out["single"] == out["parallel"]
