"""Dev probe: C3/C2 step time through semd_decompose_device -- host wall vs device-timed (semd_timer), timing on/off."""
import ctypes as C, sys, time, os
sys.path.insert(0, '.')
import numpy as np
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import _native as N, workloads as W
c = se.context()
for key in ("c3", "c2"):
    cfg = W.CONFIGS[key]
    s = se.concatenate(W.config_input(key), cfg["D"])
    L = s.size
    d_s = C.c_void_p(); c.run("semd_device_alloc", L * 8, C.byref(d_s)); c.run("semd_memcpy", d_s, s.ctypes.data_as(C.c_void_p), L * 8)
    d_i = C.c_void_p(); c.run("semd_device_alloc", 32 * L * 8, C.byref(d_i))
    d_r = C.c_void_p(); c.run("semd_device_alloc", L * 8, C.byref(d_r))
    k = C.c_size_t()
    algo = {"emd": 0, "eemd": 1, "ceemdan": 2}[cfg["algo"]]
    scfg = N.SiftCfg(0.2, cfg["max_sift_iters"], cfg["max_imfs"]); ens = N.EnsCfg(0.2, cfg["nr"], 0, 0)
    for timing in (0, 1):
        c.set_timing(bool(timing))
        for _ in range(3): c.run("semd_decompose_device", algo, d_s, L, C.byref(scfg), C.byref(ens), d_i, 32, C.byref(k), d_r)
        ts = []
        for _ in range(10):
            t = time.perf_counter(); c.run("semd_decompose_device", algo, d_s, L, C.byref(scfg), C.byref(ens), d_i, 32, C.byref(k), d_r); ts.append(time.perf_counter() - t)
        ms = C.c_double(); c.run("semd_timer_start")
        for _ in range(10): c.run("semd_decompose_device", algo, d_s, L, C.byref(scfg), C.byref(ens), d_i, 32, C.byref(k), d_r)
        c.run("semd_timer_stop", C.byref(ms))
        print(key, "timing", timing, "host wall min %.3f med %.3f ms" % (1e3 * min(ts), 1e3 * sorted(ts)[5]), "device-timed %.3f ms/step" % (ms.value / 10), "eval_ms", c.stats()["eval_ms"], flush=True)
