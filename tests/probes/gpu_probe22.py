"""Dev probe: the resident engine's per-phase SM cycles (debug bit 1) on C1-C3.
    python tests/probes/gpu_probe22.py [configs...]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W

keys = sys.argv[1:] or ["c1", "c2", "c3"]
c = se.context()
names = ["detect", "tables", "solve", "eval", "sums", "imf", "input", "-", "s.rhs", "s.fwd", "s.back", "s.table", "s.rcp", "-", "-", "-"]
for key in keys:
    cfg = W.CONFIGS[key]
    s = se.concatenate(W.config_input(key), cfg["D"])
    c.check(c.lib.semd_set_engine(c.ptr, 2))
    se.decompose_full(s, cfg["algo"], max_sift_iters=cfg["max_sift_iters"], max_imfs=cfg["max_imfs"], nr=cfg["nr"])
    c.check(c.lib.semd_set_debug(c.ptr, 2))
    prof = (C.c_uint64 * 16)()
    c.check(c.lib.semd_resident_profile(c.ptr, prof))
    t = time.perf_counter()
    d = se.decompose_full(s, cfg["algo"], max_sift_iters=cfg["max_sift_iters"], max_imfs=cfg["max_imfs"], nr=cfg["nr"])
    el = time.perf_counter() - t
    c.check(c.lib.semd_resident_profile(c.ptr, prof))
    c.check(c.lib.semd_set_debug(c.ptr, 0))
    st = d["stats"]
    sifts = st["sift_iterations"]
    tot = sum(prof)
    print(f"{key}: wall {el*1e3:.2f} ms, jobs {st['resident_jobs']}, sifts {sifts}, total CTA cycles {tot:.3e} "
          f"({tot / 1.9e9 * 1e3 / 148:.2f} ms per SM if spread over 148)")
    print("   per sift (cycles): " + "  ".join(f"{n} {p / max(1, sifts):.0f}" for n, p in zip(names, prof)))
