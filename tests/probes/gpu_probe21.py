"""Dev probe: resident vs lockstep engine on C1-C3 (bit-identity of IMFs, residue and traces; wall time).
    python tests/probes/gpu_probe21.py [configs...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W

keys = sys.argv[1:] or ["c1", "c2", "c3"]
c = se.context()
key_order = ["task", "m", "k", "iter"]
for key in keys:
    cfg = W.CONFIGS[key]
    s = se.concatenate(W.config_input(key), cfg["D"])
    out = {}
    for eng, name in ((1, "lockstep"), (2, "resident")):
        c.check(c.lib.semd_set_engine(c.ptr, eng))
        d = se.decompose_full(s, cfg["algo"], max_sift_iters=cfg["max_sift_iters"], max_imfs=cfg["max_imfs"],
                              nr=cfg["nr"], trace_cap=200000)
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            se.decompose_full(s, cfg["algo"], max_sift_iters=cfg["max_sift_iters"], max_imfs=cfg["max_imfs"],
                              nr=cfg["nr"])
            ts.append(time.perf_counter() - t)
        out[name] = d
        st = d["stats"]
        print(f"{key} {name:8s} K={d['imfs'].shape[0]} traces={d['trace_count']} sifted={st['sifted_samples']} "
              f"resident_jobs={st['resident_jobs']} hazards={st['solve_hazards']} rechecks={st['sd_rechecks']} "
              f"wall ms min {1e3 * min(ts):.2f} med {1e3 * sorted(ts)[1]:.2f}", flush=True)
    a, b = out["lockstep"], out["resident"]
    same = (a["imfs"].shape == b["imfs"].shape and np.array_equal(a["imfs"].view(np.int64), b["imfs"].view(np.int64))
            and np.array_equal(a["residue"].view(np.int64), b["residue"].view(np.int64)))
    tr = np.array_equal(np.sort(a["trace"], order=key_order), np.sort(b["trace"], order=key_order))
    print(f"{key} bit-identical imfs+residue: {same}  traces equal: {tr}", flush=True)
c.check(c.lib.semd_set_engine(c.ptr, 0))
