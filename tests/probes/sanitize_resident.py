"""Workload for compute-sanitizer on the resident engine: EMD (one job), EEMD (job queue + ordered
accumulation), CEEMDAN (the cooperative k_res_ceemdan with grid barriers), forced replays and the
sequential SD path; optionally (argv[1] == "lockstep") one small lockstep EMD instead."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

import paper_2106_15319_b200 as se

c = se.context()
rng = np.random.default_rng(5)
if len(sys.argv) > 1 and sys.argv[1] == "lockstep":
    c.check(c.lib.semd_set_engine(c.ptr, 1))
    x = np.sin(np.arange(20000) * 0.01) + 0.3 * rng.standard_normal(20000)
    d = se.decompose(x, "emd", max_imfs=3)
    print("lockstep emd K", d["imfs"].shape[0])
else:
    c.check(c.lib.semd_set_engine(c.ptr, 2))
    x = np.sin(np.arange(3000) * 0.05) + 0.3 * rng.standard_normal(3000)
    print("emd K", se.decompose(x, "emd")["imfs"].shape[0])
    print("eemd K", se.decompose(x, "eemd", nr=6, max_imfs=4)["imfs"].shape[0])
    print("ceemdan K", se.decompose(x[:1500], "ceemdan", nr=4, max_imfs=3)["imfs"].shape[0])
    c.check(c.lib.semd_set_debug(c.ptr, 1 | 4))  # forced replays, sequential SD sums
    print("emd (replays, sequential SD) K", se.decompose(np.round(x * 3) / 3, "emd", max_imfs=3)["imfs"].shape[0])
    c.check(c.lib.semd_set_debug(c.ptr, 0))
print("sanitize workload done")
