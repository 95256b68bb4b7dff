"""Workload for the bounds-checked library (tests/test_gpu_checked.py, SEMD_LIB=libsemd_b200_checked.so):
both engines, every decomposition kind, the repair paths (forced solve replays / hazards, sequential SD
sums), plateaus, multi-block solves, serial / slicewise drivers. A failed SEMD_ASSERT traps the kernel,
the call raises, and the process exits non-zero."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2106_15319_b200 as se

c = se.context()
rng = np.random.default_rng(3)
short = np.sin(np.arange(3000) * 0.05) + 0.3 * rng.standard_normal(3000)
long_ = np.sin(np.arange(40000) * 0.01) + 0.3 * rng.standard_normal(40000)  # multi-block solves
for engine in (2, 1):  # resident, lockstep
    c.check(c.lib.semd_set_engine(c.ptr, engine))
    for debug in (0, 1 | 4):  # plain; forced replays / hazards + sequential SD sums
        c.check(c.lib.semd_set_debug(c.ptr, debug))
        se.decompose(short, "emd")
        se.decompose(short, "eemd", nr=6, max_imfs=4)
        se.decompose(short[:1500], "ceemdan", nr=4, max_imfs=3)
        se.decompose(np.round(short * 3) / 3, "emd", max_imfs=3)  # plateaus
    c.check(c.lib.semd_set_debug(c.ptr, 0))
    m = rng.standard_normal((300, 4))
    se.serial_decompose(m, 40, "eemd", nr=3)
    se.slicewise_decompose(m, "eemd", nr=2)
c.check(c.lib.semd_set_engine(c.ptr, 0))
se.decompose(long_, "emd", max_imfs=4)
se.decompose(long_, "eemd", nr=3, max_imfs=3)
print("checked workload done")
