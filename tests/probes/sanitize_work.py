"""Workload for compute-sanitizer: the smoke decomposition plus short EEMD / CEEMDAN / serial /
slicewise runs exercising every engine kernel (multi-block solve, plateau paths, capacity retry)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

import __graft_entry__ as g
import paper_2106_15319_b200 as se

g.smoke()
rng = np.random.default_rng(5)
x = np.sin(np.arange(5000) * 0.05) + 0.3 * rng.standard_normal(5000)
se.decompose(x, "emd")
se.decompose(x, "ceemdan", nr=4)
se.decompose(np.round(x * 3) / 3, "eemd", nr=3)  # plateaus
m = rng.standard_normal((300, 4))
se.serial_decompose(m, 40, "eemd", nr=3)
se.slicewise_decompose(m, "eemd", nr=2)
print("sanitize workload done")
