"""Dev probe: device noise cost -- semd_white_noise of one C5-length realization (MT19937-64 +
the glibc-exact Box-Muller), timed with the context timer."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

import paper_2106_15319_b200 as se

c = se.context()
n = 17_039_296
out = np.zeros(n)
for rep in range(3):
    c.run("semd_timer_start")
    c.run("semd_white_noise", n, C.c_uint64(7 + rep), 1.0, out.ctypes.data_as(C.POINTER(C.c_double)))
    ms = C.c_double()
    c.run("semd_timer_stop", C.byref(ms))
    print("white_noise(17M): %.2f ms (incl. D2H of 136 MB)" % ms.value, flush=True)
