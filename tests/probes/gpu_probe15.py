"""Dev probe: k_solve per-phase cycle profile (debug bit 1) on C5 realizations."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W, _native as N
key = sys.argv[1] if len(sys.argv) > 1 else "c5"
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 6
s = torch.from_numpy(se.concatenate(W.config_input(key), W.CONFIGS[key]["D"])).cuda()
n = s.numel()
c = se.context()
sums = torch.zeros((64, n), dtype=torch.float64, device="cuda")
k = C.c_size_t()
def run():
    c.check(c.lib.semd_eemd_partial_device(c.ptr, C.c_void_p(s.data_ptr()), n, C.byref(N.SiftCfg(0.2, 300, 0)),
                                           C.byref(N.EnsCfg(0.2, nr, 0, 0)), 0, nr, C.c_void_p(sums.data_ptr()), 64, C.byref(k)))
run()
c.lib.semd_set_debug(c.ptr, 2)
buf = (C.c_uint64 * 16)()
c.lib.semd_solve_profile(c.ptr, buf)  # reset
run()
c.check(c.lib.semd_solve_profile(c.ptr, buf))
c.lib.semd_set_debug(c.ptr, 0)
v = list(buf)
blocks = max(1, v[10])
names = ["setup", "RHS+table xy", "phaseA", "phaseB", "1/d+phaseC", "phaseD", "outputs"]
tot = sum(v[:7]) + v[11] + v[12]
print(f"{'knot loads':14s} {v[11] / blocks:10.0f} cycles/block  {100 * v[11] / max(1, tot):5.1f}%")
print(f"{'H, 1/H':14s} {v[12] / blocks:10.0f} cycles/block  {100 * v[12] / max(1, tot):5.1f}%")
print("blocks", blocks, "B rounds/block %.2f" % (v[8] / blocks), "D rounds/block %.2f" % (v[9] / blocks))
for i, nm in enumerate(names):
    print(f"{nm:14s} {v[i] / blocks:10.0f} cycles/block  {100 * v[i] / max(1, tot):5.1f}%")
