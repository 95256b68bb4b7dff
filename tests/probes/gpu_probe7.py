"""Dev probe: determinism of repeated device-API EEMD calls."""
import sys, os, ctypes as C, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W, _native as N
key = sys.argv[1]; nr = int(sys.argv[2]); reps = int(sys.argv[3])
x = W.config_input(key)
s = torch.from_numpy(se.concatenate(x, W.CONFIGS[key]["D"])).cuda()
n = s.numel()
c = se.context()
if len(sys.argv) > 4: c.set_max_slots(int(sys.argv[4]))
sums = torch.zeros((64, n), dtype=torch.float64, device="cuda")
k = C.c_size_t()
for r in range(reps):
    c.check(c.lib.semd_eemd_partial_device(c.ptr, C.c_void_p(s.data_ptr()), n, C.byref(N.SiftCfg(0.2, 300, 0)),
                                           C.byref(N.EnsCfg(0.2, nr, 0, 0)), 0, nr, C.c_void_p(sums.data_ptr()), 64,
                                           C.byref(k)))
    torch.cuda.synchronize()
    st = c.stats()
    h = hashlib.sha256(sums[:k.value].cpu().numpy().tobytes()).hexdigest()[:16]
    print(key, "rep", r, "K", k.value, "steps", st["steps"], "sifted", st["sifted_samples"], "hash", h, flush=True)
