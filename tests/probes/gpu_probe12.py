"""Dev probe: fresh-arena vs reused-arena determinism (C4 EEMD), hazards."""
import sys, os, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2106_15319_b200 as se
from paper_2106_15319_b200 import workloads as W

key = sys.argv[1] if len(sys.argv) > 1 else "c4"
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 100
s = se.concatenate(W.config_input(key), W.CONFIGS[key]["D"])


def h(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


res = []
for tag, kw in [("fresh", {}), ("reuse1", {}), ("reuse2", {}), ("slots4", {"slots": 4}), ("after4", {})]:
    ctx = se.context()
    if "slots" in kw:
        ctx.set_max_slots(kw["slots"])
    d = se.decompose_full(s, "eemd", nr=nr)
    ctx.set_max_slots(0)
    st = d["stats"]
    print(tag, "K", d["imfs"].shape[0], "hash", h(d["imfs"]), "sifted", st["sifted_samples"], "hazards",
          st["solve_hazards"], "slots", st["slots"], flush=True)
    res.append(d["imfs"])
for i in range(1, len(res)):
    if res[i].shape == res[0].shape and not np.array_equal(res[i], res[0]):
        diff = np.nonzero(np.any(res[i] != res[0], axis=1))[0]
        print("run", i, "differs in IMF rows", diff.tolist())
