import sys, json
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2511_16592_b200 import abi, engine
name = sys.argv[1]
e, t = abi.config(name)
t.iterations = 10**6
tr = engine.Trainer(e, t)
tr.run(0, 2); tr.synchronize()
L = engine.lib()
tr.phase_timers(1)
tr.run(2, 1); tr.synchronize()
out = np.zeros(16, dtype=np.int64)
L.gfnx_phase_timers(tr.h, 2, out.ctypes.data, 16)
names = ["bld_wait_full", "bld_build", "mma_wait_full", "mma_wait_built", "prod_wait_empty", "stages", "cta_total", "ctas"]
for base, lab in ((0, "onehot"), (8, "dense")):
    v = out[base:base + 8]
    if v[7] == 0: continue
    st = max(v[5], 1)
    print(lab, {n: round(float(v[i]) / st / 1965, 3) for i, n in enumerate(names[:5])}, "stages/cta", v[5] / v[7], "cta_ms", v[6] / v[7] / 1965e3)
