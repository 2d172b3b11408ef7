#!/usr/bin/env python
"""Phase clocks of the persistent lockstep rollout (thread 0 of each CTA, averaged)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16592_b200 import abi, engine  # noqa: E402

e, t = abi.config(sys.argv[1] if len(sys.argv) > 1 else "ising_tb_b32768")
t.iterations = 1_000_000
tr = engine.Trainer(e, t, device=0)
tr.run(0, 2)
tr.synchronize()
tr.phase_timers(1)
tr.profile(True)
tr.run(2, 3)
tr.synchronize()
ph = tr.phase_timers(2)
names = list(ph.keys())
steps = e.is_side * e.is_side if hasattr(e, "is_side") else 1
for k, n in zip(range(3), ("layer1", "hidden", "head_sample")):
    print(n, round(ph[names[k]] / 3 / 148 / steps / 1965.0, 2), "us per step per CTA")
for n in ("persist_hid_wimg", "persist_hid_mma", "persist_hid_epi"):
    print(" ", n, round(ph[n] / 3 / 148 / steps / 1965.0, 2), "us per step per CTA")
print("persist ms/launch", tr.profile_read().get("k_ls_persist", (0, 1))[0] / 3)
tr.close()
