#!/usr/bin/env python
"""Iteration time with and without the per-kernel CUDA-event brackets (profile mode)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16592_b200 import abi, engine  # noqa: E402

e, t = abi.config("hypergrid_db_b65536")
t.iterations = 1_000_000
tr = engine.Trainer(e, t, device=0)
tr.run(0, 5)
snap = (tr.params(), tr.adam_state())
for prof in (False, True, False, True):
    tr.set_params(*snap[0])
    tr.set_adam_state(*snap[1])
    tr.synchronize()
    tr.profile(prof)
    tr.event_record(0)
    tr.run(5, 20)
    tr.event_record(1)
    tr.synchronize()
    print("profile" if prof else "plain  ", round(tr.event_elapsed(0, 1) / 20, 4), "ms/iter")
    tr.profile(False)
tr.close()
