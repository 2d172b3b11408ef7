#!/usr/bin/env python
"""Per-pass clock totals of k_fast_wgrad (thread 0 of every CTA, averaged over CTAs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16592_b200 import abi, engine  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "hypergrid_db_b65536"
e, t = abi.config(name)
t.iterations = 1_000_000
tr = engine.Trainer(e, t, device=0)
tr.run(0, 20)
tr.synchronize()
tr.phase_timers(1)
tr.profile(True)
tr.run(20, 10)
tr.synchronize()
ph = tr.phase_timers(2)
prof = tr.profile_read()
for k in ("wgrad_pass_a", "wgrad_pass_b", "wgrad_pass_c"):
    print(k, round(ph[k] / 10 / 148 / 1965.0, 1), "us per launch per CTA")
print("k_fast_wgrad ms/launch", prof["k_fast_wgrad"][0] / 10)
tr.close()
